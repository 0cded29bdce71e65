"""Diagnostics: live time of every library kernel inside one step (serial streams, events on the launch
stream), sorted; the sum against the step time.

    python tools/all_kernels.py <config>"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth, paper_2206_13236_b200 as R
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
b = synth.make_batch(cfg)
dev = R.batch_to_device(b, "cuda")
ids = R.kernel_ids()
args = (dev["am"], dev["lm"], dev["symbols"], dev["boundary"], dev["enc_proj"], dev["dec_proj"], dev["w_out"],
        dev["b_out"], b.S)
for _ in range(3):
    R.step(*args, overlap=False)
torch.cuda.synchronize()
st = []
for i in range(10):
    a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    R.step(*args, overlap=False)
    c.record()
    torch.cuda.synchronize()
    st.append(a.elapsed_time(c) * 1000)
res = []
for name, kid in ids.items():
    times = []
    for i in range(5):
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); c.record()
        R.rnnt_profile_kernel(kid, a, c)
        R.step(*args, overlap=False)
        R.rnnt_profile_kernel(0)
        torch.cuda.synchronize()
        try:
            times.append(a.elapsed_time(c) * 1000)
        except RuntimeError:
            times.append(0.0)
    t = statistics.median(times)
    if t > 0.05:
        res.append((t, name))
res.sort(reverse=True)
tot = sum(t for t, _ in res)
print(f"cfg {cfg}: serial step {statistics.median(st):.1f} us, kernel sum {tot:.1f} us")
for t, n in res:
    print(f"  {n:24s} {t:9.1f} us  {100 * t / tot:5.1f}%")
