"""Diagnostics: live time of one library kernel inside the whole step (events on its launch stream).

    python tools/kernel_time.py <config> <kernel-name>"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth, paper_2206_13236_b200 as R
cfg, kname = int(sys.argv[1]), sys.argv[2]
b = synth.make_batch(cfg)
dev = R.batch_to_device(b, "cuda")
ids = R.kernel_ids()
args = (dev["am"], dev["lm"], dev["symbols"], dev["boundary"], dev["enc_proj"], dev["dec_proj"], dev["w_out"],
        dev["b_out"], b.S)
for _ in range(3):
    R.step(*args)
torch.cuda.synchronize()
times = []
for i in range(10):
    a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); c.record()
    R.rnnt_profile_kernel(ids[kname], a, c)
    R.step(*args, overlap=False)
    R.rnnt_profile_kernel(0)
    torch.cuda.synchronize()
    times.append(a.elapsed_time(c) * 1000)
print(f"cfg {cfg} {kname}: median {statistics.median(times):.1f} us")
