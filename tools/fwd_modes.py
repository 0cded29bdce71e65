"""Diagnostics: joiner forward kernel time under RNNT_DBG_FWD modes (run once per mode)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2206_13236_b200 as R
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
b = synth.make_batch(cfg)
dev = R.batch_to_device(b, "cuda")
o = R.step(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], dev["enc_proj"], dev["dec_proj"],
           dev["w_out"], dev["b_out"], b.S)
torch.cuda.synchronize()
d = R.make_dims(b.N, b.T, b.U, b.V, b.J, b.S)
ws = torch.empty(R.rnnt_workspace_bytes(d), dtype=torch.uint8, device="cuda")
ids = R.kernel_ids()
kname = sys.argv[2] if len(sys.argv) > 2 else "joiner_fwd_gemm"
times = []
for i in range(12):
    a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); c.record()          # materialise the event handles
    R.rnnt_profile_kernel(ids[kname], a, c)
    R.rnnt_pruned_loss(o["h"], dev["w_out"], dev["b_out"], dev["symbols"], o["ranges"], dev["boundary"], d, 1.0,
                       o["loss_pruned"], o["d_enc"], o["d_dec"], o["d_w"], o["d_b"], o["status"], ws)
    R.rnnt_profile_kernel(0)
    torch.cuda.synchronize()
    times.append(a.elapsed_time(c) * 1000)
print(f"cfg {cfg} {kname} mode {os.environ.get('RNNT_DBG_FWD', '0')}: median {statistics.median(times[2:]):.1f} us")
