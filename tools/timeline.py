"""Diagnostics: per-CTA phase timestamps of the NormProb GEMM on config 2 (prologue / mainloop / epilogue)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2206_13236_b200 as R
b = synth.make_batch(2)
dev = R.batch_to_device(b, "cuda")
d = R.make_dims(b.N, b.T, b.U, b.V, b.J, b.S)
ws = torch.empty(R.rnnt_workspace_bytes(d), dtype=torch.uint8, device="cuda")
o = R.alloc_outputs(d, "cuda")
buf = torch.zeros(1 << 20, dtype=torch.int64, device="cuda")
lib = R.load_library()
for it in range(3):
    lib.rnnt_debug_timeline(ctypes.c_void_p(buf.data_ptr() if it == 2 else 0))
    R.rnnt_simple_loss(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], d, 0.5, o["loss_simple"], o["px_grad"],
                       o["py_grad"], None, None, o["status"], ws)
    torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(-1, 4)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = (t - t0) / 1000.0
print("CTAs", len(t))
print("start  min/med/max us", np.min(rel[:, 0]), np.median(rel[:, 0]), np.max(rel[:, 0]))
print("prolog dur med/max", np.median(rel[:, 1] - rel[:, 0]), np.max(rel[:, 1] - rel[:, 0]))
print("mainloop wait med/max", np.median(rel[:, 2] - rel[:, 1]), np.max(rel[:, 2] - rel[:, 1]))
print("epilogue med/max", np.median(rel[:, 3] - rel[:, 2]), np.max(rel[:, 3] - rel[:, 2]))
print("end max", np.max(rel[:, 3]))
