"""Diagnostics (diagnostics build: RNNT_LIB=paper_2206_13236_b200/librnnt_b200_diag.so): per-CTA phase
timestamps of the normaliser GEMM (gemm3<NormProb>) in rnnt_simple_loss (no grads) on a config:
start, prologue done, accumulator full (mainloop done), epilogue done."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2206_13236_b200 as R
b = synth.make_batch(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
dev = R.batch_to_device(b, "cuda")
d = R.make_dims(b.N, b.T, b.U, b.V, b.J, b.S)
o = R.alloc_outputs(d, "cuda")
ws = torch.empty(R.rnnt_workspace_bytes(d), dtype=torch.uint8, device="cuda")
buf = torch.zeros((8 << 20) // 8, dtype=torch.int64, device="cuda")
lib = R.load_library()
for it in range(4):
    lib.rnnt_debug_timeline(ctypes.c_void_p(buf.data_ptr() if it == 3 else 0))
    R.rnnt_simple_loss(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], d, 0.5, o["loss_simple"],
                       o["px_grad"], o["py_grad"], None, None, o["status"], ws)
    torch.cuda.synchronize()
lib.rnnt_debug_timeline(ctypes.c_void_p(0))
t = buf.cpu().numpy()[: (4 << 20) // 8].reshape(-1, 8).astype(np.float64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
t = (t - t0) / 1000.0
print("CTAs", len(t), "span us", t[:, 3].max())
for name, a, bb in [("start", 0, 0), ("prologue", 0, 1), ("mainloop", 1, 2), ("epilogue", 2, 3)]:
    dd = t[:, bb] - t[:, a] if a != bb else t[:, a]
    print(f"{name:10s} med {np.median(dd):7.2f} p90 {np.percentile(dd, 90):7.2f} max {dd.max():7.2f}")
# epilogue-internal marks (thread 0, its group's first chunk): operands of the chunk in registers, cells computed and
# staged, skewed write issued; then the group's remaining chunks
lv = t[t[:, 7] > t[:, 2]]
for name, a, bb in [("chunk 0 loads", 2, 4), ("chunk 0 compute", 4, 5), ("chunk 0 skewed write", 5, 6), ("later chunks", 6, 7), ("tail", 7, 3)]:
    dd = lv[:, bb] - lv[:, a]
    print(f"{name:22s} med {np.median(dd):7.2f} p10 {np.percentile(dd, 10):7.2f} p90 {np.percentile(dd, 90):7.2f}")
