"""Diagnostics (diagnostics build: RNNT_LIB=paper_2206_13236_b200/librnnt_b200_diag.so): per-CTA phase
timestamps of the am-gradient GEMM (gemm3<AmProb>, the last gemm3 launch of rnnt_simple_loss_backward, so its
CTAs overwrite the lm-gradient's entries) on a config: start, prologue done, accumulator full, epilogue done."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2206_13236_b200 as R
b = synth.make_batch(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
dev = R.batch_to_device(b, "cuda")
d = R.make_dims(b.N, b.T, b.U, b.V, b.J, b.S)
o = R.alloc_outputs(d, "cuda")
ws = torch.empty(R.rnnt_workspace_bytes(d), dtype=torch.uint8, device="cuda")
buf = torch.zeros((8 << 20) // 8, dtype=torch.int64, device="cuda")
lib = R.load_library()
R.rnnt_simple_loss(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], d, 0.5, o["loss_simple"],
                   o["px_grad"], o["py_grad"], None, None, o["status"], ws)
for it in range(4):
    lib.rnnt_debug_timeline(ctypes.c_void_p(buf.data_ptr() if it == 3 else 0))
    R.rnnt_simple_loss_backward(dev["am"], dev["lm"], o["px_grad"], o["py_grad"], dev["symbols"], dev["boundary"], d,
                                0.5, o["am_grad"], o["lm_grad"], ws)
    torch.cuda.synchronize()
lib.rnnt_debug_timeline(ctypes.c_void_p(0))
t = buf.cpu().numpy()[: (4 << 20) // 8].reshape(-1, 8).astype(np.float64)
t = t[(t[:, 0] > 0) & (t[:, 3] > 0)]
t0 = t[:, 0].min()
t = (t - t0) / 1000.0
t = t[np.argsort(t[:, 0])]
print("CTAs traced", len(t), "span us", t[:, 3].max())
for name, a, bb in [("prologue", 0, 1), ("mainloop (wait)", 1, 2), ("epilogue", 2, 3), ("whole CTA", 0, 3)]:
    dd = t[:, bb] - t[:, a]
    print(f"{name:16s} med {np.median(dd):7.2f} p10 {np.percentile(dd, 10):7.2f} p90 {np.percentile(dd, 90):7.2f} max {dd.max():7.2f}")
for i in list(range(0, 6)) + list(range(len(t) // 2, len(t) // 2 + 6)):
    print("  cta#%d" % i, np.round(t[i], 2).tolist())
# epilogue-internal marks of the live tiles (thread 0): picks of chunk 0 done, chunk 0's input tile landed, chunk 0
# stored, both chunks done (before the wait for the stores' shared-memory reads)
lv = t[(t[:, 4] > -1e6) & (t[:, 7] > t[:, 2])]
for name, a, bb in [("picks c0", 2, 4), ("input tile wait", 4, 5), ("chunk 0 compute+store", 5, 6), ("chunk 2", 6, 7), ("store drain", 7, 3)]:
    dd = lv[:, bb] - lv[:, a]
    print(f"{name:22s} med {np.median(dd):7.2f} p10 {np.percentile(dd, 10):7.2f} p90 {np.percentile(dd, 90):7.2f}")
