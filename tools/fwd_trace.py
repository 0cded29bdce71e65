"""Diagnostics: per-(CTA, row tile) timestamps of the persistent joiner forward pair kernel (config from argv,
default c5).  Needs the diagnostics build (make -C paper_2206_13236_b200 diag;
RNNT_LIB=paper_2206_13236_b200/librnnt_b200_diag.so)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2206_13236_b200 as R
b = synth.make_batch(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
dev = R.batch_to_device(b, "cuda")
buf = torch.zeros((8 << 20) // 8, dtype=torch.int64, device="cuda")
lib = R.load_library()
for it in range(4):
    lib.rnnt_debug_timeline(ctypes.c_void_p(buf.data_ptr() if it == 3 else 0))
    R.step(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], dev["enc_proj"], dev["dec_proj"],
           dev["w_out"], dev["b_out"], b.S, overlap=False)
    torch.cuda.synchronize()
lib.rnnt_debug_timeline(ctypes.c_void_p(0))
off = (7 << 20) // 8
t = buf.cpu().numpy()[off:off + 148 * 8 * 10].reshape(148, 8, 10).astype(np.float64)
valid = t[:, :, 0] > 0
t0 = t[valid][:, 0].min()
t = np.where(t > 0, (t - t0) / 1000.0, np.nan)
print("tiles traced", valid.sum(), "span us", np.nanmax(t))
names = ["took", "mma0 start", "mma0 issued", "mma last issued", "epi0 full", "epi0 done", "epiL full", "epiL done", "merged"]
for c in [0, 1, 2, 3, 70, 71, 146, 147]:
    print("cta", c)
    for i in range(8):
        if valid[c, i]:
            print("   ", " ".join(f"{x:7.1f}" for x in t[c, i, :9]))
print("columns:", ", ".join(names))
