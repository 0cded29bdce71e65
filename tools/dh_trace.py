"""Diagnostics: per-(CTA, item) timestamps of the persistent joiner_dh kernel (config from argv, default c5)."""
# needs the diagnostics build: make -C paper_2206_13236_b200 diag; RNNT_LIB=paper_2206_13236_b200/librnnt_b200_diag.so
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
           dev["w_out"], dev["b_out"], b.S)
    torch.cuda.synchronize()
lib.rnnt_debug_timeline(ctypes.c_void_p(0))
t = buf.cpu().numpy()[(4 << 20) // 8:(4 << 20) // 8 + 148 * 16 * 5].reshape(148, 16, 5).astype(np.float64)
valid = t[:, :, 0] > 0
t0 = t[valid][:, 0].min()
t = (t - t0) / 1000.0
print("items traced", valid.sum(), "kernel span us", t[valid][:, 4].max())
for name, a, bb in [("prod->first MMA", 0, 1), ("MMA issue span", 1, 2), ("MMA end->epi start", 2, 3), ("epilogue", 3, 4)]:
    d = (t[:, :, bb] - t[:, :, a])[valid]
    print(f"{name:22s} med {np.median(d):7.2f}  p90 {np.percentile(d, 90):7.2f}  max {d.max():7.2f}")
for c in [0, 1, 70, 147]:
    print("cta", c, np.round(t[c][valid[c]], 1).tolist())
off = (4 << 20) // 8 + 148 * 16 * 5
k = buf.cpu().numpy()[off:off + 148 * 3 * 8 * 4].reshape(148, 3, 8, 4).astype(np.float64)
k = (k - t0) / 1000.0
for c in [0, 70]:
    for it in range(2):
        print("cta", c, "item", it)
        for kb in range(8):
            print("   kb", kb, "issue %.2f loaded %.2f transformed %.2f mma %.2f" % tuple(k[c, it, kb]))
d = k[:, :, :, 1] - k[:, :, :, 0]
print("TMA latency (issue->seen) med %.2f p90 %.2f" % (np.median(d), np.percentile(d, 90)))
d = k[:, :, :, 2] - k[:, :, :, 1]
print("transform med %.2f p90 %.2f" % (np.median(d), np.percentile(d, 90)))
d = k[:, :, :, 3] - k[:, :, :, 2]
print("transform->mma med %.2f p90 %.2f" % (np.median(d), np.percentile(d, 90)))
off3 = (6 << 20) // 8
sc = buf.cpu().numpy()[off3:off3 + 32 * 2 * 5].reshape(32, 2, 5).astype(np.float64)
sc = (sc - sc[:, :, :1]) / 1000.0
print("scan phases (us from CTA start): staged / A / B / C  medians:", np.round(np.median(sc.reshape(-1, 5), axis=0), 2).tolist(),
      "max end", sc[:, :, 4].max())
