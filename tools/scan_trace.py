"""Diagnostics: phase timestamps of the pruned scan kernel (one CTA per utterance and direction):
# needs the diagnostics build: make -C paper_2206_13236_b200 diag; RNNT_LIB=paper_2206_13236_b200/librnnt_b200_diag.so
staging, A (chunk matrices), B (boundary chain), C (frames).

    python tools/scan_trace.py <config>"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2206_13236_b200 as R
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
b = synth.make_batch(cfg)
dev = R.batch_to_device(b, "cuda")
buf = torch.zeros((8 << 20) // 8, dtype=torch.int64, device="cuda")
lib = R.load_library()
for it in range(4):
    lib.rnnt_debug_timeline(ctypes.c_void_p(buf.data_ptr() if it == 3 else 0))
    R.step(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], dev["enc_proj"], dev["dec_proj"],
           dev["w_out"], dev["b_out"], b.S, overlap=False)
    torch.cuda.synchronize()
lib.rnnt_debug_timeline(ctypes.c_void_p(0))
off = (6 << 20) // 8
raw = buf.cpu().numpy()[off:off + b.N * 2 * 8].reshape(b.N, 2, 8)
sc = raw[:, :, :5].astype(np.float64)
cyc, ncs = raw[:, :, 5].astype(np.float64), raw[:, :, 6].astype(np.float64)
sc = (sc - sc[:, :, :1]) / 1000.0
d = np.diff(sc, axis=2).reshape(-1, 4)
print(f"cfg {cfg}: T={b.T} S={b.S}; per-CTA phase durations (us) median / max")
for i, nm in enumerate(["stage", "A chunk matrices", "B boundary chain", "C frames"]):
    print(f"  {nm:18s} {np.median(d[:, i]):8.2f} {d[:, i].max():8.2f}")
print("  end max", sc[:, :, 4].max())
print("  phase B loop: cycles median %.0f, chunks %.0f, cycles/step %.0f" % (np.median(cyc), np.median(ncs), np.median(cyc / np.maximum(ncs, 1))))
