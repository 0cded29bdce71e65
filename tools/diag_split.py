"""Diagnostics: simple stage with/without the NormProb column split (RNNT_NORM_SPLIT), where do they differ."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import synth
from gpu_common import run_simple
b = synth.make_batch(2, zero_logits=True)
g = run_simple(b)
print("loss nan", np.isnan(g["loss_simple"]).sum(), g["loss_simple"][:4])
px = g["px_grad"]
bad = np.argwhere(~np.isfinite(px))
print("nonfinite px_grad cells", len(bad), bad[:10])
for n in range(3):
    T, U = int(b.T_n[n]), int(b.U_n[n])
    print(n, T, U, "px row0", px[n, 0, :8], "sum", np.nansum(px[n, :T, :U+1]))
bad_n = [n for n in range(b.N) if not np.isfinite(g["loss_simple"][n])]
print("bad", [(n, int(b.T_n[n]), int(b.U_n[n])) for n in bad_n])
print("good", [(n, int(b.T_n[n]), int(b.U_n[n])) for n in range(b.N) if n not in bad_n][:20])
