"""Diagnostics: the normaliser GEMM's N (= round16(U+1)) against the uniform closed form."""
import os, sys, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import synth
from gpu_common import run_simple
for U1 in [17, 33, 48, 64, 72, 80, 88, 96, 104, 112, 120, 128, 144, 160, 176, 192, 208, 224, 240, 256]:
    U = U1 - 1
    b = synth.make_custom([U + 30, U + 5], [U, U // 2], 50, 8, 3, seed=1)
    b.am[:] = 0; b.lm[:] = 0
    g = run_simple(b)
    ok = []
    for n in range(b.N):
        T, Un = int(b.T_n[n]), int(b.U_n[n])
        ref = -(math.lgamma(T + Un) - math.lgamma(Un + 1) - math.lgamma(T) - (T + Un) * math.log(50))
        ok.append(abs(g["loss_simple"][n] - ref) <= 1e-4 * abs(ref))
    print("U+1", U1, "BN", min(256, (U1 + 15) // 16 * 16), "ok", ok, g["loss_simple"])
