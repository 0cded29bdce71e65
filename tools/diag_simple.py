"""Diagnostic: error structure of the simple stage on config 2 (GPU vs oracle)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import synth, oracle as O
from gpu_common import run_simple
b = synth.make_batch(2)
g = run_simple(b)
for n in range(4):
    d = b.utterance(n)
    s = O.simple_loss(d["am"], d["lm"], d["y"], 0.5)
    T, U = d["T"], d["U"]
    Lg = g["loss_simple"][n]
    print(f"utt {n} T={T} U={U} loss gpu={Lg:.6f} ora={s['loss']:.6f} abs={Lg-s['loss']:.3e}")
    dy = g["px_grad"][n, :T, :U+1] - s["px_grad"]
    db = g["py_grad"][n, :T, :U+1] - s["py_grad"]
    print("  px_grad maxabs %.2e mean %.2e | py_grad maxabs %.2e mean %.2e" % (abs(dy).max(), dy.mean(), abs(db).max(), db.mean()))
    print("  rel err py_grad (cells>1e-3): median %.2e" % np.median(np.abs(db[s['py_grad']>1e-3]/s['py_grad'][s['py_grad']>1e-3])))
    print("  colsum py err max %.2e  rowsum py err max %.2e" % (abs(db.sum(0)).max(), abs(db.sum(1)).max()))
    dl = g["lm_grad"][n, :U+1] - s["lm_grad"]
    i = np.unravel_index(np.argmax(abs(dl)), dl.shape)
    print("  lm_grad maxabs %.2e at %s ref %.4f; col0 maxabs %.2e; others maxabs %.2e" % (abs(dl).max(), i, s['lm_grad'][i], abs(dl[:,0]).max(), abs(dl[:,1:]).max()))
    da = g["am_grad"][n, :T] - s["am_grad"]
    print("  am_grad maxabs %.2e" % abs(da).max())
