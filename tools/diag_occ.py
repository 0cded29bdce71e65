"""Diagnostic: max occupancy / loss error of the simple stage vs the oracle on a config."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle as O
import synth
from gpu_common import run_simple
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nutt = int(sys.argv[2]) if len(sys.argv) > 2 else 32
b = synth.make_batch(cfg)
g = run_simple(b)
worst = {}
for n in range(min(nutt, b.N)):
    d = b.utterance(n)
    s = O.simple_loss(d["am"], d["lm"], d["y"], 0.5)
    T, U = d["T"], d["U"]
    e = dict(loss=abs(g["loss_simple"][n] - s["loss"]) / abs(s["loss"]),
             px=np.abs(g["px_grad"][n, :T, :U + 1] - s["px_grad"]).max(),
             py=np.abs(g["py_grad"][n, :T, :U + 1] - s["py_grad"]).max(),
             am=np.abs(g["am_grad"][n, :T] - s["am_grad"]).max(),
             lm=(np.abs(g["lm_grad"][n, :U + 1] - s["lm_grad"]) / np.maximum(1, np.abs(s["lm_grad"]))).max())
    for k, v in e.items():
        worst[k] = max(worst.get(k, 0), v)
    print(n, T, U, " ".join(f"{k}={v:.2e}" for k, v in e.items()), flush=True)
print("WORST", " ".join(f"{k}={v:.2e}" for k, v in worst.items()))
