"""One eager step of the whole hot path (plus the smoothed simple stage and the full loss) on config 1
and on a 4-utterance shard of config 2, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck).  Usage: compute-sanitizer --tool memcheck python tools/sanitize_step.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2206_13236_b200 as R
import synth


def sub_batch(b, idx):
    import copy
    s = copy.copy(b)
    idx = np.asarray(idx)
    s.N = len(idx)
    s.T_n, s.U_n = b.T_n[idx], b.U_n[idx]
    s.T, s.U = int(s.T_n.max()), int(s.U_n.max())
    s.symbols = np.ascontiguousarray(b.symbols[idx, :s.U])
    s.boundary = np.ascontiguousarray(b.boundary[idx])
    s.am = np.ascontiguousarray(b.am[idx, :s.T])
    s.lm = np.ascontiguousarray(b.lm[idx, :s.U + 1])
    s.enc_proj = np.ascontiguousarray(b.enc_proj[idx, :s.T])
    s.dec_proj = np.ascontiguousarray(b.dec_proj[idx, :s.U + 1])
    return s


for name, b in [("c1", synth.make_batch(1)), ("c2[0:4]", sub_batch(synth.make_batch(2), [0, 1, 2, 3]))]:
    dev = R.batch_to_device(b, "cuda")
    args = (dev["am"], dev["lm"], dev["symbols"], dev["boundary"], dev["enc_proj"], dev["dec_proj"], dev["w_out"],
            dev["b_out"], b.S)
    o = R.step(*args)
    o2 = R.step(*args, lm_only_scale=0.25, am_only_scale=0.1)
    f = R.full_loss(dev["enc_proj"], dev["dec_proj"], dev["w_out"], dev["b_out"], dev["symbols"], dev["boundary"])
    torch.cuda.synchronize()
    print(name, "loss_simple", o["loss_simple"].cpu().numpy()[:2], "loss_pruned", o["loss_pruned"].cpu().numpy()[:2],
          "smoothed", o2["loss_simple"].cpu().numpy()[:2], "full", f["loss"].cpu().numpy()[:2], flush=True)
print("launches", R.rnnt_launch_count())
