"""Run W warm-up steps and then one step of the whole hot path on a BASELINE config (for ncu
captures: skip W x kernels-per-step launches)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth, paper_2206_13236_b200 as R
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
W = int(sys.argv[2]) if len(sys.argv) > 2 else 2
b = synth.make_batch(cfg)
dev = R.batch_to_device(b, "cuda")
for i in range(W + 1):
    o = R.step(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], dev["enc_proj"], dev["dec_proj"],
               dev["w_out"], dev["b_out"], b.S)
    torch.cuda.synchronize()
print("ok", R.rnnt_launch_count())
