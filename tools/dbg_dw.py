import sys, ctypes; sys.path.insert(0, ".")
import torch, synth, paper_2206_13236_b200 as R
from tests.gpu_common import *
b = synth.make_batch(1)
dev = R.batch_to_device(b, "cuda")
o = R.step(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], dev["enc_proj"], dev["dec_proj"], dev["w_out"], dev["b_out"], b.S, overlap=False)
try:
    torch.cuda.synchronize()
except Exception as e:
    print("sync error", e)
cudart = ctypes.CDLL("libcudart.so.12") if False else None
