"""Experiment: step(groups=k) -- the batch cut into k sub-batches whose chains run concurrently on their
own streams -- against the single chain: CUDA-graph replay time per step (L2 flushed between
replays) and the largest output differences.  Usage: python tools/exp_groups.py [config] [k ...]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2206_13236_b200 as R
import synth

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ks = [int(x) for x in sys.argv[2:]] or [1, 2, 4]
b = synth.make_batch(cfg)
dev = R.batch_to_device(b, "cuda")
dims = R.make_dims(b.N, b.T, b.U, b.V, b.J, b.S)
stream = R.critical_stream()
torch.cuda.set_stream(stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {}
ref = None
for k in ks:
    outs = R.alloc_outputs(dims, "cuda")
    ws = torch.empty(R.rnnt_workspace_bytes(dims), dtype=torch.uint8, device="cuda")

    def run():
        outs["status"].zero_()
        R.step(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], dev["enc_proj"], dev["dec_proj"],
               dev["w_out"], dev["b_out"], b.S, out=outs, workspace=ws, groups=k)

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        run()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    o = {kk: v.clone() for kk, v in outs.items()}
    if ref is None:
        ref = o
    diff = {kk: float((o[kk].float() - ref[kk].float()).abs().max()) for kk in o if kk != "h"}
    diff["h_equal"] = bool(torch.equal(o["h"], ref["h"]))
    res[k] = {"ms": statistics.median(ts), "min_ms": min(ts), "frames_per_s": b.frames / (statistics.median(ts) / 1e3),
              "maxdiff_vs_k1": diff}
    print(json.dumps({"config": cfg, "groups": k, **res[k]}), flush=True)
