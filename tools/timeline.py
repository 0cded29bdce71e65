"""Diagnostics: the GPU timeline of one bench step (CUDA-graph replay, as bench.py times it), from
CUPTI kernel records (torch.profiler): per kernel its stream, start and end relative to the step's
first kernel, so the critical path and the side-stream overlap can be read off.

    python tools/timeline.py [config=5] [replays=3]"""
import collections, json, os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth, paper_2206_13236_b200 as R
from paper_2206_13236_b200.dist import GradBuffer

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
b = synth.make_batch(cfg)
dev = R.batch_to_device(b, "cuda")
dims = R.make_dims(b.N, b.T, b.U, b.V, b.J, b.S)
outs = R.alloc_outputs(dims, "cuda")
gbuf = GradBuffer(b.V, b.J, "cuda", mode="local")
outs["d_w"], outs["d_b"] = gbuf.d_w, gbuf.d_b
ws = torch.empty(R.rnnt_workspace_bytes(dims), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
stream = R.critical_stream()
torch.cuda.set_stream(stream)


def step():
    outs["status"].zero_()
    R.step(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], dev["enc_proj"], dev["dec_proj"],
           dev["w_out"], dev["b_out"], b.S, out=outs, workspace=ws, exchange=gbuf)


for _ in range(3):
    step()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=stream):
    step()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        flush.zero_()
        g.replay()
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "trace.json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("ph") == "X" and e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
# split into replays at the flush kernels (torch's fill)
steps, cur = [], None
for e in ev:
    if "rnnt::" not in e["name"]:
        if cur:
            steps.append(cur)
        cur = []
        continue
    if cur is not None:
        cur.append(e)
if cur:
    steps.append(cur)
last = steps[-1]
t0 = last[0]["ts"]
print(f"config c{cfg}: {len(last)} kernels; step span {last[-1]['ts'] + last[-1]['dur'] - t0:.1f} us "
      f"(first kernel start -> last kernel end)")
streams = {}
for e in last:
    s = e["args"].get("stream", e.get("tid"))
    streams.setdefault(s, len(streams))
    nm = e["name"].replace("void ", "").split("(")[0].replace("rnnt::", "")
    print(f"  s{streams[s]}  {e['ts'] - t0:8.1f} -> {e['ts'] + e['dur'] - t0:8.1f}  {e['dur']:7.1f}  {nm[:60]}")
tot = collections.Counter()
for e in last:
    tot[e["name"].split("(")[0]] += e["dur"]
