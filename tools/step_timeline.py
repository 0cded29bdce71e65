"""Diagnostics: start/end of every C-ABI call of one step (events on the call's stream), c2."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth, paper_2206_13236_b200 as R
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
b = synth.make_batch(cfg)
dev = R.batch_to_device(b, "cuda")
d = R.make_dims(b.N, b.T, b.U, b.V, b.J, b.S)
o = R.alloc_outputs(d, "cuda")
ws = torch.empty(R.rnnt_workspace_bytes(d), dtype=torch.uint8, device="cuda")
cur = R.critical_stream()
torch.cuda.set_stream(cur)
side, side2 = R._side_stream("cuda", 0), R._side_stream("cuda", 1)
marks = []


def ev(name, s):
    e = torch.cuda.Event(enable_timing=True)
    e.record(s)
    marks.append((name, e))


def run():
    marks.clear()
    ev("start", cur)
    R.rnnt_simple_loss(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], d, 0.5, o["loss_simple"], o["px_grad"],
                       o["py_grad"], None, None, o["status"], ws, cur)
    ev("simple_fwd", cur)
    side.wait_stream(cur)
    R.rnnt_simple_loss_backward(dev["am"], dev["lm"], o["px_grad"], o["py_grad"], dev["symbols"], dev["boundary"], d,
                                0.5, o["am_grad"], o["lm_grad"], ws, side)
    ev("simple_bwd(side)", side)
    R.rnnt_get_ranges(o["px_grad"], o["py_grad"], dev["boundary"], d, o["ranges"], o["status"], cur)
    ev("ranges", cur)
    R.rnnt_prune(dev["enc_proj"], dev["dec_proj"], o["ranges"], dev["boundary"], d, o["h"], cur)
    ev("prune", cur)
    R.rnnt_pruned_loss_forward(o["h"], dev["w_out"], dev["b_out"], dev["symbols"], o["ranges"], dev["boundary"], d, 1.0,
                               o["loss_pruned"], o["status"], ws, cur)
    ev("pruned_fwd", cur)
    side2.wait_stream(cur)
    R.rnnt_pruned_loss_backward_weight(o["h"], d, o["d_w"], o["d_b"], ws, side2)
    ev("dW(side2)", side2)
    R.rnnt_pruned_loss_backward_input(o["h"], dev["w_out"], o["ranges"], dev["boundary"], d, o["d_enc"], o["d_dec"],
                                      ws, cur)
    ev("dh", cur)
    cur.wait_stream(side)
    cur.wait_stream(side2)
    ev("end", cur)


for _ in range(5):
    run()
torch.cuda.synchronize()
acc = {}
for rep in range(10):
    run()
    torch.cuda.synchronize()
    t0 = marks[0][1]
    for name, e in marks[1:]:
        acc.setdefault(name, []).append(t0.elapsed_time(e) * 1000)
for name, v in acc.items():
    v.sort()
    print(f"{name:18s} ends at {v[len(v) // 2]:7.1f} us")
