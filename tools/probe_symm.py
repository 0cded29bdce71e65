"""Probe: does this box give NVLS multicast through torch symmetric memory at world size 1, and does
the library's MULTIMEM exchange (multimem.red.add) deliver into it?  Prints one JSON line."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29555")
out = {}
try:
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    import torch.distributed._symmetric_memory as symm_mem
    out["backend"] = str(symm_mem.get_backend(torch.device("cuda", 0))) if hasattr(symm_mem, "get_backend") else None
    t = symm_mem.empty(1 << 20, dtype=torch.float32, device="cuda")
    h = symm_mem.rendezvous(t, dist.group.WORLD)
    out["multicast_ptr"] = int(h.multicast_ptr)
    if out["multicast_ptr"]:
        import paper_2206_13236_b200 as R
        t.zero_()
        ls = torch.arange(8, dtype=torch.float32, device="cuda")
        lp = torch.ones(8, device="cuda")
        R.rnnt_loss_sums(ls, lp, None, 8, 0.5, 1.0, R.EXCHANGE_MULTIMEM, out["multicast_ptr"])
        R.rnnt_loss_sums(ls, lp, None, 8, 0.5, 1.0, R.EXCHANGE_MULTIMEM, out["multicast_ptr"])
        h.barrier(channel=0)
        torch.cuda.synchronize()
        out["multimem_sums"] = t[:2].tolist()      # expect [28.0, 16.0]
except Exception as e:
    out["error"] = f"{type(e).__name__}: {e}"[:300]
print(json.dumps(out), flush=True)
