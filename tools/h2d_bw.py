"""Host->device copy bandwidth from pinned memory (56 MB like bench.py's e2e inputs): one stream vs
several streams (copy engines) in parallel, pinned with pin_memory() vs cudaHostAlloc'd (torch's
pinned allocator)."""
import torch
sizes = [22_000_000, 5_300_000, 23_000_000, 5_500_000]


def run(nstreams, hs, ds, reps=20):
    sts = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    e0.record(cur)
    for st in sts:
        st.wait_stream(cur)
    for _ in range(reps):
        for i, (h, d) in enumerate(zip(hs, ds)):
            # split every tensor into nstreams parts
            n = h.numel()
            for k, st in enumerate(sts):
                a, b = n * k // nstreams, n * (k + 1) // nstreams
                with torch.cuda.stream(st):
                    d[a:b].copy_(h[a:b], non_blocking=True)
    for st in sts:
        cur.wait_stream(st)
    e1.record(cur)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return sum(sizes) / ms / 1e6


hs = [torch.empty(s // 4, dtype=torch.float32).pin_memory() for s in sizes]
ds = [torch.empty(s // 4, dtype=torch.float32, device="cuda") for s in sizes]
for ns in (1, 2, 4):
    run(ns, hs, ds, 3)
    print(f"pin_memory, {ns} stream(s): {run(ns, hs, ds):.1f} GB/s")
hs2 = [torch.empty(s // 4, dtype=torch.float32, pin_memory=True) for s in sizes]
for ns in (1, 2, 4):
    run(ns, hs2, ds, 3)
    print(f"pin_memory=True alloc, {ns} stream(s): {run(ns, hs2, ds):.1f} GB/s")
