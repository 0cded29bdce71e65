"""Host->device copy bandwidth from pinned memory (56.7 MB in 4 copies, like bench.py's e2e inputs)."""
import torch, time
sizes = [22_000_000, 5_300_000, 23_000_000, 5_500_000]
hs = [torch.empty(s // 4, dtype=torch.float32).pin_memory() for s in sizes]
ds = [torch.empty(s // 4, dtype=torch.float32, device="cuda") for s in sizes]
st = torch.cuda.Stream()
for _ in range(3):
    with torch.cuda.stream(st):
        for h, d in zip(hs, ds):
            d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
with torch.cuda.stream(st):
    for _ in range(20):
        for h, d in zip(hs, ds):
            d.copy_(h, non_blocking=True)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"H2D {sum(sizes) / 1e6:.1f} MB in {ms:.3f} ms = {sum(sizes) / ms / 1e6:.1f} GB/s")
