"""H2D bandwidth of 56 MB from page-locked host memory: untouched vs CPU-filled torch pinned buffers,
and cudaHostAlloc(write-combined) buffers filled by the CPU."""
import ctypes
import numpy as np, torch
sizes = [22_000_000, 5_300_000, 23_000_000, 5_500_000]
ds = [torch.empty(s // 4, dtype=torch.float32, device="cuda") for s in sizes]
def bw(hs, reps=20):
    for h, d in zip(hs, ds): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        for h, d in zip(hs, ds): d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    return sum(sizes) / (e0.elapsed_time(e1) / reps) / 1e6
a = [torch.empty(s // 4, dtype=torch.float32, pin_memory=True) for s in sizes]
print("pinned untouched %.1f GB/s" % bw(a))
for t in a: t.copy_(torch.randn(t.numel()))
print("pinned CPU-filled %.1f GB/s" % bw(a))
b = [torch.empty(s // 4, dtype=torch.float32, pin_memory=True) for s in sizes]
for t in b: t.fill_(1.0)
print("pinned fill_ %.1f GB/s" % bw(b))
cudart = ctypes.CDLL("libcudart.so")
def wc(n):
    p = ctypes.c_void_p()
    assert cudart.cudaHostAlloc(ctypes.byref(p), ctypes.c_size_t(n * 4), ctypes.c_uint(4)) == 0   # WriteCombined
    arr = np.ctypeslib.as_array((ctypes.c_float * n).from_address(p.value))
    return torch.from_numpy(arr)
try:
    c = [wc(s // 4) for s in sizes]
    for t in c: t.copy_(torch.randn(t.numel()))
    print("write-combined CPU-filled %.1f GB/s (is_pinned %s)" % (bw(c), c[0].is_pinned()))
except Exception as e:
    print("wc failed", e)
