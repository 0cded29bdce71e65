"""Memory-safety checks of the CUDA path without compute-sanitizer (closed on the GPU pool: runs under it
left GPUs needing a reset):

* guard bands: every output tensor and the workspace are carved out of one device buffer with 64 KiB
  of a byte pattern before and after each region; after a full step (plain, smoothed, full loss) the
  patterns must be intact -- an out-of-bounds write anywhere in them shows up;
* uninitialised reads: a step whose workspace and outputs start as 0xFF garbage (NaN / -1 patterns)
  must give bit-identical outputs to a step whose buffers start zeroed -- a read of a workspace or
  output element before the library writes it shows up as a difference.
Shapes: config 1, ragged edge cases, and a 4-utterance shard of config 2.
"""
import numpy as np
import pytest

import synth
from gpu_common import to_dev

pytestmark = pytest.mark.gpu

GUARD = 64 << 10
PATTERN = 0xA5


class Carver:
    """Regions of one uint8 device buffer, each with GUARD pattern bytes before and after it."""

    def __init__(self, sizes):
        import torch
        self.offs = []
        off = GUARD
        for n in sizes:
            off = (off + 255) // 256 * 256
            self.offs.append((off, n))
            off += n + GUARD
        self.buf = torch.full((off + GUARD,), PATTERN, dtype=torch.uint8, device="cuda")

    def region(self, i, dtype, shape, fill=None):
        import torch
        off, n = self.offs[i]
        t = self.buf[off:off + n]
        if fill is not None:
            t.fill_(fill)
        return t.view(dtype).view(*shape)

    def guards_intact(self):
        import torch
        mask = torch.ones_like(self.buf, dtype=torch.bool)
        for off, n in self.offs:
            mask[off:off + n] = False
        return bool((self.buf[mask] == PATTERN).all())


def _out_specs(b):
    import torch
    N, T, U, V, J, S = b.N, b.T, b.U, b.V, b.J, b.S
    f32, i32, i16 = torch.float32, torch.int32, torch.int16
    return [("loss_simple", f32, (N,)), ("px_grad", f32, (N, T, U + 1)), ("py_grad", f32, (N, T, U + 1)),
            ("am_grad", f32, (N, T, V)), ("lm_grad", f32, (N, U + 1, V)), ("ranges", i32, (N, T)),
            ("h", i16, (N, T, S, J)), ("loss_pruned", f32, (N,)), ("d_enc", f32, (N, T, J)),
            ("d_dec", f32, (N, U + 1, J)), ("d_w", f32, (V, J)), ("d_b", f32, (V,)), ("status", i32, (N,))]


def _run(b, fill, smoothed=False):
    import torch
    import paper_2206_13236_b200 as R
    dev = to_dev(b)
    dims = R.make_dims(b.N, b.T, b.U, b.V, b.J, b.S)
    specs = _out_specs(b)
    esz = {torch.float32: 4, torch.int32: 4, torch.int16: 2}
    sizes = [int(np.prod(shape)) * esz[dt] for _, dt, shape in specs] + [R.rnnt_workspace_bytes(dims)]
    c = Carver(sizes)
    out = {name: c.region(i, dt, shape, fill) for i, (name, dt, shape) in enumerate(specs)}
    out["status"].zero_()                       # status is OR-ed into (include/rnnt.h)
    ws = c.region(len(specs), torch.uint8, (sizes[-1],), fill)
    kw = dict(lm_only_scale=0.25, am_only_scale=0.1) if smoothed else {}
    R.step(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], dev["enc_proj"], dev["dec_proj"], dev["w_out"],
           dev["b_out"], b.S, out=out, workspace=ws, **kw)
    torch.cuda.synchronize()
    return {k: v.clone() for k, v in out.items()}, c.guards_intact()


def _sub(b, idx):
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


CASES = {
    "c1": lambda: synth.make_batch(1),
    "ragged": lambda: synth.make_custom([40, 3, 17, 1], [13, 2, 16, 0], 33, 16, 4, seed=4, logit_scale=2.0),
    "infeasible+S7": lambda: synth.make_custom([30, 12], [20, 40], 65, 24, 7, seed=6),
    "c2[0:4]": lambda: _sub(synth.make_batch(2), [0, 1, 2, 3]),
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("smoothed", [False, True])
def test_guards_and_uninitialised_reads(case, smoothed):
    import torch
    b = CASES[case]()
    clean, ok_clean = _run(b, 0x00, smoothed)
    dirty, ok_dirty = _run(b, 0xFF, smoothed)
    assert ok_clean and ok_dirty, "a guard band was overwritten (out-of-bounds write)"
    for k in clean:
        assert torch.equal(clean[k], dirty[k]), f"{k}: depends on the initial buffer contents"


def test_full_loss_guards():
    import torch
    import paper_2206_13236_b200 as R
    b = synth.make_custom([40, 3, 17], [13, 2, 16], 33, 16, 3, seed=8, logit_scale=2.0)
    dev = to_dev(b)
    dims = R.make_dims(b.N, b.T, b.U, b.V, b.J, 1)
    f32 = torch.float32
    specs = [("loss", f32, (b.N,)), ("d_enc", f32, (b.N, b.T, b.J)), ("d_dec", f32, (b.N, b.U + 1, b.J)),
             ("d_w", f32, (b.V, b.J)), ("d_b", f32, (b.V,)), ("status", torch.int32, (b.N,))]
    res = []
    for fill in (0x00, 0xFF):
        sizes = [int(np.prod(s)) * 4 for _, _, s in specs] + [R.rnnt_full_workspace_bytes(dims)]
        c = Carver(sizes)
        o = {n: c.region(i, dt, s, fill) for i, (n, dt, s) in enumerate(specs)}
        o["status"].zero_()
        ws = c.region(len(specs), torch.uint8, (sizes[-1],), fill)
        R.rnnt_full_loss(dev["enc_proj"], dev["dec_proj"], dev["w_out"], dev["b_out"], dev["symbols"],
                         dev["boundary"], dims, 1.0, o["loss"], o["d_enc"], o["d_dec"], o["d_w"], o["d_b"],
                         o["status"], ws)
        torch.cuda.synchronize()
        assert c.guards_intact()
        res.append({k: v.clone() for k, v in o.items()})
    for k in res[0]:
        assert torch.equal(res[0][k], res[1][k]), k
