"""Shared helpers for the GPU parity tests (tolerances from BASELINE north_star / DESIGN.md D6)."""
import numpy as np
import torch

import oracle as O
import paper_2206_13236_b200 as R

LOSS_RTOL = 1e-5          # losses: relative, fp32 (north_star)
OCC_ATOL = 1e-4           # fp32 gradients / occupancies: absolute, elementwise (north_star)
BF16_ATOL, BF16_RTOL = 1e-4, 5e-3   # bf16-GEMM gradients: max|d| <= 1e-4 + 5e-3 max|ref| (D6)


def to_dev(b):
    return R.batch_to_device(b, "cuda")


def dims_of_batch(b):
    return R.make_dims(b.N, b.T, b.U, b.V, b.J, b.S)


def run_simple(b, gs=0.5, dev=None):
    dev = dev or to_dev(b)
    d = dims_of_batch(b)
    o = R.alloc_outputs(d, "cuda")
    ws = torch.empty(R.rnnt_workspace_bytes(d), dtype=torch.uint8, device="cuda")
    R.rnnt_simple_loss(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], d, gs, o["loss_simple"],
                       o["px_grad"], o["py_grad"], o["am_grad"], o["lm_grad"], o["status"], ws)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in o.items() if k in
            ("loss_simple", "px_grad", "py_grad", "am_grad", "lm_grad", "status")}


def run_ranges(b, px_grad, py_grad):
    d = dims_of_batch(b)
    st = torch.zeros(b.N, dtype=torch.int32, device="cuda")
    rg = torch.empty(b.N, b.T, dtype=torch.int32, device="cuda")
    R.rnnt_get_ranges(torch.from_numpy(np.ascontiguousarray(px_grad, np.float32)).cuda(),
                      torch.from_numpy(np.ascontiguousarray(py_grad, np.float32)).cuda(),
                      torch.from_numpy(b.boundary).cuda(), d, rg, st)
    torch.cuda.synchronize()
    return rg.cpu().numpy(), st.cpu().numpy()


def run_prune(b, ranges, dev=None):
    dev = dev or to_dev(b)
    d = dims_of_batch(b)
    h = torch.empty(b.N, b.T, b.S, b.J, dtype=torch.int16, device="cuda")
    R.rnnt_prune(dev["enc_proj"], dev["dec_proj"], torch.from_numpy(np.ascontiguousarray(ranges, np.int32)).cuda(),
                 dev["boundary"], d, h)
    torch.cuda.synchronize()
    return h.cpu().numpy().view(np.uint16)


def run_pruned(b, h_bits, ranges, gs=1.0, dev=None):
    dev = dev or to_dev(b)
    d = dims_of_batch(b)
    o = R.alloc_outputs(d, "cuda")
    ws = torch.empty(R.rnnt_workspace_bytes(d), dtype=torch.uint8, device="cuda")
    h = torch.from_numpy(np.ascontiguousarray(h_bits).view(np.int16)).cuda()
    R.rnnt_pruned_loss(h, dev["w_out"], dev["b_out"], dev["symbols"],
                       torch.from_numpy(np.ascontiguousarray(ranges, np.int32)).cuda(), dev["boundary"], d, gs,
                       o["loss_pruned"], o["d_enc"], o["d_dec"], o["d_w"], o["d_b"], o["status"], ws)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in o.items() if k in
            ("loss_pruned", "d_enc", "d_dec", "d_w", "d_b", "status")}


def oracle_h_bits(b, ranges):
    """The oracle's joiner input on the band, taken from O.pruned_lattice (matched mode, D6:
    bf16_rn(tanh(enc + dec)) in fp64), laid out as the C-ABI's h (N, T, S, J) bf16 bits."""
    import synth
    h = np.zeros((b.N, b.T, b.S, b.J), np.float64)
    for n in range(b.N):
        d = b.utterance(n)
        T = d["T"]
        if T == 0:
            continue
        rg = np.asarray(ranges[n, :T], np.int64)
        lat = O.pruned_lattice(d["enc"], d["dec"], d["W"], d["b"], d["y"], rg, b.S, matched=True)
        tt, uu = lat["tt"], lat["uu"]
        h[n, tt, uu - rg[tt]] = lat["h"]
    return synth.f32_to_bf16_bits(h.astype(np.float32))


H_FLIP_MAX = 1e-4     # fraction of h elements allowed one bf16 ulp off
FLIP_LOG = []         # (case, flips, elements) of every check: printed by the tests


def h_flip_rate(h, ref, case=""):
    diff = h.astype(np.int32) - ref.astype(np.int32)
    assert np.abs(diff).max() <= 1, f"{case}: h differs by more than one bf16 ulp"
    flips = int(np.count_nonzero(diff))
    FLIP_LOG.append((case, flips, diff.size))
    print(f"h flips {case}: {flips} of {diff.size} = {flips / max(1, diff.size):.2e}")
    return flips / max(1, diff.size)


def assert_bf16_grad(got, ref, name):
    err = np.max(np.abs(got - ref)) if got.size else 0.0
    lim = BF16_ATOL + BF16_RTOL * (np.max(np.abs(ref)) if ref.size else 0.0)
    assert err <= lim, f"{name}: max|d|={err:.3e} > {lim:.3e}"


def worst_abs_above_one(got, ref):
    """Worst absolute error over the entries with |ref| > 1 (am_grad[t,0], lm_grad[u,0], lm_grad[u,y]):
    the entries where assert_close_abs's tolerance is relative (D6 deviation note)."""
    m = np.abs(ref) > 1
    return float(np.max(np.abs(got[m] - ref[m]))) if m.any() else 0.0


def assert_close_abs(got, ref, atol, name):
    """|got - ref| <= atol * max(1, |ref|) elementwise: 1e-4 absolute for O(1) values (occupancies
    in [0,1], most gradient entries), relative for the few entries far above 1 (e.g. lm_grad[u,0]
    ~ -170 sums hundreds of blank occupancies, where an fp32 ulp alone is 1.5e-5).  DESIGN.md D6."""
    if not got.size:
        return
    lim = atol * np.maximum(1.0, np.abs(ref))
    bad = np.abs(got - ref) > lim
    assert not bad.any(), (f"{name}: {bad.sum()} elements off, worst |d|="
                           f"{np.max(np.abs(got - ref)):.3e} (ref there {ref.flat[np.argmax(np.abs(got - ref))]:.4g})")


def assert_loss(got, ref, name):
    ref = np.asarray(ref, np.float64)
    got = np.asarray(got, np.float64)
    fin = np.isfinite(ref)
    assert np.array_equal(fin, np.isfinite(got)), f"{name}: finiteness differs"
    rel = np.abs(got[fin] - ref[fin]) / np.maximum(np.abs(ref[fin]), 1e-30)
    assert rel.size == 0 or rel.max() <= LOSS_RTOL, f"{name}: max rel {rel.max():.3e}"
