"""GPU parity: every C-ABI stage against the fp64 oracle on the same seeded inputs.

Each stage gets its inputs from the generator or the oracle (never from the CUDA
path) so a mismatch is attributable to one stage.  Tolerances: gpu_common.py."""
import numpy as np
import pytest

import oracle as O
import synth
from gpu_common import (H_FLIP_MAX, OCC_ATOL, assert_bf16_grad, assert_close_abs, assert_loss, h_flip_rate,
                        oracle_h_bits, worst_abs_above_one, run_prune, run_pruned, run_ranges, run_simple, to_dev)

pytestmark = pytest.mark.gpu


def _oracle_simple(b, gs=0.5):
    r = dict(loss=np.zeros(b.N), px_grad=np.zeros((b.N, b.T, b.U + 1)), py_grad=np.zeros((b.N, b.T, b.U + 1)),
             am_grad=np.zeros((b.N, b.T, b.V)), lm_grad=np.zeros((b.N, b.U + 1, b.V)))
    for n in range(b.N):
        d = b.utterance(n)
        s = O.simple_loss(d["am"], d["lm"], d["y"], gs)
        T, U = d["T"], d["U"]
        r["loss"][n] = s["loss"]
        r["px_grad"][n, :T, :U + 1] = s["px_grad"]
        r["py_grad"][n, :T, :U + 1] = s["py_grad"]
        r["am_grad"][n, :T] = s["am_grad"]
        r["lm_grad"][n, :U + 1] = s["lm_grad"]
    return r


def _oracle_ranges(b, pxg, pyg):
    rg = np.zeros((b.N, b.T), np.int64)
    for n in range(b.N):
        T, U = int(b.T_n[n]), int(b.U_n[n])
        if not O.feasible(T, U, b.S):
            continue
        rg[n, :T] = O.adjust_bounds(O.raw_bounds(pxg[n, :T, :U + 1], pyg[n, :T, :U + 1], b.S), T, U, b.S)
        rg[n, T:] = O.umax(U, b.S)
    return rg


def _oracle_pruned(b, ranges, gs=1.0):
    r = dict(loss=np.zeros(b.N), d_enc=np.zeros((b.N, b.T, b.J)), d_dec=np.zeros((b.N, b.U + 1, b.J)),
             d_w=np.zeros((b.V, b.J)), d_b=np.zeros(b.V))
    for n in range(b.N):
        d = b.utterance(n)
        T, U = d["T"], d["U"]
        if not O.feasible(T, U, b.S):
            r["loss"][n] = np.inf
            continue
        p = O.pruned_loss(d["enc"], d["dec"], d["W"], d["b"], d["y"], ranges[n, :T], b.S, gs, matched=True)
        r["loss"][n] = p["loss"]
        r["d_enc"][n, :T] = p["d_enc"]
        r["d_dec"][n, :U + 1] = p["d_dec"]
        r["d_w"] += p["d_w"]
        r["d_b"] += p["d_b"]
    return r


def check_simple(b):
    g = run_simple(b)
    o = _oracle_simple(b)
    assert_loss(g["loss_simple"], o["loss"], "loss_simple")
    assert_close_abs(g["px_grad"], o["px_grad"], OCC_ATOL, "px_grad")
    assert_close_abs(g["py_grad"], o["py_grad"], OCC_ATOL, "py_grad")
    assert_close_abs(g["am_grad"], o["am_grad"], OCC_ATOL, "am_grad")
    assert_close_abs(g["lm_grad"], o["lm_grad"], OCC_ATOL, "lm_grad")
    print(f"worst |d| on |ref|>1 entries (N={b.N} V={b.V}): am_grad "
          f"{worst_abs_above_one(g['am_grad'], o['am_grad']):.2e}, lm_grad {worst_abs_above_one(g['lm_grad'], o['lm_grad']):.2e}")
    return g, o


def check_ranges(b, o):
    pxg = o["px_grad"].astype(np.float32)
    pyg = o["py_grad"].astype(np.float32)
    rg, st = run_ranges(b, pxg, pyg)
    ref = _oracle_ranges(b, pxg, pyg)
    assert np.array_equal(rg, ref), f"ranges differ at {np.argwhere(rg != ref)[:5]}"
    return ref


def check_prune(b, ranges, case=""):
    h = run_prune(b, ranges)
    ref = oracle_h_bits(b, ranges)
    # rows outside the band / past T_n are exact zeros on both sides and count in the denominator only
    # through the band rows: the rate is over the band rows actually computed
    live = np.zeros(h.shape[:3], bool)
    for n in range(b.N):
        T, U = int(b.T_n[n]), int(b.U_n[n])
        live[n, :T] = (ranges[n, :T, None] + np.arange(b.S)[None, :]) <= U
    rate = h_flip_rate(h[live], ref[live], case or f"N={b.N} V={b.V} J={b.J}")
    assert rate <= H_FLIP_MAX, f"h flip rate {rate:.2e} > {H_FLIP_MAX}"
    assert np.array_equal(h[~live], ref[~live])
    return ref


def check_pruned(b, ranges, h_ref):
    g = run_pruned(b, h_ref, ranges)
    o = _oracle_pruned(b, ranges)
    assert_loss(g["loss_pruned"], o["loss"], "loss_pruned")
    for k in ("d_w", "d_b", "d_enc", "d_dec"):
        assert_bf16_grad(g[k], o[k], k)


@pytest.mark.parametrize("cfg", [1, 2])
def test_stagewise_parity(cfg):
    b = synth.make_batch(cfg)
    g, o = check_simple(b)
    ranges = check_ranges(b, o)
    h_ref = check_prune(b, ranges)
    check_pruned(b, ranges, h_ref)


@pytest.mark.parametrize("case", [
    dict(T=[1, 5, 9], U=[0, 0, 3], V=7, J=8, S=2),        # T=1, U=0 single-path utterances
    dict(T=[40, 3, 17], U=[13, 2, 16], V=33, J=16, S=4),  # ragged, one S >= U+1, one U = T-1
    dict(T=[70, 66], U=[40, 2], V=300, J=24, S=1),        # S = 1 (U=40 infeasible, U=2 infeasible)
    dict(T=[7, 30], U=[20, 9], V=11, J=8, S=3),           # U=20 > T(S-1)=14 infeasible
    dict(T=[300, 129], U=[257, 60], V=40, J=16, S=6),     # U+1 > 256: multi-warp recursion
    dict(T=[90, 41], U=[70, 12], V=65, J=16, S=7),        # runtime-S scan (SMAX 8), cluster of 2
    dict(T=[60, 33], U=[150, 20], V=65, J=16, S=20),      # runtime-S scan (SMAX 32), cluster of 4
    dict(T=[1200, 700], U=[1000, 600], V=24, J=16, S=3),  # U + 1 > 512: the combine's two column windows
    dict(T=[2000, 900], U=[300, 100], V=16, J=8, S=16),   # T S 8 B > smem: the pruned scan reads its arcs from L2
    dict(T=[50, 23], U=[20, 9], V=40, J=1160, S=5),       # J > 1024: partial 256-column part, d_dec in two passes
])
def test_edge_cases(case):
    b = synth.make_custom(case["T"], case["U"], case["V"], case["J"], case["S"], seed=11, logit_scale=2.0)
    g, o = check_simple(b)
    ranges = check_ranges(b, o)
    h_ref = check_prune(b, ranges)
    check_pruned(b, ranges, h_ref)


@pytest.mark.parametrize("gs", [1e-6, 3e4])
def test_pruned_grad_scale(gs):
    """joiner_dh stores dpre as fp16 dpre / gs (D21): the input gradients scale linearly with the
    loss scale, with no fp16 underflow at a tiny gs or overflow at a large one."""
    b = synth.make_batch(1)
    o = _oracle_simple(b)
    ranges = _oracle_ranges(b, o["px_grad"].astype(np.float32), o["py_grad"].astype(np.float32))
    h_ref = oracle_h_bits(b, ranges)
    g = run_pruned(b, h_ref, ranges, gs=gs)
    r = _oracle_pruned(b, ranges)
    for k in ("d_w", "d_b", "d_enc", "d_dec"):
        assert_bf16_grad(g[k] / gs, r[k], k)


def test_pruned_stage_very_long_utterance():
    """T = 8000 frames (the pruned scan's arcs are read from L2, its chunk chain is long), the pruned
    stage alone on the oracle's bounds and joiner input: loss and every gradient."""
    b = synth.make_custom([8000, 3000], [1000, 400], 16, 8, 10, seed=41, logit_scale=2.0)
    o = _oracle_simple(b)
    ranges = _oracle_ranges(b, o["px_grad"].astype(np.float32), o["py_grad"].astype(np.float32))
    h_ref = oracle_h_bits(b, ranges)
    check_pruned(b, ranges, h_ref)


def test_poison_padding():
    """NaN in every padded input element: outputs finite, padded outputs exactly 0."""
    b = synth.make_custom([12, 30, 5], [4, 9, 1], 19, 16, 3, seed=3, poison=True)
    g = run_simple(b)
    for n in range(b.N):
        T, U = int(b.T_n[n]), int(b.U_n[n])
        for k in ("px_grad", "py_grad"):
            assert np.all(np.isfinite(g[k][n]))
            assert np.all(g[k][n, T:] == 0) and np.all(g[k][n, :, U + 1:] == 0)
        assert np.all(g["am_grad"][n, T:] == 0) and np.all(np.isfinite(g["am_grad"][n]))
        assert np.all(g["lm_grad"][n, U + 1:] == 0) and np.all(np.isfinite(g["lm_grad"][n]))
    o = _oracle_simple(b)
    ranges = _oracle_ranges(b, o["px_grad"].astype(np.float32), o["py_grad"].astype(np.float32))
    h = run_prune(b, ranges)
    h_ref = oracle_h_bits(b, ranges)
    assert np.abs(h.astype(np.int32) - h_ref.astype(np.int32)).max() <= 1
    p = run_pruned(b, h_ref, ranges)
    for k in ("d_w", "d_b", "d_enc", "d_dec", "loss_pruned"):
        assert np.all(np.isfinite(p[k]))
    for n in range(b.N):
        T, U = int(b.T_n[n]), int(b.U_n[n])
        assert np.all(p["d_enc"][n, T:] == 0) and np.all(p["d_dec"][n, U + 1:] == 0)


def test_end_to_end_step_config2():
    """The whole path on the GPU (its own ranges) against the whole oracle path.

    Ranges (D5): on the GPU's own fp32 occupancies the GPU ranges equal the oracle's Eq. 8 +
    ADJ-scan bit for bit; against the fp64 occupancies the raw Eq. 8 argmax may differ only at
    near-tie frames (top-2 gap below 2(S+1)*1e-4) -- a flip there may move the adjusted bounds of
    neighbouring frames through Eq. 9-10.  The pruned loss is compared for utterances whose ranges
    agree with the oracle's."""
    import torch
    import paper_2206_13236_b200 as R
    b = synth.make_batch(2)
    dev = to_dev(b)
    o = R.step(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], dev["enc_proj"], dev["dec_proj"],
               dev["w_out"], dev["b_out"], b.S)
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in o.items()}
    ref = O.full_step(b)
    assert_loss(g["loss_simple"], ref["loss_simple"], "loss_simple")
    same = []
    for n in range(b.N):
        T, U = int(b.T_n[n]), int(b.U_n[n])
        gx, gy = g["px_grad"][n, :T, :U + 1], g["py_grad"][n, :T, :U + 1]
        own = O.adjust_bounds(O.raw_bounds(gx, gy, b.S), T, U, b.S)
        assert np.array_equal(g["ranges"][n, :T], own), f"utt {n}: ranges differ on identical inputs"
        raw_g = O.raw_bounds(gx, gy, b.S)
        raw_o = O.raw_bounds(ref["px_grad"][n, :T, :U + 1], ref["py_grad"][n, :T, :U + 1], b.S)
        for t in np.nonzero(raw_g != raw_o)[0]:
            v = O.bound_scores(ref["px_grad"][n, t, :U + 1], ref["py_grad"][n, t, :U + 1], b.S)
            top = np.sort(v)[-2:]
            assert top[1] - top[0] < 2 * (b.S + 1) * 1e-4, f"utt {n} frame {t}: raw bound flipped, not a near-tie"
        if np.array_equal(g["ranges"][n, :T], ref["ranges"][n, :T]):
            same.append(n)
    assert len(same) > 0
    assert_loss(g["loss_pruned"][same], ref["loss_pruned"][same], "loss_pruned")


def test_simple_backward_split_matches():
    """rnnt_simple_loss(grads=NULL) + rnnt_simple_loss_backward on a side stream gives bit-identical
    am/lm gradients to rnnt_simple_loss with both gradient pointers (include/rnnt.h)."""
    import torch
    import paper_2206_13236_b200 as R
    b = synth.make_batch(2)
    dev = to_dev(b)
    d = R.make_dims(b.N, b.T, b.U, b.V, b.J, b.S)
    ws = torch.empty(R.rnnt_workspace_bytes(d), dtype=torch.uint8, device="cuda")
    o1 = R.alloc_outputs(d, "cuda")
    R.rnnt_simple_loss(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], d, 0.5, o1["loss_simple"], o1["px_grad"],
                       o1["py_grad"], o1["am_grad"], o1["lm_grad"], o1["status"], ws)
    o2 = R.alloc_outputs(d, "cuda")
    R.rnnt_simple_loss(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], d, 0.5, o2["loss_simple"], o2["px_grad"],
                       o2["py_grad"], None, None, o2["status"], ws)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    R.rnnt_simple_loss_backward(dev["am"], dev["lm"], o2["px_grad"], o2["py_grad"], dev["symbols"], dev["boundary"], d,
                                0.5, o2["am_grad"], o2["lm_grad"], ws, side)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    for k in ("loss_simple", "px_grad", "py_grad", "am_grad", "lm_grad"):
        assert torch.equal(o1[k], o2[k]), k


def _oracle_smoothed(b, a_lm, a_ac, gs=0.5):
    r = dict(loss=np.zeros(b.N), px_grad=np.zeros((b.N, b.T, b.U + 1)), py_grad=np.zeros((b.N, b.T, b.U + 1)),
             am_grad=np.zeros((b.N, b.T, b.V)), lm_grad=np.zeros((b.N, b.U + 1, b.V)))
    for n in range(b.N):
        d = b.utterance(n)
        s = O.smoothed_loss(d["am"], d["lm"], d["y"], a_lm, a_ac, gs)
        T, U = d["T"], d["U"]
        r["loss"][n] = s["loss"]
        r["px_grad"][n, :T, :U + 1] = s["px_grad"]
        r["py_grad"][n, :T, :U + 1] = s["py_grad"]
        r["am_grad"][n, :T] = s["am_grad"]
        r["lm_grad"][n, :U + 1] = s["lm_grad"]
    return r


@pytest.mark.parametrize("case", [
    dict(cfg=1, a_lm=0.25, a_ac=0.0),
    dict(cfg=1, a_lm=0.0, a_ac=0.25),
    dict(cfg=2, a_lm=0.25, a_ac=0.1),
    dict(T=[40, 1, 17], U=[13, 0, 16], V=33, J=16, S=4, a_lm=0.2, a_ac=0.3),   # V % 4 != 0: generic epilogues
])
def test_smoothed_simple_stage(case):
    """Smoothed trivial joiner (Eq. 11-15, D18) on the GPU against the fp64 oracle: loss, occupancies
    and the am/lm gradients through all three terms (the split forward / side-stream backward form)."""
    import torch
    import paper_2206_13236_b200 as R
    if "cfg" in case:
        b = synth.make_batch(case["cfg"])
    else:
        b = synth.make_custom(case["T"], case["U"], case["V"], case["J"], case["S"], seed=5, logit_scale=2.0)
    a_lm, a_ac = case["a_lm"], case["a_ac"]
    dev = to_dev(b)
    d = R.make_dims(b.N, b.T, b.U, b.V, b.J, b.S)
    ws = torch.empty(R.rnnt_workspace_bytes(d), dtype=torch.uint8, device="cuda")
    o = R.alloc_outputs(d, "cuda")
    R.rnnt_simple_loss_smoothed(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], d, a_lm, a_ac, 0.5,
                                o["loss_simple"], o["px_grad"], o["py_grad"], None, None, o["status"], ws)
    R.rnnt_simple_loss_smoothed_backward(dev["am"], dev["lm"], o["px_grad"], o["py_grad"], dev["symbols"],
                                         dev["boundary"], d, a_lm, a_ac, 0.5, o["am_grad"], o["lm_grad"], ws)
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in o.items()}
    ref = _oracle_smoothed(b, a_lm, a_ac)
    assert_loss(g["loss_simple"], ref["loss"], "loss_simple")
    for k in ("px_grad", "py_grad", "am_grad", "lm_grad"):
        assert_close_abs(g[k], ref[k], OCC_ATOL, k)


def test_smoothed_zero_scales_bit_identical():
    """lm_only_scale = am_only_scale = 0 runs exactly the plain trivial-joiner path."""
    import torch
    import paper_2206_13236_b200 as R
    b = synth.make_batch(2)
    dev = to_dev(b)
    d = R.make_dims(b.N, b.T, b.U, b.V, b.J, b.S)
    ws = torch.empty(R.rnnt_workspace_bytes(d), dtype=torch.uint8, device="cuda")
    o1, o2 = R.alloc_outputs(d, "cuda"), R.alloc_outputs(d, "cuda")
    R.rnnt_simple_loss(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], d, 0.5, o1["loss_simple"], o1["px_grad"],
                       o1["py_grad"], o1["am_grad"], o1["lm_grad"], o1["status"], ws)
    R.rnnt_simple_loss_smoothed(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], d, 0.0, 0.0, 0.5,
                                o2["loss_simple"], o2["px_grad"], o2["py_grad"], o2["am_grad"], o2["lm_grad"],
                                o2["status"], ws)
    torch.cuda.synchronize()
    for k in ("loss_simple", "px_grad", "py_grad", "am_grad", "lm_grad"):
        assert torch.equal(o1[k], o2[k]), k
