"""GPU parity at BASELINE.json's full sizes (configs 2-4), in the launch configuration bench.py
times (the whole batch through ``paper_2206_13236_b200.step`` with stream overlap).

Two kinds of checks, because the oracle cannot run whole c3/c4 batches in seconds:

1. Closed forms that hold at any size (SURVEY.md 8(c) "full-size GPU pins"):
   * am = lm = 0 (uniform trivial joiner, every arc -ln V):
       L_s = ln C(T-1+U, U) - (T+U) ln V  and the occupancies are path-count ratios
       y'(t,u) = C(t+u,u) C(T-2-t+U-u, U-u-1) / C(T-1+U,U),
       0'(t,u) = C(t+u,u) C(T-2-t+U-u, U-u)   / C(T-1+U,U)   (t < T-1),  0'(T-1,U) = 1;
     am/lm gradients follow from them with P(t,u,v) = 1/V (chain rule through Eq. 5-6).
   * W_out = 0, b_out = 0 (uniform pruned joiner): every in-band arc is -ln V, so
       L_p = ln N_band - (T+U) ln V,  N_band = exact integer count of band-respecting paths
     over the GPU's own ranges; dh = W^T dz = 0 so d_enc = d_dec = 0 exactly; and
       d_b[v] = gs (sum_n (T_n+U_n)/V - [v=0] sum_n T_n - sum_n #{u : y_{n,u} = v})
     because every path has T blanks, emits each label once and has T+U arcs.
2. Sampled utterances of the real seeded batch, each checked against the fp64 oracle
   (D5/D6 tolerances): simple loss, occupancies, am/lm gradients; pruned loss and
   d_enc/d_dec at the GPU's ranges; ranges bit-exact on the GPU's own occupancies for every
   utterance.  d_w is a sum over the batch, so it is checked on a sub-batch of the sampled
   utterances run through the same kernels at the full V/J/S.
"""
import math

import numpy as np
import pytest

import oracle as O
import synth
from gpu_common import OCC_ATOL, assert_bf16_grad, assert_close_abs, assert_loss, to_dev

pytestmark = pytest.mark.gpu


def _run_step(b):
    import torch
    import paper_2206_13236_b200 as R
    dev = to_dev(b)
    o = R.step(dev["am"], dev["lm"], dev["symbols"], dev["boundary"], dev["enc_proj"], dev["dec_proj"],
               dev["w_out"], dev["b_out"], b.S)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in o.items() if k != "h"}


def _lC(n, k):
    """ln C(n, k) elementwise (fp64), -inf where the binomial is 0."""
    n = np.asarray(n, np.float64)
    k = np.asarray(k, np.float64)
    ok = (k >= 0) & (n >= k)
    from scipy.special import gammaln
    with np.errstate(invalid="ignore"):
        v = gammaln(np.where(ok, n, 0) + 1) - gammaln(np.where(ok, k, 0) + 1) - gammaln(np.where(ok, n - k, 0) + 1)
    return np.where(ok, v, -np.inf)


def _uniform_occupancies(T, U):
    t = np.arange(T)[:, None].astype(np.float64)
    u = np.arange(U + 1)[None, :].astype(np.float64)
    tot = _lC(T - 1 + U, U)
    ypr = np.exp(_lC(t + u, u) + _lC(T - 2 - t + U - u, U - u - 1) - tot)
    ypr[:, U] = 0.0
    bpr = np.exp(_lC(t + u, u) + _lC(T - 2 - t + U - u, U - u) - tot)
    bpr[T - 1, :] = 0.0
    bpr[T - 1, U] = 1.0
    return ypr, bpr


def _band_paths(ranges, T, U, S):
    """Exact integer count of monotone paths (0,0)->(T-1,U) + terminal blank whose every node
    lies in the band p_t <= u < p_t + S (python big integers)."""
    prev = {}
    for t in range(T):
        cur = {}
        for u in range(int(ranges[t]), min(int(ranges[t]) + S, U + 1)):
            c = 1 if (t == 0 and u == 0) else 0
            c += prev.get(u, 0)           # blank arc from (t-1, u), kept iff (t-1, u) is in the band
            c += cur.get(u - 1, 0)        # label arc from (t, u-1), kept iff (t, u-1) is in the band
            cur[u] = c
        prev = cur
    return prev.get(U, 0)


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_uniform_closed_forms_full_size(cfg):
    b = synth.make_batch(cfg, zero_logits=True)
    g = _run_step(b)
    V, S, gs_s, gs_p = b.V, b.S, 0.5, 1.0
    exp_db = np.zeros(V)
    for n in range(b.N):
        T, U = int(b.T_n[n]), int(b.U_n[n])
        Ls = float(_lC(T - 1 + U, U)) - (T + U) * math.log(V)
        assert_loss(g["loss_simple"][n:n + 1], [-Ls], f"loss_simple[{n}]")
        ypr, bpr = _uniform_occupancies(T, U)
        assert_close_abs(g["px_grad"][n, :T, :U + 1], ypr, OCC_ATOL, f"px_grad[{n}]")
        assert_close_abs(g["py_grad"][n, :T, :U + 1], bpr, OCC_ATOL, f"py_grad[{n}]")
        occ = ypr + bpr
        y = b.symbols[n, :U]
        am_g = np.repeat(occ.sum(axis=1)[:, None] / V, V, axis=1)
        for u in range(U):
            am_g[:, y[u]] -= ypr[:, u]
        am_g[:, 0] -= bpr.sum(axis=1)
        lm_g = np.repeat(occ.sum(axis=0)[:, None] / V, V, axis=1)
        lm_g[np.arange(U), y] -= ypr[:, :U].sum(axis=0)
        lm_g[:, 0] -= bpr.sum(axis=0)
        assert_close_abs(g["am_grad"][n, :T], gs_s * am_g, OCC_ATOL, f"am_grad[{n}]")
        assert_close_abs(g["lm_grad"][n, :U + 1], gs_s * lm_g, OCC_ATOL, f"lm_grad[{n}]")
        # pruned stage on the GPU's own ranges
        rg = g["ranges"][n, :T].astype(np.int64)
        own = O.adjust_bounds(O.raw_bounds(g["px_grad"][n, :T, :U + 1], g["py_grad"][n, :T, :U + 1], S), T, U, S)
        assert np.array_equal(rg, own), f"utt {n}: ranges differ from Eq. 8 + ADJ-scan on identical inputs"
        nb = _band_paths(rg, T, U, S)
        assert nb > 0
        Lp = math.log(nb) - (T + U) * math.log(V)
        assert_loss(g["loss_pruned"][n:n + 1], [-Lp], f"loss_pruned[{n}]")
        exp_db += gs_p * (T + U) / V
        exp_db[0] -= gs_p * T
        np.subtract.at(exp_db, y, gs_p)
    assert np.all(g["d_enc"] == 0) and np.all(g["d_dec"] == 0), "W=0 must give d_enc = d_dec = 0 exactly"
    assert_bf16_grad(g["d_b"], exp_db, "d_b")
    assert np.all(g["status"] == 0)


def _samples(b, k):
    """k utterances spanning the length mix: the longest, the shortest, then evenly spaced."""
    order = np.argsort(b.T_n * (b.U_n + 1), kind="stable")
    pick = [int(order[-1]), int(order[0])] + [int(order[i]) for i in np.linspace(1, b.N - 2, max(0, k - 2)).astype(int)]
    return list(dict.fromkeys(pick))[:k]


def _sub_batch(b, idx):
    """The utterances ``idx`` of ``b`` as their own batch (same V, J, S, weights)."""
    import copy
    s = copy.copy(b)
    idx = np.asarray(idx)
    s.N = len(idx)
    s.T_n, s.U_n = b.T_n[idx], b.U_n[idx]
    s.T, s.U = int(s.T_n.max()), int(s.U_n.max())
    s.symbols = np.ascontiguousarray(b.symbols[idx, :max(s.U, 1)][:, :s.U])
    s.boundary = np.ascontiguousarray(b.boundary[idx])
    s.am = np.ascontiguousarray(b.am[idx, :s.T])
    s.lm = np.ascontiguousarray(b.lm[idx, :s.U + 1])
    s.enc_proj = np.ascontiguousarray(b.enc_proj[idx, :s.T])
    s.dec_proj = np.ascontiguousarray(b.dec_proj[idx, :s.U + 1])
    return s


@pytest.mark.parametrize("cfg,k", [(3, 3), (4, 1)])
def test_sampled_utterances_full_size(cfg, k):
    b = synth.make_batch(cfg)
    g = _run_step(b)
    S = b.S
    # ranges: bit-exact on the GPU's own fp32 occupancies, every utterance (D5)
    for n in range(b.N):
        T, U = int(b.T_n[n]), int(b.U_n[n])
        own = O.adjust_bounds(O.raw_bounds(g["px_grad"][n, :T, :U + 1], g["py_grad"][n, :T, :U + 1], S), T, U, S)
        assert np.array_equal(g["ranges"][n, :T], own), f"utt {n}: ranges differ on identical inputs"
        assert np.all(g["ranges"][n, T:] == O.umax(U, S))
    picks = _samples(b, k)
    sb = _sub_batch(b, picks)     # d_w / d_b: the sampled utterances as their own batch
    gs = _run_step(sb)
    dw_ref = np.zeros((b.V, b.J))
    db_ref = np.zeros(b.V)
    for i, n in enumerate(picks):
        d = b.utterance(n)
        T, U = d["T"], d["U"]
        s = O.simple_loss(d["am"], d["lm"], d["y"], 0.5)
        assert_loss(g["loss_simple"][n:n + 1], [s["loss"]], f"loss_simple[{n}]")
        assert_close_abs(g["px_grad"][n, :T, :U + 1], s["px_grad"], OCC_ATOL, f"px_grad[{n}]")
        assert_close_abs(g["py_grad"][n, :T, :U + 1], s["py_grad"], OCC_ATOL, f"py_grad[{n}]")
        assert_close_abs(g["am_grad"][n, :T], s["am_grad"], OCC_ATOL, f"am_grad[{n}]")
        assert_close_abs(g["lm_grad"][n, :U + 1], s["lm_grad"], OCC_ATOL, f"lm_grad[{n}]")
        p = O.pruned_loss(d["enc"], d["dec"], d["W"], d["b"], d["y"], g["ranges"][n, :T].astype(np.int64), S, 1.0,
                          matched=True)
        assert_loss(g["loss_pruned"][n:n + 1], [p["loss"]], f"loss_pruned[{n}]")
        assert_bf16_grad(g["d_enc"][n, :T], p["d_enc"], f"d_enc[{n}]")
        assert_bf16_grad(g["d_dec"][n, :U + 1], p["d_dec"], f"d_dec[{n}]")
        rs = gs["ranges"][i, :T].astype(np.int64)
        if not np.array_equal(rs, g["ranges"][n, :T]):     # a near-tie resolved differently (D5)
            p = O.pruned_loss(d["enc"], d["dec"], d["W"], d["b"], d["y"], rs, S, 1.0, matched=True)
        assert_loss(gs["loss_pruned"][i:i + 1], [p["loss"]], f"sub-batch loss_pruned[{i}]")
        dw_ref += p["d_w"]
        db_ref += p["d_b"]
    assert_bf16_grad(gs["d_w"], dw_ref, "d_w")
    assert_bf16_grad(gs["d_b"], db_ref, "d_b")


@pytest.mark.parametrize("which", [0, -1])
def test_dynamic_batch_end_to_end(which):
    """A batch of the dynamic-batch workload (sorted lengths, <= 2,500 encoder frames):
    the whole path against the oracle, pruned stage at the GPU's own (bit-exact, D5) ranges."""
    b = synth.make_dynamic_corpus()[which]
    g = _run_step(b)
    S = b.S
    dw_ref = np.zeros((b.V, b.J))
    db_ref = np.zeros(b.V)
    for n in range(b.N):
        d = b.utterance(n)
        T, U = d["T"], d["U"]
        s = O.simple_loss(d["am"], d["lm"], d["y"], 0.5)
        assert_loss(g["loss_simple"][n:n + 1], [s["loss"]], f"loss_simple[{n}]")
        assert_close_abs(g["px_grad"][n, :T, :U + 1], s["px_grad"], OCC_ATOL, f"px_grad[{n}]")
        assert_close_abs(g["py_grad"][n, :T, :U + 1], s["py_grad"], OCC_ATOL, f"py_grad[{n}]")
        assert_close_abs(g["am_grad"][n, :T], s["am_grad"], OCC_ATOL, f"am_grad[{n}]")
        assert_close_abs(g["lm_grad"][n, :U + 1], s["lm_grad"], OCC_ATOL, f"lm_grad[{n}]")
        own = O.adjust_bounds(O.raw_bounds(g["px_grad"][n, :T, :U + 1], g["py_grad"][n, :T, :U + 1], S), T, U, S)
        assert np.array_equal(g["ranges"][n, :T], own), f"utt {n}: ranges differ on identical inputs"
        p = O.pruned_loss(d["enc"], d["dec"], d["W"], d["b"], d["y"], own, S, 1.0, matched=True)
        assert_loss(g["loss_pruned"][n:n + 1], [p["loss"]], f"loss_pruned[{n}]")
        assert_bf16_grad(g["d_enc"][n, :T], p["d_enc"], f"d_enc[{n}]")
        assert_bf16_grad(g["d_dec"][n, :U + 1], p["d_dec"], f"d_dec[{n}]")
        dw_ref += p["d_w"]
        db_ref += p["d_b"]
    assert_bf16_grad(g["d_w"], dw_ref, "d_w")
    assert_bf16_grad(g["d_b"], db_ref, "d_b")


def _oracle_full(b, idx=None):
    """Full (unpruned) loss: the oracle's pruned loss with every frame's band [0, U_n] (S = U_n+1,
    all bounds 0), which the oracle pins equal to the dense RNN-T loss (test_oracle_pruned)."""
    idx = range(b.N) if idx is None else idx
    r = dict(loss={}, d_enc={}, d_dec={}, d_w=np.zeros((b.V, b.J)), d_b=np.zeros(b.V))
    for n in idx:
        d = b.utterance(n)
        T, U = d["T"], d["U"]
        p = O.pruned_loss(d["enc"], d["dec"], d["W"], d["b"], d["y"], np.zeros(T, np.int64), U + 1, 1.0, matched=True)
        r["loss"][n] = p["loss"]
        r["d_enc"][n] = p["d_enc"]
        r["d_dec"][n] = p["d_dec"]
        r["d_w"] += p["d_w"]
        r["d_b"] += p["d_b"]
    return r


def _run_full(b):
    import torch
    import paper_2206_13236_b200 as R
    dev = to_dev(b)
    o = R.full_loss(dev["enc_proj"], dev["dec_proj"], dev["w_out"], dev["b_out"], dev["symbols"], dev["boundary"])
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in o.items()}


@pytest.mark.parametrize("case", [
    dict(cfg=1),
    dict(T=[40, 1, 17, 9], U=[13, 0, 16, 2], V=33, J=16),          # ragged, T=1/U=0, U=T-1
    dict(T=[30, 200], U=[150, 60], V=40, J=24),                     # U+1 > 128: 128-row tiles across frames
])
def test_full_loss_small(case):
    """the full (unpruned) loss on the GPU against the oracle, every output."""
    b = synth.make_batch(1) if "cfg" in case else synth.make_custom(case["T"], case["U"], case["V"], case["J"], 3,
                                                                    seed=7, logit_scale=2.0)
    g = _run_full(b)
    ref = _oracle_full(b)
    for n in range(b.N):
        T, U = int(b.T_n[n]), int(b.U_n[n])
        assert_loss(g["loss"][n:n + 1], [ref["loss"][n]], f"loss[{n}]")
        assert_bf16_grad(g["d_enc"][n, :T], ref["d_enc"][n], f"d_enc[{n}]")
        assert_bf16_grad(g["d_dec"][n, :U + 1], ref["d_dec"][n], f"d_dec[{n}]")
        assert np.all(g["d_enc"][n, T:] == 0) and np.all(g["d_dec"][n, U + 1:] == 0)
    assert_bf16_grad(g["d_w"], ref["d_w"], "d_w")
    assert_bf16_grad(g["d_b"], ref["d_b"], "d_b")


def test_full_loss_config2_sampled():
    """The full loss at c2 size (10.7 GiB workspace): sampled utterances against the oracle, and the
    pruned loss bounded by it (L_pruned <= L_full: the band keeps a subset of the paths)."""
    import torch
    import paper_2206_13236_b200 as R
    b = synth.make_batch(2)
    g = _run_full(b)
    picks = _samples(b, 2)
    ref = _oracle_full(b, picks)
    for n in picks:
        T, U = int(b.T_n[n]), int(b.U_n[n])
        assert_loss(g["loss"][n:n + 1], [ref["loss"][n]], f"loss[{n}]")
        assert_bf16_grad(g["d_enc"][n, :T], ref["d_enc"][n], f"d_enc[{n}]")
        assert_bf16_grad(g["d_dec"][n, :U + 1], ref["d_dec"][n], f"d_dec[{n}]")
    p = _run_step(b)
    assert np.all(p["loss_pruned"] >= g["loss"] - 1e-3 * np.abs(g["loss"]))


def test_grad_hook_sees_final_weight_grads():
    """step(grad_hook=...) runs the hook (the data-parallel all_reduce in bench.py) on the d_w stream
    while the input-gradient kernels still run: it must see the final d_w, d_b and both losses, and the
    returned outputs must equal a step without the hook (c2 batch, launch configuration of bench.py)."""
    import torch
    import paper_2206_13236_b200 as R
    b = synth.make_batch(2)
    dev = R.batch_to_device(b, "cuda")
    args = (dev["am"], dev["lm"], dev["symbols"], dev["boundary"], dev["enc_proj"], dev["dec_proj"],
            dev["w_out"], dev["b_out"], b.S)
    ref = {k: v.clone() for k, v in R.step(*args).items()}
    torch.cuda.synchronize()
    seen = {}
    holder = {}

    def hook():
        o = holder["o"]
        seen["d_w"] = o["d_w"].clone()
        seen["d_b"] = o["d_b"].clone()
        seen["ls"] = o["loss_simple"].clone()
        seen["lp"] = o["loss_pruned"].clone()

    holder["o"] = R.alloc_outputs(R.make_dims(b.N, b.T, b.U, b.V, b.J, b.S), "cuda")
    o = R.step(*args, out=holder["o"], grad_hook=hook)
    torch.cuda.synchronize()
    for k in ("d_w", "d_b", "loss_pruned", "loss_simple", "d_enc", "d_dec", "am_grad"):
        assert torch.equal(o[k], ref[k]), k
    assert torch.equal(seen["d_w"], ref["d_w"]) and torch.equal(seen["d_b"], ref["d_b"])
    assert torch.equal(seen["ls"], ref["loss_simple"]) and torch.equal(seen["lp"], ref["loss_pruned"])
