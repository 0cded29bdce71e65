"""Pins of the pruned stage of the oracle."""
import math

import numpy as np
import pytest
import torch

import oracle as O
import synth


def _dense_joiner_logits(d, matched):
    h = np.tanh(d["enc"].astype(np.float64)[:, None, :] + d["dec"].astype(np.float64)[None, :, :])
    if matched:
        h = O.bf16_round(h)
    return h @ d["W"].astype(np.float64).T + d["b"].astype(np.float64)


def _torchaudio(logits, y):
    import torchaudio.functional as F
    lg = torch.tensor(logits[None], dtype=torch.float32, requires_grad=True)
    loss = F.rnnt_loss(lg, torch.tensor(np.asarray(y)[None], dtype=torch.int32),
                       torch.tensor([logits.shape[0]], dtype=torch.int32),
                       torch.tensor([logits.shape[1] - 1], dtype=torch.int32),
                       blank=0, reduction="sum")
    loss.backward()
    return float(loss.detach()), lg.grad[0].double().numpy()


@pytest.mark.parametrize("matched", [True, False])
def test_full_band_equals_dense_rnnt_torchaudio(matched):
    """S >= U+1 makes the pruned loss the full RNN-T loss with the same joiner
    (BASELINE north_star identity); torchaudio computes it independently from the
    materialised (T, U+1, V) logits, and its logit gradient is dz."""
    b = synth.make_batch(1)
    d = b.utterance(1)      # config 1's 2nd utterance has S = U+1
    assert d["S"] >= d["U"] + 1
    p = np.zeros(d["T"], np.int64)
    pr = O.pruned_loss(d["enc"], d["dec"], d["W"], d["b"], d["y"], p, d["S"], matched=matched)
    logits = _dense_joiner_logits(d, matched)
    ref, g = _torchaudio(logits, d["y"])
    assert abs(pr["loss"] - ref) < 1e-5 * abs(ref)
    lat = pr["lattice"]
    assert np.allclose(pr["dz"], g[lat["tt"], lat["uu"]], atol=2e-6)


def test_pruned_equals_band_brute_force_and_bounds_loss():
    rng = np.random.default_rng(4)
    for trial in range(6):
        T, U, S, V, J = 5, 4, 2, 5, 3
        enc = rng.standard_normal((T, J)); dec = rng.standard_normal((U + 1, J))
        W = rng.standard_normal((V, J)); bb = rng.standard_normal(V)
        y = rng.integers(1, V, size=U)
        raw = rng.integers(0, O.umax(U, S) + 1, size=T)
        p = O.adjust_bounds(raw, T, U, S)
        pr = O.pruned_loss(enc, dec, W, bb, y, p, S, matched=False)
        # brute force over band-respecting paths of the dense lattice
        logits = np.tanh(enc[:, None, :] + dec[None]) @ W.T + bb
        lp = logits - O.logsumexp(logits, axis=2)[..., None]
        px = np.full((T, U + 1), -np.inf); px[:, :U] = lp[:, np.arange(U), y]
        py = lp[..., 0]
        mask = O.band_mask(p, U, S)
        assert abs(-pr["loss"] - O.brute_force_logprob(px, py, mask)) < 1e-10
        # pruning removes mass: L_pruned <= L_full
        assert -pr["loss"] <= O.total_logprob(px, py) + 1e-12


def test_nested_bands_monotone():
    rng = np.random.default_rng(8)
    T, U, V, J = 12, 6, 7, 4
    d = dict(enc=rng.standard_normal((T, J)), dec=rng.standard_normal((U + 1, J)),
             W=rng.standard_normal((V, J)), b=rng.standard_normal(V), y=rng.integers(1, V, U))
    prev = -np.inf
    for S in range(2, U + 2):
        # bands [p_t, p_t+S) nested as S grows when p is the same "diagonal" clipped sequence
        p = O.adjust_bounds(np.zeros(T, np.int64), T, U, S)
        Lp = -O.pruned_loss(d["enc"], d["dec"], d["W"], d["b"], d["y"], p, S, matched=False)["loss"]
        if S > 2:
            # band(S) contains band(S-1) when p(S) <= p(S-1) pointwise and p(S)+S >= p(S-1)+S-1
            if np.all(p <= prev_p) and np.all(p + S >= prev_p + S - 1):
                assert Lp >= prev - 1e-12
        prev, prev_p = Lp, p


def test_joiner_grads_finite_differences_and_row_sums():
    rng = np.random.default_rng(9)
    T, U, S, V, J = 4, 3, 2, 6, 3
    enc = rng.standard_normal((T, J)); dec = rng.standard_normal((U + 1, J))
    W = rng.standard_normal((V, J)); bb = rng.standard_normal(V)
    y = rng.integers(1, V, size=U)
    p = O.adjust_bounds(np.array([0, 1, 1, 2]), T, U, S)
    gs = 1.0
    pr = O.pruned_loss(enc, dec, W, bb, y, p, S, grad_scale=gs, matched=False)
    assert np.allclose(pr["dz"].sum(axis=1), 0, atol=1e-12)   # softmax gradient rows sum to 0
    assert np.allclose(pr["d_b"], pr["dz"].sum(axis=0))
    h = 1e-6

    def f(**kw):
        a = dict(enc=enc, dec=dec, W=W, b=bb)
        a.update(kw)
        return O.pruned_loss(a["enc"], a["dec"], a["W"], a["b"], y, p, S, matched=False,
                             with_grads=False)["loss"]
    for name, arr, grad in (("enc", enc, pr["d_enc"]), ("dec", dec, pr["d_dec"]),
                            ("W", W, pr["d_w"]), ("b", bb, pr["d_b"])):
        it = np.nditer(arr, flags=["multi_index"])
        for _ in it:
            i = it.multi_index
            a = arr.copy(); a[i] += h
            c = arr.copy(); c[i] -= h
            fd = (f(**{name: a}) - f(**{name: c})) / (2 * h)
            assert abs(fd - grad[i]) < 1e-6, (name, i)


def test_uniform_joiner_band_count_closed_form():
    """W = 0, b = 0: every in-band arc is -ln V, so L_p = ln(#band paths) - (T+U) ln V,
    the path count taken by brute-force enumeration (independent of the recursion)."""
    T, U, S, V, J = 7, 5, 3, 9, 2
    rng = np.random.default_rng(1)
    enc = rng.standard_normal((T, J)); dec = rng.standard_normal((U + 1, J))
    y = rng.integers(1, V, size=U)
    p = O.adjust_bounds(np.array([0, 2, 2, 2, 3, 3, 3]), T, U, S)
    pr = O.pruned_loss(enc, dec, np.zeros((V, J)), np.zeros(V), y, p, S, matched=False)
    mask = O.band_mask(p, U, S)
    count = sum(1 for a in O.brute_force_paths(T, U) if all(mask[t, u] for (t, u, _) in a))
    assert abs(-pr["loss"] - (math.log(count) - (T + U) * math.log(V))) < 1e-10


def test_full_step_config1_composition():
    """loss = 0.5*(-L_simple) + 1.0*(-L_pruned) summed over the batch;
    pruned_scale = 0 reproduces 0.5 * simple."""
    b = synth.make_batch(1)
    r = O.full_step(b)
    assert abs(r["loss"] - (0.5 * r["loss_simple"].sum() + r["loss_pruned"].sum())) < 1e-9
    r0 = O.full_step(b, pruned_scale=0.0)
    assert abs(r0["loss"] - 0.5 * r0["loss_simple"].sum()) < 1e-9
    assert np.all(r0["d_w"] == 0)
    # ranges satisfy the invariants and pad with Umax
    for n in range(b.N):
        T, U = int(b.T_n[n]), int(b.U_n[n])
        p = r["ranges"][n]
        assert p[0] == 0 and p[T - 1] == O.umax(U, b.S) and np.all(p[T:] == O.umax(U, b.S))
