"""Pins of the trivial (linear) joiner stage of the oracle (Eq. 5-6):
hand values, shift invariance, finite differences, and identity with
torchaudio's independent ``rnnt_loss`` on the materialised linear joiner."""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle as O
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_examples.json")))


@pytest.mark.parametrize("case", GOLD["normalizer"])
def test_normalizer_hand_values(case):
    out = O.trivial_normalizer(np.array(case["am"]), np.array(case["lm"]))
    assert np.allclose(out, case["Lnorm"], atol=1e-12)


def test_trivial_lattice_hand_values():
    c = GOLD["trivial_lattice"][0]
    px, py, _ = O.trivial_lattice(np.array(c["am"]), np.array(c["lm"]), np.array(c["y"]))
    assert abs(px[0, 0] - c["px00"]) < 1e-12
    assert abs(py[0, 0] - c["py00"]) < 1e-12
    assert px[0, 1] == -np.inf


def test_normalizer_shift_invariance_and_direct():
    rng = np.random.default_rng(1)
    am = rng.standard_normal((8, 16))
    lm = rng.standard_normal((8, 16))
    L0 = O.trivial_normalizer(am, lm)
    shift_t = rng.choice([-500.0, 500.0], size=(8, 1))
    shift_u = rng.choice([-500.0, 500.0], size=(8, 1))
    L1 = O.trivial_normalizer(am + shift_t, lm + shift_u)
    assert np.allclose(L1, L0 + shift_t + shift_u.T, atol=1e-9)
    # direct triple loop, scalar math
    for t in range(8):
        for u in range(8):
            s = sum(math.exp(am[t, v] + lm[u, v]) for v in range(16))
            assert abs(L0[t, u] - math.log(s)) < 1e-12
    # arcs are log-probs of one softmax: e^y + e^empty <= 1
    y = rng.integers(1, 16, size=7)
    px, py, _ = O.trivial_lattice(am, lm, y)
    assert np.all(np.exp(px[:, :7]) + np.exp(py[:, :7]) <= 1 + 1e-12)


def _torchaudio_rnnt(logits, y):
    import torchaudio.functional as F
    lg = torch.tensor(logits[None], dtype=torch.float32, requires_grad=True)
    T, U1 = logits.shape[0], logits.shape[1]
    loss = F.rnnt_loss(lg, torch.tensor(np.asarray(y)[None], dtype=torch.int32),
                       torch.tensor([T], dtype=torch.int32), torch.tensor([U1 - 1], dtype=torch.int32),
                       blank=0, reduction="sum", fused_log_softmax=True)
    loss.backward()
    return float(loss.detach()), lg.grad[0].double().numpy()


@pytest.mark.parametrize("cfg", [1])
def test_simple_loss_matches_torchaudio(cfg):
    """Identity (BASELINE north_star): the simple loss equals a fully materialised
    linear-joiner RNN-T loss, logits(t,u,v) = am[t,v] + lm[u,v], computed by
    torchaudio (independent library, fp32).  Its logit gradient summed over u / t
    gives am_grad / lm_grad."""
    b = synth.make_batch(cfg)
    for n in range(b.N):
        d = b.utterance(n)
        s = O.simple_loss(d["am"], d["lm"], d["y"], grad_scale=1.0)
        logits = d["am"][:, None, :].astype(np.float64) + d["lm"][None, :, :]
        ref, g = _torchaudio_rnnt(logits, d["y"])
        assert abs(s["loss"] - ref) < 2e-5 * abs(ref)
        assert np.allclose(s["am_grad"], g.sum(axis=1), atol=2e-5)
        assert np.allclose(s["lm_grad"], g.sum(axis=0), atol=2e-5)


def test_simple_loss_matches_torchaudio_larger():
    b = synth.make_custom([40, 33], [12, 9], V=30, J=8, S=4, seed=5, logit_scale=2.0)
    for n in range(b.N):
        d = b.utterance(n)
        s = O.simple_loss(d["am"], d["lm"], d["y"])
        logits = d["am"][:, None, :].astype(np.float64) + d["lm"][None, :, :]
        ref, g = _torchaudio_rnnt(logits, d["y"])
        assert abs(s["loss"] - ref) < 2e-5 * abs(ref)
        # torchaudio runs its recursion in fp32 (|alpha| ~ 200 here), so compare normwise
        for mine, theirs in ((s["am_grad"], g.sum(axis=1)), (s["lm_grad"], g.sum(axis=0))):
            assert np.linalg.norm(mine - theirs) < 1e-3 * np.linalg.norm(theirs)


def test_simple_grads_finite_differences():
    rng = np.random.default_rng(11)
    T, U, V = 4, 2, 5
    am = rng.standard_normal((T, V))
    lm = rng.standard_normal((U + 1, V))
    y = np.array([3, 1])
    s = O.simple_loss(am, lm, y, grad_scale=0.5)
    h = 1e-6

    def f(a, l):
        return 0.5 * O.simple_loss(a, l, y, with_grads=False)["loss"]
    for t in range(T):
        for v in range(V):
            a = am.copy(); a[t, v] += h
            b_ = am.copy(); b_[t, v] -= h
            assert abs((f(a, lm) - f(b_, lm)) / (2 * h) - s["am_grad"][t, v]) < 1e-7
    for u in range(U + 1):
        for v in range(V):
            a = lm.copy(); a[u, v] += h
            b_ = lm.copy(); b_[u, v] -= h
            assert abs((f(am, a) - f(am, b_)) / (2 * h) - s["lm_grad"][u, v]) < 1e-7
    # rows of am_grad / lm_grad sum to zero (softmax gradient)
    assert np.allclose(s["am_grad"].sum(axis=1), 0, atol=1e-12)
    assert np.allclose(s["lm_grad"].sum(axis=1), 0, atol=1e-12)
