"""Pins of the smoothed trivial joiner (Eq. 11-15, D18):
reduction to the plain trivial joiner, closed forms of the pure LM-only and pure acoustic-only
lattices by a DP independent of the lattice recursion, the uniform closed form, brute-force path
enumeration, and central finite differences of the loss w.r.t. am and lm."""
import math

import numpy as np
import pytest

import oracle as O


def _rand(T, U, V, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    am = scale * rng.standard_normal((T, V))
    lm = scale * rng.standard_normal((U + 1, V))
    y = rng.integers(1, V, size=U)
    return am, lm, y


def test_zero_scales_is_the_trivial_joiner():
    am, lm, y = _rand(7, 4, 9, 1)
    a = O.smoothed_loss(am, lm, y, 0.0, 0.0, 0.5)
    b = O.simple_loss(am, lm, y, 0.5)
    for k in ("loss", "px_grad", "py_grad", "am_grad", "lm_grad"):
        assert np.allclose(a[k], b[k], atol=1e-12, rtol=1e-12), k


def test_lm_only_closed_form():
    """a_lm = 1: px(t,u) = L_lm(u, y_{u+1}), py(t,u) = L_lm(u, 0) do not depend on t.  Every path emits
    each label once and T blanks, b_u of them on row u with sum b_u = T and b_U >= 1 (terminal blank),
    so L = sum_u L_lm(u, y_{u+1}) + log(x_U h_{T-1}(x_0..x_U)), x_u = exp L_lm(u, 0), h_k the complete
    homogeneous symmetric polynomial (computed by its own recurrence)."""
    T, U, V = 6, 3, 5
    am, lm, y = _rand(T, U, V, 2)
    L_lm = O.log_softmax(lm, axis=1)
    x = np.exp(L_lm[:, 0])
    h = np.zeros(T)                      # h_k over the variables seen so far, k = 0..T-1
    h[0] = 1.0
    for j in range(U + 1):
        for k in range(1, T):
            h[k] = h[k] + x[j] * h[k - 1]
    ref = sum(L_lm[u, y[u]] for u in range(U)) + math.log(x[U] * h[T - 1])
    got = -O.smoothed_loss(am, lm, y, 1.0, 0.0)["loss"]
    assert abs(got - ref) < 1e-10


def test_acoustic_only_closed_form():
    """a_ac = 1: px(t,u) = L_ac(t, y_{u+1}), py(t,u) = L_ac(t, 0) do not depend on u.  Every path has
    exactly one blank out of each frame (sum_t L_ac(t,0)) and emits label u+1 at a frame t_u with
    t_0 <= t_1 <= ... <= t_{U-1}: a DP over non-decreasing frame sequences."""
    T, U, V = 5, 3, 6
    am, lm, y = _rand(T, U, V, 3)
    _, _, L_ac = O.smoothed_parts(am, lm)
    e = np.exp(L_ac[:, y])               # (T, U): weight of emitting label u+1 at frame t
    f = e[:, 0].copy()                   # f[t] = sum over sequences ending with t_0 = t
    for u in range(1, U):
        f = np.cumsum(f) * e[:, u]
    ref = L_ac[:, 0].sum() + math.log(f.sum())
    got = -O.smoothed_loss(am, lm, y, 0.0, 1.0)["loss"]
    assert abs(got - ref) < 1e-10


def test_uniform_closed_form():
    """am = lm = 0: the trivial, LM-only and acoustic distributions are all uniform, so every arc is
    -ln V for any scales and L = ln C(T-1+U, U) - (T+U) ln V."""
    T, U, V = 9, 4, 7
    am, lm = np.zeros((T, V)), np.zeros((U + 1, V))
    y = np.arange(1, U + 1)
    ref = math.log(math.comb(T - 1 + U, U)) - (T + U) * math.log(V)
    for a_lm, a_ac in ((0.25, 0.0), (0.0, 0.25), (0.3, 0.2)):
        assert abs(-O.smoothed_loss(am, lm, y, a_lm, a_ac)["loss"] - ref) < 1e-10


def test_brute_force_paths():
    am, lm, y = _rand(5, 2, 6, 4)
    px, py = O.smoothed_lattice(am, lm, y, 0.2, 0.15)
    got = -O.smoothed_loss(am, lm, y, 0.2, 0.15)["loss"]
    assert abs(got - O.brute_force_logprob(px, py)) < 1e-10


def test_lavg_is_a_distribution():
    am, lm, y = _rand(4, 5, 11, 5)
    _, Lavg, L_ac = O.smoothed_parts(am, lm)
    assert abs(np.exp(Lavg).sum() - 1.0) < 1e-12
    assert np.allclose(np.exp(L_ac).sum(axis=1), 1.0, atol=1e-12)


@pytest.mark.parametrize("a_lm,a_ac", [(0.25, 0.0), (0.0, 0.25), (0.1, 0.3)])
def test_finite_differences(a_lm, a_ac):
    am, lm, y = _rand(4, 3, 5, 6)
    r = O.smoothed_loss(am, lm, y, a_lm, a_ac, 1.0)
    eps = 1e-6
    f = lambda a, l: O.smoothed_loss(a, l, y, a_lm, a_ac, 1.0, with_grads=False)["loss"]
    for t in range(am.shape[0]):
        for v in range(am.shape[1]):
            d = np.zeros_like(am); d[t, v] = eps
            fd = (f(am + d, lm) - f(am - d, lm)) / (2 * eps)
            assert abs(fd - r["am_grad"][t, v]) < 1e-7, ("am", t, v)
    for u in range(lm.shape[0]):
        for v in range(lm.shape[1]):
            d = np.zeros_like(lm); d[u, v] = eps
            fd = (f(am, lm + d) - f(am, lm - d)) / (2 * eps)
            assert abs(fd - r["lm_grad"][u, v]) < 1e-7, ("lm", u, v)
