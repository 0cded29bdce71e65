"""Pins of the oracle's lattice recursion and occupancies
against things other than itself: hand values, brute-force path enumeration,
binomial closed forms, finite differences and the occupancy sum rules."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_examples.json")))


def _f(x):
    return -math.inf if x == "-inf" else float(x)


def rand_lattice(rng, T, U, scale=1.0):
    """Random normalised arcs: per node softmax over {y, blank, rest} so arcs are log-probs."""
    logits = scale * rng.standard_normal((T, U + 1, 3))
    lp = logits - O.logsumexp(logits, axis=2)[..., None]
    px = lp[..., 0].copy()
    px[:, U] = -np.inf
    py = lp[..., 1].copy()
    return px, py


@pytest.mark.parametrize("case", GOLD["log_add"])
def test_log_add_hand_values(case):
    out = float(O.log_add(_f(case["x"]), _f(case["y"])))
    exp = _f(case["out"])
    if math.isinf(exp):
        assert out == exp
    else:
        assert abs(out - exp) < 1e-12


def test_log_add_commutative_associative():
    rng = np.random.default_rng(0)
    a, b, c = rng.uniform(-50, 50, (3, 1000))
    assert np.allclose(O.log_add(a, b), O.log_add(b, a), atol=1e-12)
    assert np.allclose(O.log_add(O.log_add(a, b), c), O.log_add(a, O.log_add(b, c)), atol=1e-12)
    assert np.all(O.log_add(a, -np.inf) == a)


def test_uniform_T2_U1_hand_example():
    g = GOLD["uniform_T2_U1"]
    px = np.full((2, 2), g["arc"])
    px[:, 1] = -np.inf
    py = np.full((2, 2), g["arc"])
    alpha = O.forward_alpha(px, py)
    assert abs(alpha[1, 1] - g["alpha11"]) < 1e-14
    L, ypr, bpr = O.occupancies(px, py)
    assert abs(L - g["L_tot"]) < 1e-14
    assert np.allclose(ypr, g["px_grad"], atol=1e-14)
    assert np.allclose(bpr, g["py_grad"], atol=1e-14)


@pytest.mark.parametrize("T,U", [(1, 0), (1, 3), (2, 1), (3, 2), (4, 4), (5, 3), (7, 4), (5, 0)])
def test_alpha_equals_brute_force(T, U):
    rng = np.random.default_rng(T * 10 + U)
    for _ in range(5):
        px, py = rand_lattice(rng, T, U, scale=2.0)
        L = O.total_logprob(px, py)
        assert abs(L - O.brute_force_logprob(px, py)) < 1e-10
        beta = O.backward_beta(px, py)
        assert abs(beta[0, 0] - L) < 1e-10


@pytest.mark.parametrize("T,U,V", [(3, 2, 3), (12, 8, 7), (300, 80, 500), (1000, 250, 8000)])
def test_uniform_closed_form(T, U, V):
    """Uniform arcs -ln V: L = ln C(T-1+U, U) - (T+U) ln V (path counting)."""
    px = np.full((T, U + 1), -math.log(V))
    px[:, U] = -np.inf
    py = np.full((T, U + 1), -math.log(V))
    L = O.total_logprob(px, py)
    exact = (math.lgamma(T + U) - math.lgamma(U + 1) - math.lgamma(T)) - (T + U) * math.log(V)
    assert abs(L - exact) <= 1e-9 * max(1.0, abs(exact))


@pytest.mark.parametrize("T,U", [(9, 5), (40, 12)])
def test_uniform_occupancy_closed_form(T, U):
    """With uniform arcs, y'(t,u) = C(t+u,u) C(T-2-t+U-u, U-u-1) / C(T-1+U,U) and
    empty'(t,u) = C(t+u,u) C(T-2-t+U-u, U-u) / C(T-1+U,U) for t<T-1 (path counting)."""
    px = np.full((T, U + 1), -1.0)
    px[:, U] = -np.inf
    py = np.full((T, U + 1), -1.0)
    L, ypr, bpr = O.occupancies(px, py)
    tot = math.comb(T - 1 + U, U)
    for t in range(T):
        for u in range(U + 1):
            into = math.comb(t + u, u)
            if u < U:
                rest = T - 1 - t + U - u - 1
                ey = into * (math.comb(rest, U - u - 1) if rest >= 0 else 0) / tot
                assert abs(ypr[t, u] - ey) < 1e-12
            if t < T - 1:
                rest = T - 2 - t + U - u
                eb = into * math.comb(rest, U - u) / tot
                assert abs(bpr[t, u] - eb) < 1e-12
    assert abs(bpr[T - 1, U] - 1.0) < 1e-14


def test_single_path_special_cases():
    rng = np.random.default_rng(3)
    # U = 0: one path, all blanks
    px, py = rand_lattice(rng, 6, 0)
    assert abs(O.total_logprob(px, py) - py[:, 0].sum()) < 1e-12
    # T = 1: one path, all tokens then the terminal blank
    px, py = rand_lattice(rng, 1, 5)
    assert abs(O.total_logprob(px, py) - (px[0, :5].sum() + py[0, 5])) < 1e-12


def test_occupancies_match_finite_differences():
    rng = np.random.default_rng(7)
    T, U = 5, 3
    px, py = rand_lattice(rng, T, U, scale=1.5)
    L, ypr, bpr = O.occupancies(px, py)
    h = 1e-5
    for arr, grad in ((px, ypr), (py, bpr)):
        for t in range(T):
            for u in range(U + 1):
                if not np.isfinite(arr[t, u]):
                    continue
                a = arr.copy(); a[t, u] += h
                b = arr.copy(); b[t, u] -= h
                if arr is px:
                    fd = (O.total_logprob(a, py) - O.total_logprob(b, py)) / (2 * h)
                else:
                    fd = (O.total_logprob(px, a) - O.total_logprob(px, b)) / (2 * h)
                assert abs(fd - grad[t, u]) < 1e-7


@pytest.mark.parametrize("T,U", [(20, 7), (60, 20), (7, 0), (1, 6)])
def test_occupancy_sum_rules(T, U):
    """Every path leaves each frame by exactly one blank (sum_u empty'(t,u)=1), emits each
    token once (sum_t y'(t,u)=1, u<U), and leaves each anti-diagonal once."""
    rng = np.random.default_rng(T + U)
    px, py = rand_lattice(rng, T, U, scale=3.0)
    L, ypr, bpr = O.occupancies(px, py)
    assert np.allclose(bpr.sum(axis=1), 1.0, atol=1e-10)
    if U > 0:
        assert np.allclose(ypr[:, :U].sum(axis=0), 1.0, atol=1e-10)
    for k in range(T + U):
        s = sum(ypr[t, k - t] + bpr[t, k - t] for t in range(T) if 0 <= k - t <= U)
        assert abs(s - 1.0) < 1e-10
    assert ypr.min() >= 0 and bpr.min() >= 0 and ypr.max() <= 1 + 1e-12 and bpr.max() <= 1 + 1e-12
