"""Pins of the pruning-bound stage (Eq. 7-10)."""
import itertools
import json
import os

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_examples.json")))


def test_eq7_worked_example():
    g = GOLD["eq7_example"]
    vals = O.bound_scores(np.array(g["px_grad_row"]), np.array(g["py_grad_row"]), g["S"])
    assert abs(vals[g["p"]] - g["value"]) < 1e-12
    assert len(vals) == len(g["py_grad_row"]) - g["S"] + 1  # p = 0..U-S+1


def test_eq8_uniform_T2_U1_S1():
    """S:281 hand example: T=2, U=1 uniform, S=1 -> raw p = [0, 1]."""
    g = GOLD["uniform_T2_U1"]
    raw = O.raw_bounds(np.array(g["px_grad"]), np.array(g["py_grad"]), 1)
    assert list(raw) == [0, 1]


def _enter_leave_identity(px, py, S):
    """Independent formula for Eq. 8's candidate values (D5): by path
    enumeration, v_t(p) = P(path enters frame t at row >= p) - P(leaves frame t at row >= p+S)."""
    T, U1 = px.shape
    paths = list(O.brute_force_paths(T, U1 - 1))
    lps = np.array([sum(px[t, u] if k == "y" else py[t, u] for (t, u, k) in a) for a in paths])
    w = np.exp(lps - O.logsumexp(lps))
    out = np.zeros((T, O.umax(U1 - 1, S) + 1))
    for a, wi in zip(paths, w):
        rows = {}
        for (t, u, k) in a:
            rows.setdefault(t, []).append(u)
        for t in range(T):
            enter, leave = min(rows[t]), max(rows[t])
            for p in range(out.shape[1]):
                out[t, p] += wi * ((enter >= p) - (leave >= p + S))
    return out


@pytest.mark.parametrize("T,U,S", [(6, 4, 2), (5, 5, 3), (7, 3, 2), (4, 4, 4)])
def test_eq8_entry_exit_identity(T, U, S):
    rng = np.random.default_rng(T * 100 + U * 10 + S)
    logits = 1.5 * rng.standard_normal((T, U + 1, 3))
    lp = logits - O.logsumexp(logits, axis=2)[..., None]
    px, py = lp[..., 0].copy(), lp[..., 1].copy()
    px[:, U] = -np.inf
    L, ypr, bpr = O.occupancies(px, py)
    ident = _enter_leave_identity(px, py, S)
    for t in range(T):
        assert np.allclose(O.bound_scores(ypr[t], bpr[t], S), ident[t], atol=1e-12)


@pytest.mark.parametrize("case", GOLD["adjust_examples"])
def test_adjust_examples(case):
    assert list(O.adjust_bounds(case["raw"], case["T"], case["U"], case["S"])) == case["p"]


def test_infeasible_example():
    """T=2, U=3, S=2 has no band-respecting path (3 > 2*1)."""
    assert not O.feasible(2, 3, 2)
    assert O.feasible(2, 2, 2)


def _check_invariants(p, T, U, S):
    Um = O.umax(U, S)
    assert p[0] == 0 and p[-1] == Um
    assert np.all((0 <= p) & (p <= Um))
    assert np.all(np.diff(p) >= 0)           # Eq. 9
    assert np.all(np.diff(p) < S)            # Eq. 10


@settings(max_examples=3000, deadline=None)
@given(st.integers(1, 40), st.integers(1, 8), st.data())
def test_adjust_invariants_idempotent_fixed_point(T, S, data):
    U = data.draw(st.integers(0, T * (S - 1)))
    Um = O.umax(U, S)
    raw = np.array(data.draw(st.lists(st.integers(0, Um), min_size=T, max_size=T)))
    p = O.adjust_bounds(raw, T, U, S)
    _check_invariants(p, T, U, S)
    assert np.array_equal(O.adjust_bounds(p, T, U, S), p)
    feas = (raw[0] == 0 and raw[-1] == Um and np.all(np.diff(raw) >= 0) and np.all(np.diff(raw) < S))
    if feas:
        assert np.array_equal(p, raw)


def test_adjust_is_least_feasible_above_monotone_hull():
    """Brute force over ALL feasible sequences: ADJ-scan returns the pointwise least
    feasible sequence that dominates the monotone hull of the clamped raw bounds
    (the 'change as little as possible' reading, D3)."""
    rng = np.random.default_rng(0)
    for _ in range(150):
        T = int(rng.integers(1, 6)); S = int(rng.integers(2, 4))
        U = int(rng.integers(0, T * (S - 1) + 1)); Um = O.umax(U, S)
        raw = rng.integers(0, Um + 1, size=T)
        t = np.arange(T)
        lo = np.maximum(0, Um - (T - 1 - t) * (S - 1)); hi = np.minimum(Um, t * (S - 1))
        hull = np.maximum.accumulate(np.clip(raw, lo, hi))
        cands = []
        for seq in itertools.product(range(Um + 1), repeat=T):
            s = np.array(seq)
            if s[0] != 0 or s[-1] != Um or np.any(np.diff(s) < 0) or np.any(np.diff(s) >= S):
                continue
            if np.all(s >= hull):
                cands.append(s)
        least = np.min(np.array(cands), axis=0)
        assert any(np.array_equal(least, c) for c in cands)   # the set has a least element
        assert np.array_equal(O.adjust_bounds(raw, T, U, S), least)


def test_full_band_gives_zero_bounds():
    rng = np.random.default_rng(2)
    ypr = rng.random((9, 4)); bpr = rng.random((9, 4))
    assert np.all(O.raw_bounds(ypr, bpr, 4) == 0)
    assert np.all(O.adjust_bounds(rng.integers(0, 3, 9), 9, 3, 5) == 0)


def test_diagonal_occupancy_tracks_diagonal():
    """one-hot empty' on a strict diagonal -> p_t tracks it, clipped to [0,U-S+1]."""
    T, U, S = 10, 9, 3
    bpr = np.zeros((T, U + 1), np.float32); ypr = np.zeros((T, U + 1), np.float32)
    for t in range(T):
        bpr[t, t] = 1.0
    raw = O.raw_bounds(ypr, bpr, S)
    # v(p) = [p <= t <= p+S-1]; the smallest maximiser is max(0, t-S+1) (<= U-S+1 here)
    assert list(raw) == [max(0, t - S + 1) for t in range(T)]
