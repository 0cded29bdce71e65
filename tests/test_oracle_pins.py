"""Round-2 pins of oracle parts that were only checked against themselves:

* the smoothed trivial joiner's L_dec^avg (Eq. 15) and L_acoustic (Eq. 13), against hand-derived
  fractions at T=2, U=1, V=3 (tests/golden/hand_pins_r2.json) -- fails if L_dec^avg is dropped from
  L_acoustic or averaged over u < U instead of u <= U;
* the band's upper edge u < p_t + S, against a hand-counted band and path count;
* bf16_round (D6 matched mode), against torch's own fp32 -> bf16 conversion;
* the bound adjustment (D3) on the inputs where it differs from SPEC.md's forward clamp.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_pins_r2.json")))


def _lg(fr):
    return math.log(Fraction(fr))


def _terms(pairs):
    return sum(float(Fraction(w)) * _lg(p) for w, p in pairs)


# ------------------------------------------------------------------ smoothed joiner
def _smoothed_case():
    g = GOLD["smoothed_U1_V3"]
    am = np.array([[_lg(x) for x in row] for row in g["am_probs"]])
    lm = np.array([[_lg(x) for x in row] for row in g["lm_probs"]])
    return g, am, lm, np.array(g["y"], np.int64)


def test_smoothed_parts_hand_golden():
    g, am, lm, _ = _smoothed_case()
    L_lm, Lavg, L_ac = O.smoothed_parts(am, lm)
    ref_lm = np.array([[_lg(x) for x in row] for row in g["L_lm_probs"]])
    ref_avg = np.array([_lg(x) for x in g["L_dec_avg_probs"]])
    ref_ac = np.array([[_lg(x) for x in row] for row in g["L_acoustic_probs"]])
    assert np.allclose(L_lm, ref_lm, atol=1e-14, rtol=0)
    assert np.allclose(Lavg, ref_avg, atol=1e-14, rtol=0)
    assert np.allclose(L_ac, ref_ac, atol=1e-14, rtol=0)


def test_smoothed_lattice_and_loss_hand_golden():
    g, am, lm, y = _smoothed_case()
    px, py = O.smoothed_lattice(am, lm, y, g["a_lm"], g["a_ac"])
    for key, pairs in g["px_terms"].items():
        t, u = map(int, key.split(","))
        assert abs(px[t, u] - _terms(pairs)) < 1e-14, ("px", key)
    for key, pairs in g["py_terms"].items():
        t, u = map(int, key.split(","))
        assert abs(py[t, u] - _terms(pairs)) < 1e-14, ("py", key)
    assert np.isneginf(px[:, 1]).all()
    # the two paths of a T=2, U=1 lattice, built from the hand terms only
    pxh = {k: _terms(v) for k, v in g["px_terms"].items()}
    pyh = {k: _terms(v) for k, v in g["py_terms"].items()}
    a = pxh["0,0"] + pyh["0,1"] + pyh["1,1"]
    b = pyh["0,0"] + pxh["1,0"] + pyh["1,1"]
    ref = -(max(a, b) + math.log1p(math.exp(min(a, b) - max(a, b))))
    got = O.smoothed_loss(am, lm, y, g["a_lm"], g["a_ac"], with_grads=False)["loss"]
    assert abs(got - ref) < 1e-13


def test_smoothed_golden_rejects_plausible_mistakes():
    """The golden distinguishes the readings a plausible slip would produce."""
    g, am, lm, _ = _smoothed_case()
    sm = np.exp(lm - np.log(np.exp(lm).sum(1, keepdims=True)))
    wrong_avg = np.log(sm[:-1].mean(0))                        # mean over u < U
    ref_avg = np.array([_lg(x) for x in g["L_dec_avg_probs"]])
    assert np.max(np.abs(wrong_avg - ref_avg)) > 0.1
    no_avg = am - np.log(np.exp(am).sum(1, keepdims=True))     # L_acoustic without L_dec^avg
    ref_ac = np.array([[_lg(x) for x in row] for row in g["L_acoustic_probs"]])
    assert np.max(np.abs(no_avg - ref_ac)) > 0.1


# ---------------------------------------------------------------------- band edge
def test_band_mask_hand_golden():
    g = GOLD["band_T4_U3_S2"]
    m = O.band_mask(np.array(g["ranges"]), g["U"], g["S"])
    assert m.astype(int).tolist() == g["band"]


@pytest.mark.parametrize("V", [5, 16])
def test_band_path_count_hand_golden(V):
    """W_out = 0, b = 0: every in-band arc is -ln V, so L_pruned = ln(n_paths) - (T+U) ln V with the
    hand-counted n_paths = 2."""
    g = GOLD["band_T4_U3_S2"]
    T, U, S, J = g["T"], g["U"], g["S"], 8
    rng = np.random.default_rng(7)
    enc, dec = rng.standard_normal((T, J)), rng.standard_normal((U + 1, J))
    y = rng.integers(1, V, size=U)
    out = O.pruned_loss(enc, dec, np.zeros((V, J)), np.zeros(V), y, np.array(g["ranges"]), S, with_grads=False)
    assert abs(-out["loss"] - (math.log(g["n_paths"]) - (T + U) * math.log(V))) < 1e-12


# ------------------------------------------------------------------------ bf16
def test_bf16_round_matches_torch():
    rng = np.random.default_rng(11)
    x = np.concatenate([
        rng.standard_normal(400_000) * 10.0 ** rng.integers(-6, 6, size=400_000),
        rng.uniform(-1, 1, 400_000),
        np.tanh(rng.standard_normal(200_000) * 3),
    ]).astype(np.float32)
    # exact ties (lower 16 bits = 0x8000, both parities of bit 16) and their neighbours
    base = rng.integers(0x3F000000, 0x40800000, size=20_000, dtype=np.int64) & ~0xFFFF
    ties = np.concatenate([base | 0x8000, base | 0x7FFF, base | 0x8001, (base | 0x10000) | 0x8000])
    x = np.concatenate([x, ties.astype(np.uint32).view(np.float32), np.float32([0.0, -0.0, 1e-40, -1e-40])])
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    got = O.bf16_round(x.astype(np.float64))
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)) or np.array_equal(got, ref)
    assert np.array_equal(got, ref)


# ------------------------------------------------------------- bound adjustment
@pytest.mark.parametrize("case", GOLD["adjust_spec_deviation"]["cases"], ids=lambda c: str(c["raw"]))
def test_adjust_bounds_spec_deviation_cases(case):
    p = O.adjust_bounds(np.array(case["raw"]), case["T"], case["U"], case["S"])
    assert p.tolist() == case["p"]
    # both the D3 result and SPEC's hand result are feasible band sequences (Eq. 9-10 + endpoints)
    for seq in (case["p"], case["spec"]):
        s = np.array(seq)
        Um = max(0, case["U"] - case["S"] + 1)
        assert s[0] == 0 and s[-1] == Um
        assert np.all(np.diff(s) >= 0) and np.all(np.diff(s) <= case["S"] - 1)
