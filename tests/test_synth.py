"""The seeded generator is deterministic and honours the BASELINE.json config recipes."""
import math

import numpy as np
import pytest

import synth


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_deterministic(cfg):
    a, b = synth.make_batch(cfg), synth.make_batch(cfg)
    for k in ("am", "lm", "enc_proj", "dec_proj", "symbols", "w_out_bits", "b_out_bits", "T_n", "U_n"):
        assert np.array_equal(getattr(a, k), getattr(b, k))
    c = synth.make_batch(cfg, rank=1)
    assert not np.array_equal(a.am[:, :5, :5], c.am[:, :5, :5])


def test_config_recipes():
    b = synth.make_batch(2)
    assert b.N == 32 and b.V == 500 and b.J == 512 and b.S == 5
    assert np.all((b.T_n >= 200) & (b.T_n <= 500))
    for t, u in zip(b.T_n, b.U_n):
        assert math.ceil(t / 8) <= u <= t // 3
    for n in range(b.N):
        y = b.symbols[n, :b.U_n[n]]
        assert np.all((y >= 1) & (y < b.V))
    c3 = synth.make_batch(3)
    assert np.all((c3.U_n >= 10) & (c3.U_n <= 60))
    toks = np.concatenate([c3.symbols[n, :c3.U_n[n]] for n in range(c3.N)])
    assert np.all((toks >= 1) & (toks < 5000))
    assert np.mean(toks == 1) > 0.05        # Zipf(1.1): rank 1 is frequent
    c1 = synth.make_batch(1)
    assert list(c1.T_n) == [8, 6] and list(c1.U_n) == [3, 2] and c1.S == 3 and c1.J == 8


def test_bf16_cast_round_to_nearest_even():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -2.5, 3.14159], np.float32)
    bits = synth.f32_to_bf16_bits(x)
    back = synth.bf16_bits_to_f32(bits)
    assert back[0] == 1.0 and back[1] == 1.0          # tie -> even
    assert back[2] == np.float32(1.0 + 4 * 2 ** -8)    # tie -> even (up)
    assert back[3] == -2.5
    assert abs(back[4] - 3.14159) < 2 ** -7 * 4


def test_poison_padding():
    b = synth.make_batch(2, poison=True)
    n = int(np.argmin(b.T_n))
    assert np.all(np.isnan(b.am[n, b.T_n[n]:]))
    assert np.all(np.isfinite(b.am[n, :b.T_n[n]]))


def test_dynamic_corpus_packing():
    """Table-2 protocol (PAPER.md 384-386): sorted lengths, every batch under the frame cap, all
    utterances used once, shared joiner weights."""
    import synth
    c = synth.make_dynamic_corpus(n_utts=64)
    assert sum(b.N for b in c) == 64
    Ts = np.concatenate([b.T_n for b in c])
    assert np.all(np.diff(Ts) >= 0)
    for b in c:
        assert int(b.T_n.sum()) <= synth.DYNAMIC_CAP_FRAMES
        assert np.array_equal(b.w_out_bits, c[0].w_out_bits)
    for b0, b1 in zip(c[:-1], c[1:]):   # greedy: the next utterance would not have fit
        assert int(b0.T_n.sum()) + int(b1.T_n[0]) > synth.DYNAMIC_CAP_FRAMES
