"""Seeded synthetic inputs for the pruned RNN-T hot path (BASELINE.json configs 1-5).

This module is shared by the oracle (``oracle/``) and the CUDA path
(``paper_2206_13236_b200``).  It holds NO arithmetic of the method: it only
draws lengths, labels and input tensors from a seeded generator and pads them.
The one numeric operation it performs is the storage cast of the joiner
weights to bf16 (round-to-nearest-even), which is a property of the *inputs*
(BASELINE.json: "joiner weights bf16 Xavier"), not of the loss.

Shapes stand in for the paper's LibriSpeech test-clean / Chinese-character
workloads (Sec. 4.1), which are not in the container;
see DESIGN.md "Input recipe".

Draw order (fixed): lengths, symbols, am, lm, enc_proj, dec_proj,
W_out, b_out, from ``numpy.random.Generator(PCG64(seed))`` with
``seed = 2206_13236 + 100*config + rank`` unless given explicitly.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEED_BASE = 2206_13236

# BASELINE.json "configs" (1-based, in the order listed there).
CONFIGS = {
    1: dict(name="c1-tiny", N=2, T=(8, 6), U=(3, 2), V=16, J=8, S=3, labels="uniform"),
    2: dict(name="c2-librispeech-bpe", N=32, T_range=(200, 500), U_rule="T/8..T/3",
            V=500, J=512, S=5, labels="uniform"),
    3: dict(name="c3-chinese-char", N=32, T_range=(100, 400), U_range=(10, 60),
            V=5000, J=512, S=5, labels="zipf1.1"),
    4: dict(name="c4-long-utterance", N=16, T_fixed=1000, U_fixed=250, V=8000, J=768, S=10,
            labels="uniform"),
    5: dict(name="c5-dp8", N=32, T_range=(200, 500), U_rule="T/8..T/3", V=500, J=512, S=5,
            labels="uniform"),
}


@dataclasses.dataclass
class Batch:
    """One padded batch.  Padded entries are 0 (perf mode) or NaN (poison mode)."""
    config: int
    N: int
    T: int            # padded max frames  (T-hat)
    U: int            # padded max tokens  (U-hat)
    V: int
    J: int
    S: int
    T_n: np.ndarray   # (N,) int64 real frames
    U_n: np.ndarray   # (N,) int64 real tokens
    symbols: np.ndarray   # (N, U) int64, y_1..y_U in [1, V); padding 0
    boundary: np.ndarray  # (N, 4) int64 {0, 0, U_n, T_n}
    am: np.ndarray        # (N, T, V) float32
    lm: np.ndarray        # (N, U+1, V) float32
    enc_proj: np.ndarray  # (N, T, J) float32
    dec_proj: np.ndarray  # (N, U+1, J) float32
    w_out_bits: np.ndarray  # (V, J) uint16 bf16 bit patterns
    b_out_bits: np.ndarray  # (V,) uint16 bf16 bit patterns

    @property
    def w_out(self) -> np.ndarray:
        """W_out values as float32 (exact: bf16 widened)."""
        return bf16_bits_to_f32(self.w_out_bits)

    @property
    def b_out(self) -> np.ndarray:
        return bf16_bits_to_f32(self.b_out_bits)

    @property
    def frames(self) -> int:
        return int(self.T_n.sum())

    def utterance(self, n: int) -> dict:
        """Unpadded per-utterance view (numpy arrays, no copies of padding)."""
        T, U = int(self.T_n[n]), int(self.U_n[n])
        return dict(T=T, U=U, V=self.V, J=self.J, S=self.S,
                    y=self.symbols[n, :U].copy(),
                    am=self.am[n, :T], lm=self.lm[n, :U + 1],
                    enc=self.enc_proj[n, :T], dec=self.dec_proj[n, :U + 1],
                    W=self.w_out, b=self.b_out)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Storage cast fp32 -> bf16 with round-to-nearest-even (finite inputs)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def _zipf_tokens(rng: np.random.Generator, size: int, V: int, s: float = 1.1) -> np.ndarray:
    """Finite-support Zipf(s) over ranks 1..V-1, token id = rank (inverse CDF)."""
    ranks = np.arange(1, V, dtype=np.float64)
    cdf = np.cumsum(ranks ** (-s))
    cdf /= cdf[-1]
    u = rng.random(size)
    return (np.searchsorted(cdf, u, side="right") + 1).clip(1, V - 1).astype(np.int64)


def draw_lengths(cfg: dict, rng: np.random.Generator, N: int):
    if "T_fixed" in cfg:
        return (np.full(N, cfg["T_fixed"], np.int64), np.full(N, cfg["U_fixed"], np.int64))
    if "T" in cfg:  # explicit tiny lists
        return np.array(cfg["T"], np.int64), np.array(cfg["U"], np.int64)
    lo, hi = cfg["T_range"]
    T_n = rng.integers(lo, hi + 1, size=N).astype(np.int64)
    if cfg.get("U_rule") == "T/8..T/3":
        U_n = np.array([rng.integers(math.ceil(t / 8), t // 3 + 1) for t in T_n], np.int64)
    else:
        ulo, uhi = cfg["U_range"]
        U_n = rng.integers(ulo, uhi + 1, size=N).astype(np.int64)
    return T_n, U_n


def make_batch(config: int, rank: int = 0, seed: int | None = None, poison: bool = False,
               N: int | None = None, zero_logits: bool = False) -> Batch:
    """Draw one synthetic batch for ``config`` (1..5).

    ``poison`` fills every padded element with NaN (labels with 0) so tests can
    check padded inputs are never read.  ``zero_logits`` sets am = lm = 0 and
    W_out = b_out = 0 after drawing (the uniform full-size pins of SURVEY 8(c)).
    """
    cfg = CONFIGS[config]
    if seed is None:
        seed = SEED_BASE + 100 * config + rank
    rng = np.random.Generator(np.random.PCG64(seed))
    N = cfg["N"] if N is None else N
    V, J, S = cfg["V"], cfg["J"], cfg["S"]
    T_n, U_n = draw_lengths(cfg, rng, N)
    Tm, Um = int(T_n.max()), int(U_n.max())

    symbols = np.zeros((N, Um), np.int64)
    for n in range(N):
        u = int(U_n[n])
        if cfg["labels"] == "zipf1.1":
            symbols[n, :u] = _zipf_tokens(rng, u, V)
        else:
            symbols[n, :u] = rng.integers(1, V, size=u)

    fill = np.float32(np.nan) if poison else np.float32(0)
    am = np.full((N, Tm, V), fill, np.float32)
    lm = np.full((N, Um + 1, V), fill, np.float32)
    enc = np.full((N, Tm, J), fill, np.float32)
    dec = np.full((N, Um + 1, J), fill, np.float32)
    for n in range(N):
        am[n, :T_n[n]] = rng.standard_normal((int(T_n[n]), V), dtype=np.float32)
    for n in range(N):
        lm[n, :U_n[n] + 1] = rng.standard_normal((int(U_n[n]) + 1, V), dtype=np.float32)
    for n in range(N):
        enc[n, :T_n[n]] = rng.standard_normal((int(T_n[n]), J), dtype=np.float32)
    for n in range(N):
        dec[n, :U_n[n] + 1] = rng.standard_normal((int(U_n[n]) + 1, J), dtype=np.float32)
    a = math.sqrt(6.0 / (J + V))  # Xavier-uniform bound; reused for b (D13)
    # c5 (data parallel): every rank shares the joiner weights, so they come from a rank-independent
    # stream; the other configs keep the single fixed draw order.
    wrng = np.random.Generator(np.random.PCG64(SEED_BASE + 100 * config)) if config == 5 else rng
    W = wrng.uniform(-a, a, size=(V, J)).astype(np.float32)
    b = wrng.uniform(-a, a, size=(V,)).astype(np.float32)
    if zero_logits:
        for n in range(N):
            am[n, :T_n[n]] = 0
            lm[n, :U_n[n] + 1] = 0
        W[:] = 0
        b[:] = 0
    boundary = np.zeros((N, 4), np.int64)
    boundary[:, 2] = U_n
    boundary[:, 3] = T_n
    return Batch(config=config, N=N, T=Tm, U=Um, V=V, J=J, S=S, T_n=T_n, U_n=U_n,
                 symbols=symbols, boundary=boundary, am=am, lm=lm, enc_proj=enc, dec_proj=dec,
                 w_out_bits=f32_to_bf16_bits(W), b_out_bits=f32_to_bf16_bits(b))


def make_custom(T_n, U_n, V, J, S, seed=0, logit_scale=1.0, poison=False, joiner_scale=1.0) -> Batch:
    """Arbitrary-shape batch for edge-case tests (same draw order as make_batch).  ``logit_scale``
    multiplies am / lm, ``joiner_scale`` W_out / b_out (peaky, trained-like lattices)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    T_n = np.asarray(T_n, np.int64)
    U_n = np.asarray(U_n, np.int64)
    N = len(T_n)
    Tm, Um = int(T_n.max()), int(U_n.max())
    symbols = np.zeros((N, Um), np.int64)
    for n in range(N):
        symbols[n, :U_n[n]] = rng.integers(1, V, size=int(U_n[n]))
    fill = np.float32(np.nan) if poison else np.float32(0)
    am = np.full((N, Tm, V), fill, np.float32)
    lm = np.full((N, Um + 1, V), fill, np.float32)
    enc = np.full((N, Tm, J), fill, np.float32)
    dec = np.full((N, Um + 1, J), fill, np.float32)
    for n in range(N):
        am[n, :T_n[n]] = logit_scale * rng.standard_normal((int(T_n[n]), V), dtype=np.float32)
    for n in range(N):
        lm[n, :U_n[n] + 1] = logit_scale * rng.standard_normal((int(U_n[n]) + 1, V), dtype=np.float32)
    for n in range(N):
        enc[n, :T_n[n]] = rng.standard_normal((int(T_n[n]), J), dtype=np.float32)
    for n in range(N):
        dec[n, :U_n[n] + 1] = rng.standard_normal((int(U_n[n]) + 1, J), dtype=np.float32)
    a = math.sqrt(6.0 / (J + V))
    W = (joiner_scale * rng.uniform(-a, a, size=(V, J))).astype(np.float32)
    b = (joiner_scale * rng.uniform(-a, a, size=(V,))).astype(np.float32)
    boundary = np.zeros((N, 4), np.int64)
    boundary[:, 2] = U_n
    boundary[:, 3] = T_n
    return Batch(config=0, N=N, T=Tm, U=Um, V=V, J=J, S=S, T_n=T_n, U_n=U_n, symbols=symbols,
                 boundary=boundary, am=am, lm=lm, enc_proj=enc, dec_proj=dec,
                 w_out_bits=f32_to_bf16_bits(W), b_out_bits=f32_to_bf16_bits(b))


# Dynamic-batch workload (Table 2): utterances sorted by
# duration and packed so that the frames of a batch BEFORE padding stay within 10k input frames at
# 100 fps, i.e. 2,500 encoder frames after the 4x subsampling the c2 lengths already assume
# (reading D17).  Lengths follow the c2 recipe; the joiner weights are shared by all batches.
DYNAMIC_CAP_FRAMES = 2500


def make_dynamic_corpus(n_utts: int = 320, cap: int = DYNAMIC_CAP_FRAMES, seed: int | None = None) -> list:
    """List of Batch: n_utts c2-shaped utterances, sorted by T, greedily packed under ``cap``."""
    seed = SEED_BASE + 600 if seed is None else seed
    rng = np.random.Generator(np.random.PCG64(seed))
    T_n, U_n = draw_lengths(CONFIGS[2], rng, n_utts)
    order = np.argsort(T_n, kind="stable")
    T_n, U_n = T_n[order], U_n[order]
    groups, cur, tot = [], [], 0
    for i in range(n_utts):
        if cur and tot + int(T_n[i]) > cap:
            groups.append(cur)
            cur, tot = [], 0
        cur.append(i)
        tot += int(T_n[i])
    if cur:
        groups.append(cur)
    cfg = CONFIGS[2]
    V, J, S = cfg["V"], cfg["J"], cfg["S"]
    a = math.sqrt(6.0 / (J + V))
    W = rng.uniform(-a, a, size=(V, J)).astype(np.float32)
    b = rng.uniform(-a, a, size=(V,)).astype(np.float32)
    wb, bb = f32_to_bf16_bits(W), f32_to_bf16_bits(b)
    out = []
    for k, g in enumerate(groups):
        bt = make_custom(T_n[g], U_n[g], V, J, S, seed=seed + 1 + k)
        bt.config = 6
        bt.w_out_bits, bt.b_out_bits = wb, bb
        out.append(bt)
    return out
