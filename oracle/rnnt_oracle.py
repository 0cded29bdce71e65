"""Plain, slow, fp64 oracle of the pruned RNN-T loss (arXiv 2206.13236).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Everything is a direct
transcription of the paper's definitions, in the paper's order and notation;
no blocking, fusion or matmul tricks beyond a library matmul / logsumexp used
as a single step.  ``P:<n>`` cites /root/reference/PAPER.md line n.

Lattice convention (D1/D2): frames t in [0,T),
token positions u in [0,U]; real tokens y_1..y_U in [1,V); blank id 0.
y(t,u) = L(t,u,y_{u+1}) (vertical arc, u<U), empty(t,u) = L(t,u,0) (horizontal
arc).  Arrays below are (T, U+1) with px = y(t,u), py = empty(t,u); px[:,U] = -inf.
"""
from __future__ import annotations

import math

import numpy as np

NEG_INF = -np.inf

__all__ = [
    "log_add", "logsumexp", "trivial_normalizer", "trivial_lattice", "forward_alpha",
    "backward_beta", "total_logprob", "occupancies", "simple_grads", "simple_loss",
    "bound_scores", "raw_bounds", "adjust_bounds", "bf16_round", "pruned_lattice", "pruned_loss",
    "brute_force_logprob", "brute_force_paths", "band_mask", "full_step", "feasible",
    "umax", "log_softmax", "smoothed_parts", "smoothed_lattice", "smoothed_loss",
]


# --------------------------------------------------------------------------- LogAdd
def log_add(x, y):
    """LogAdd(x,y) = log(e^x + e^y)  (Eq. 4).

    Computed as max + log1p(exp(min - max)); LogAdd(-inf,-inf) = -inf (D8)."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    m = np.maximum(x, y)
    n = np.minimum(x, y)
    with np.errstate(invalid="ignore"):
        d = n - m
    d = np.where(np.isneginf(m), NEG_INF, d)
    out = m + np.log1p(np.exp(d))
    return np.where(np.isneginf(m), NEG_INF, out)


def logsumexp(a, axis=-1):
    """log sum_v exp(a_v) along ``axis`` with the max taken out (library-style step)."""
    a = np.asarray(a, np.float64)
    m = np.max(a, axis=axis, keepdims=True)
    m_safe = np.where(np.isfinite(m), m, 0.0)
    with np.errstate(divide="ignore"):
        s = np.log(np.sum(np.exp(a - m_safe), axis=axis, keepdims=True)) + m_safe
    return np.squeeze(s, axis=axis)


# ------------------------------------------------------------ trivial joiner (Sec 3.1)
def trivial_normalizer(am, lm):
    """L_normalizer(t,u) = log sum_v exp(L_enc(t,v) + L_dec(u,v))  (Eq. 6).

    Direct definition (no matmul trick): for each t the (U+1, V) sum is formed
    explicitly and log-sum-exp'd.  am = L_enc (T,V), lm = L_dec (U+1,V)."""
    am = np.asarray(am, np.float64)
    lm = np.asarray(lm, np.float64)
    T = am.shape[0]
    out = np.empty((T, lm.shape[0]), np.float64)
    for t in range(T):
        out[t] = logsumexp(am[t][None, :] + lm, axis=1)
    return out


def trivial_lattice(am, lm, y):
    """(px, py, L_norm) of the trivial joiner (Eq. 5 with P:143-147 Eq. 1-2).

    px(t,u) = L_enc(t,y_{u+1}) + L_dec(u,y_{u+1}) - L_norm(t,u) for u<U, -inf at u=U.
    py(t,u) = L_enc(t,0) + L_dec(u,0) - L_norm(t,u)."""
    am = np.asarray(am, np.float64)
    lm = np.asarray(lm, np.float64)
    y = np.asarray(y, np.int64)
    T, U = am.shape[0], len(y)
    Lnorm = trivial_normalizer(am, lm)
    px = np.full((T, U + 1), NEG_INF)
    if U > 0:
        px[:, :U] = am[:, y] + lm[np.arange(U), y][None, :] - Lnorm[:, :U]
    py = am[:, 0][:, None] + lm[:, 0][None, :] - Lnorm
    return px, py, Lnorm


# ------------------------------------------------------- recursion (Sec 2, Eq. 3)
def forward_alpha(px, py):
    """alpha(t,u) = LogAdd(alpha(t-1,u)+empty(t-1,u), alpha(t,u-1)+y(t,u-1)), alpha(0,0)=0.

    P:153-168 (Eq. 3).  Evaluated over anti-diagonals k=t+u (vectorised in u);
    out-of-range terms are -inf."""
    T, U1 = px.shape
    alpha = np.full((T, U1), NEG_INF)
    alpha[0, 0] = 0.0
    for k in range(1, T + U1 - 1):
        u = np.arange(max(0, k - T + 1), min(U1 - 1, k) + 1)
        t = k - u
        from_left = np.where(t >= 1, alpha[np.maximum(t - 1, 0), u] + py[np.maximum(t - 1, 0), u],
                             NEG_INF)
        from_below = np.where(u >= 1, alpha[t, np.maximum(u - 1, 0)] + px[t, np.maximum(u - 1, 0)],
                              NEG_INF)
        alpha[t, u] = log_add(from_left, from_below)
    return alpha


def backward_beta(px, py):
    """beta(t,u): log-prob of finishing from node (t,u), terminal blank included.

    beta(T-1,U) = empty(T-1,U); beta(t,u) = LogAdd(beta(t+1,u)+empty(t,u), beta(t,u+1)+y(t,u)).
    The backward half of the forward-backward algorithm the paper names."""
    T, U1 = px.shape
    beta = np.full((T, U1), NEG_INF)
    beta[T - 1, U1 - 1] = py[T - 1, U1 - 1]
    for k in range(T + U1 - 3, -1, -1):
        u = np.arange(max(0, k - T + 1), min(U1 - 1, k) + 1)
        t = k - u
        right = np.where(t + 1 < T, beta[np.minimum(t + 1, T - 1), u] + py[t, u], NEG_INF)
        up = np.where(u + 1 < U1, beta[t, np.minimum(u + 1, U1 - 1)] + px[t, u], NEG_INF)
        beta[t, u] = log_add(right, up)
    return beta


def total_logprob(px, py):
    """L_tot = alpha(T-1,U) + empty(T-1,U)."""
    a = forward_alpha(px, py)
    return a[-1, -1] + py[-1, -1]


def occupancies(px, py):
    """(L_tot, y', empty') with y' = dL_tot/dy, empty' = dL_tot/dempty.

    y'(t,u)     = exp(alpha(t,u) + y(t,u)     + beta(t,u+1) - L_tot)
    empty'(t,u) = exp(alpha(t,u) + empty(t,u) + beta(t+1,u) - L_tot), with the
    terminal arc empty'(T-1,U) = exp(alpha(T-1,U) + empty(T-1,U) - L_tot)."""
    alpha = forward_alpha(px, py)
    beta = backward_beta(px, py)
    T, U1 = px.shape
    L = alpha[-1, -1] + py[-1, -1]
    ypr = np.zeros((T, U1))
    bpr = np.zeros((T, U1))
    if not np.isfinite(L):
        return L, ypr, bpr
    with np.errstate(invalid="ignore"):
        if U1 > 1:
            ypr[:, :-1] = np.exp(alpha[:, :-1] + px[:, :-1] + beta[:, 1:] - L)
        if T > 1:
            bpr[:-1, :] = np.exp(alpha[:-1, :] + py[:-1, :] + beta[1:, :] - L)
        bpr[-1, -1] = np.exp(alpha[-1, -1] + py[-1, -1] - L)
    ypr = np.nan_to_num(ypr, nan=0.0)
    bpr = np.nan_to_num(bpr, nan=0.0)
    return L, ypr, bpr


def simple_grads(am, lm, y, Lnorm, ypr, bpr, grad_scale=1.0):
    """Gradients of -L_tot of the trivial joiner w.r.t. L_enc (am) and L_dec (lm).

    Chain rule through Eq. 5-6 and Eq. 1-2: with
    P(t,u,v) = exp(am[t,v] + lm[u,v] - L_norm(t,u)),
      d(-L)/d am[t,v] = sum_u (y'+empty')(t,u) P(t,u,v) - sum_u y'(t,u)[v=y_{u+1}] - [v=0] sum_u empty'(t,u)
      d(-L)/d lm[u,v] = sum_t (y'+empty')(t,u) P(t,u,v) - [v=y_{u+1}] sum_t y'(t,u) - [v=0] sum_t empty'(t,u)
    P is formed one frame at a time (never the full (T,U+1,V) array at once)."""
    am = np.asarray(am, np.float64)
    lm = np.asarray(lm, np.float64)
    T, V = am.shape
    U = len(y)
    occ = ypr + bpr
    am_grad = np.zeros((T, V))
    lm_grad = np.zeros((U + 1, V))
    for t in range(T):
        P = np.exp(am[t][None, :] + lm - Lnorm[t][:, None])  # (U+1, V)
        w = occ[t][:, None] * P
        am_grad[t] = w.sum(axis=0)
        lm_grad += w
    for u in range(U):
        am_grad[:, y[u]] -= ypr[:, u]
        lm_grad[u, y[u]] -= ypr[:, u].sum()
    am_grad[:, 0] -= bpr.sum(axis=1)
    lm_grad[:, 0] -= bpr.sum(axis=0)
    return grad_scale * am_grad, grad_scale * lm_grad


def simple_loss(am, lm, y, grad_scale=1.0, with_grads=True):
    """Full trivial-joiner stage for one utterance: returns dict with
    loss = -L_tot, px, py, Lnorm, px_grad = y', py_grad = empty', am_grad, lm_grad."""
    px, py, Lnorm = trivial_lattice(am, lm, y)
    L, ypr, bpr = occupancies(px, py)
    out = dict(loss=-L, px=px, py=py, Lnorm=Lnorm, px_grad=ypr, py_grad=bpr)
    if with_grads:
        out["am_grad"], out["lm_grad"] = simple_grads(am, lm, y, Lnorm, ypr, bpr, grad_scale)
    return out


# ------------------------------------------- smoothed trivial joiner (Sec 3.1.1, Eq. 11-15)
def log_softmax(x, axis=-1):
    """x - logsumexp(x) along ``axis`` (the LogSoftmax of P:331)."""
    x = np.asarray(x, np.float64)
    return x - np.expand_dims(logsumexp(x, axis=axis), axis)


def smoothed_parts(am, lm):
    """The three log-prob tables of the smoothed trivial joiner, returned as callables
    over (t, u, v) index arrays plus the utterance-level pieces:
      L_lm(u,v)      = LogSoftmax_v L_dec(u,v)                                   (Eq. 14)
      L_dec^avg(v)   = log (1/(U+1)) sum_{u=0}^{U} Softmax_v L_dec(u,v)          (Eq. 15; no t, u dependence)
      L_acoustic(t,v)= LogSoftmax_v (L_enc(t,v) + L_dec^avg(v))                  (Eq. 13)
    L_trivial is Eq. 12 (= Eq. 5-6): L_enc(t,v) + L_dec(u,v) - L_normalizer(t,u)."""
    am = np.asarray(am, np.float64)
    lm = np.asarray(lm, np.float64)
    L_lm = log_softmax(lm, axis=1)                               # (U+1, V)
    Lavg = logsumexp(L_lm, axis=0) - math.log(lm.shape[0])       # (V,)
    L_ac = log_softmax(am + Lavg[None, :], axis=1)               # (T, V)
    return L_lm, Lavg, L_ac


def smoothed_lattice(am, lm, y, lm_only_scale, am_only_scale):
    """(px, py) of the smoothed trivial joiner, Eq. 11:
        L_smoothed = (1 - a_lm - a_ac) L_trivial + a_lm L_lm + a_ac L_acoustic,
    with a_lm = lm_only_scale, a_ac = am_only_scale.  Eq. 11 as printed multiplies a_ac by L_lm a
    second time; Eq. 13 defines L_acoustic for exactly this slot, so the third term is read as
    a_ac L_acoustic (D18).  px(t,u) = L_smoothed(t,u,y_{u+1}) (-inf at u=U),
    py(t,u) = L_smoothed(t,u,0)."""
    am = np.asarray(am, np.float64)
    lm = np.asarray(lm, np.float64)
    y = np.asarray(y, np.int64)
    T, U = am.shape[0], len(y)
    a_lm, a_ac = float(lm_only_scale), float(am_only_scale)
    w0 = 1.0 - a_lm - a_ac
    px_t, py_t, Lnorm = trivial_lattice(am, lm, y)
    L_lm, Lavg, L_ac = smoothed_parts(am, lm)
    px = np.full((T, U + 1), NEG_INF)
    if U > 0:
        u = np.arange(U)
        px[:, :U] = w0 * px_t[:, :U] + a_lm * L_lm[u, y][None, :] + a_ac * L_ac[:, y]
    py = w0 * py_t + a_lm * L_lm[:, 0][None, :] + a_ac * L_ac[:, 0][:, None]
    return px, py


def smoothed_loss(am, lm, y, lm_only_scale, am_only_scale, grad_scale=1.0, with_grads=True):
    """Smoothed-joiner stage for one utterance: loss = -L_tot on the Eq. 11 lattice, occupancies
    px_grad = y', py_grad = empty', and gs * d(-L_tot)/d{am, lm}.

    The gradient is plain reverse-mode through the definitions: with dL(t,u,v) = d(-L_tot)/dL(t,u,v)
    = -(y'(t,u) [v = y_{u+1}] + empty'(t,u) [v = 0]), each LogSoftmax z -> z - LSE(z) passes back
    g - softmax(z) sum_v g, and L_dec^avg = log mean_u softmax(L_dec(u)) passes dLavg(v) back as
    sum_v dLavg(v) P(u,v) ([v = v'] - P(u,v')) / ((U+1) avg(v)).  The (T, U+1, V) tensors are formed
    one frame at a time."""
    am = np.asarray(am, np.float64)
    lm = np.asarray(lm, np.float64)
    y = np.asarray(y, np.int64)
    T, V = am.shape
    U = len(y)
    a_lm, a_ac = float(lm_only_scale), float(am_only_scale)
    w0 = 1.0 - a_lm - a_ac
    px, py = smoothed_lattice(am, lm, y, a_lm, a_ac)
    L, ypr, bpr = occupancies(px, py)
    out = dict(loss=-L, px=px, py=py, px_grad=ypr, py_grad=bpr)
    if not with_grads:
        return out
    L_lm, Lavg, L_ac = smoothed_parts(am, lm)
    Lnorm = trivial_normalizer(am, lm)
    P_lm = np.exp(L_lm)                                          # (U+1, V)
    P_ac = np.exp(L_ac)                                          # (T, V)
    avg = np.exp(Lavg)                                           # (V,)
    am_grad = np.zeros((T, V))
    lm_grad = np.zeros((U + 1, V))
    dLavg = np.zeros(V)
    for t in range(T):
        dL = np.zeros((U + 1, V))                                # d(-L)/dL(t, u, v)
        if U > 0:
            dL[np.arange(U), y] -= ypr[t, :U]
        dL[:, 0] -= bpr[t]
        sdl = dL.sum(axis=1)                                     # (U+1,)
        # trivial term: LogSoftmax_v(am[t] + lm[u]) per u
        P_tr = np.exp(am[t][None, :] + lm - Lnorm[t][:, None])   # (U+1, V)
        g_tr = w0 * (dL - P_tr * sdl[:, None])
        am_grad[t] += g_tr.sum(axis=0)
        lm_grad += g_tr
        # LM-only term: LogSoftmax_v(lm[u]) per u
        lm_grad += a_lm * (dL - P_lm * sdl[:, None])
        # acoustic term: LogSoftmax_v(am[t] + Lavg), summed over u first
        g_ac = a_ac * (dL.sum(axis=0) - P_ac[t] * sdl.sum())
        am_grad[t] += g_ac
        dLavg += g_ac
    # through L_dec^avg(v) = log mean_u softmax(lm[u])(v)
    q = P_lm * (dLavg / ((U + 1) * avg))[None, :]                # (U+1, V)
    lm_grad += q - P_lm * q.sum(axis=1)[:, None]
    out["am_grad"] = grad_scale * am_grad
    out["lm_grad"] = grad_scale * lm_grad
    return out


# --------------------------------------------------------------- pruning bounds
def umax(U, S):
    """Largest legal bound U-S+1, floored at 0 when S > U+1 (D10)."""
    return max(0, U - S + 1)


def feasible(T, U, S):
    """A band-respecting path exists iff U <= T(S-1)  (Eq. 9-10 with p_0=0, p_{T-1}=Umax)."""
    return U <= T * (S - 1)


def bound_scores(px_grad_row, py_grad_row, S):
    """Candidate values of Eq. 8 for one frame (Eq. 7-8):
        v(p) = -y'(t,p-1) + sum_{u=p}^{p+S-1} empty'(t,u),   p = 0..max(0,U-S+1),
    with y'(t,-1) = 0.  fp32 inputs promoted to fp64, summed u ascending, then the
    subtraction (fixed order, D5).  Window terms with u > U are absent (D10)."""
    ypr = np.asarray(px_grad_row)
    bpr = np.asarray(py_grad_row)
    U1 = bpr.shape[0]
    P = umax(U1 - 1, S) + 1
    vals = np.empty(P, np.float64)
    for p in range(P):
        acc = 0.0
        for u in range(p, min(p + S, U1)):
            acc = acc + float(np.float64(bpr[u]))
        if p > 0:
            acc = acc - float(np.float64(ypr[p - 1]))
        vals[p] = acc
    return vals


def raw_bounds(px_grad, py_grad, S):
    """Locally optimal bounds, Eq. 8:
        p_t = argmax_{p=0..U-S+1} ( -y'(t,p-1) + sum_{u=p}^{p+S-1} empty'(t,u) ),
    ties to the smallest p (numpy argmax returns the first maximum)."""
    T = np.asarray(py_grad).shape[0]
    raw = np.zeros(T, np.int64)
    for t in range(T):
        raw[t] = int(np.argmax(bound_scores(px_grad[t], py_grad[t], S)))
    return raw


def adjust_bounds(raw, T, U, S):
    """Consistency adjustment (Eq. 9-10; algorithm = DESIGN.md D3 'ADJ-scan').

    1. clamp q_t into [l_t, h_t], l_t = max(0, Umax-(T-1-t)(S-1)), h_t = min(Umax, t(S-1));
    2. q_t <- max_{t'<=t} q_t'           (Eq. 9, monotone)
    3. p_t = max_{t'>=t} (q_t' - (t'-t)(S-1))   (Eq. 10, steps < S)
    The result is the least feasible sequence >= the monotone hull of the
    clamped raw bounds ("changing them as little as possible").
    Infeasible (U > T(S-1)): returns zeros (caller flags status bit0)."""
    Um = umax(U, S)
    if not feasible(T, U, S):
        return np.zeros(T, np.int64)
    raw = np.asarray(raw, np.int64)
    t = np.arange(T, dtype=np.int64)
    lo = np.maximum(0, Um - (T - 1 - t) * (S - 1))
    hi = np.minimum(Um, t * (S - 1))
    q = np.clip(raw, lo, hi)
    q = np.maximum.accumulate(q)
    g = q - t * (S - 1)
    suf = np.maximum.accumulate(g[::-1])[::-1]
    return (suf + t * (S - 1)).astype(np.int64)


# ------------------------------------------------------------ pruned joiner / loss
def bf16_round(x):
    """Round fp64 values to the nearest bf16 (round-to-nearest-even), as fp64.
    Matched mode of DESIGN.md D6 (the GPU stores h in bf16)."""
    f = np.asarray(x, np.float64).astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def band_mask(ranges, U, S):
    """Boolean (T, U+1): node (t,u) kept iff p_t <= u < p_t + S."""
    T = len(ranges)
    u = np.arange(U + 1)[None, :]
    p = np.asarray(ranges)[:, None]
    return (u >= p) & (u < p + S)


def pruned_lattice(enc, dec, W, b, y, ranges, S, matched=True):
    """Full (non-linear) joiner evaluated only inside the band.

    Joiner form (BASELINE.json north_star; D13): z = W_out tanh(enc[t] + dec[u]) + b,
    L(t,u,.) = log_softmax(z).  Returns px, py of shape (T,U+1) with -inf outside
    the band, plus the per-node h, z and log-softmax for the gradient.  In matched
    mode h is rounded to bf16 (D6)."""
    enc = np.asarray(enc, np.float64)
    dec = np.asarray(dec, np.float64)
    W = np.asarray(W, np.float64)
    b = np.asarray(b, np.float64)
    T, U = enc.shape[0], len(y)
    mask = band_mask(ranges, U, S)
    px = np.full((T, U + 1), NEG_INF)
    py = np.full((T, U + 1), NEG_INF)
    tt, uu = np.nonzero(mask)
    h = np.tanh(enc[tt] + dec[uu])
    if matched:
        h = bf16_round(h)
    z = h @ W.T + b[None, :]
    lse = logsumexp(z, axis=1)
    logp = z - lse[:, None]
    py[tt, uu] = logp[:, 0]
    lab = uu < U
    px[tt[lab], uu[lab]] = logp[lab, np.asarray(y, np.int64)[uu[lab]]]
    return dict(px=px, py=py, tt=tt, uu=uu, h=h, z=z, logp=logp)


def pruned_loss(enc, dec, W, b, y, ranges, S, grad_scale=1.0, matched=True, with_grads=True):
    """Pruned recursion and its gradients (out-of-band arcs -inf, then Eq. 3).

    dz(t,u,v) = gs * ((g_b + g_l) softmax(z)(v) - g_b [v=0] - g_l [v=y_{u+1}]) with
    g_b = empty'_p(t,u), g_l = y'_p(t,u) (function merging);
    dW = sum dz h^T, db = sum dz, dh = W^T dz, dpre = dh (1 - h^2),
    d_enc[t] += dpre, d_dec[u] += dpre."""
    J = np.asarray(enc).shape[1]
    T, U = np.asarray(enc).shape[0], len(y)
    V = np.asarray(W).shape[0]
    lat = pruned_lattice(enc, dec, W, b, y, ranges, S, matched)
    L, ypr, bpr = occupancies(lat["px"], lat["py"])
    out = dict(loss=-L, px=lat["px"], py=lat["py"], g_l=ypr, g_b=bpr, lattice=lat)
    if not with_grads:
        return out
    tt, uu, h, logp = lat["tt"], lat["uu"], lat["h"], lat["logp"]
    gb = bpr[tt, uu]
    gl = ypr[tt, uu]
    sm = np.exp(logp)
    dz = (gb + gl)[:, None] * sm
    dz[:, 0] -= gb
    lab = uu < U
    yy = np.asarray(y, np.int64)
    dz[np.nonzero(lab)[0], yy[uu[lab]]] -= gl[lab]
    dz *= grad_scale
    W64 = np.asarray(W, np.float64)
    dW = dz.T @ h
    db = dz.sum(axis=0)
    dh = dz @ W64
    dpre = dh * (1.0 - h * h)
    d_enc = np.zeros((T, J))
    d_dec = np.zeros((U + 1, J))
    np.add.at(d_enc, tt, dpre)
    np.add.at(d_dec, uu, dpre)
    out.update(dz=dz, d_w=dW, d_b=db, d_enc=d_enc, d_dec=d_dec)
    return out


# ------------------------------------------------------------------ brute force
def brute_force_paths(T, U):
    """All monotone lattice paths (0,0)->(T-1,U): each is a choice of which of the
    T-1+U moves are vertical; yields lists of (t,u,kind) arcs incl. terminal blank."""
    from itertools import combinations
    moves = T - 1 + U
    for ups in combinations(range(moves), U):
        ups = set(ups)
        t = u = 0
        arcs = []
        for i in range(moves):
            if i in ups:
                arcs.append((t, u, "y"))
                u += 1
            else:
                arcs.append((t, u, "b"))
                t += 1
        arcs.append((T - 1, U, "b"))
        yield arcs


def brute_force_logprob(px, py, mask=None):
    """log sum over all paths of exp(sum of arc log-probs); with ``mask`` only paths
    whose visited nodes are all kept count (pruned lattice)."""
    T, U1 = px.shape
    lps = []
    for arcs in brute_force_paths(T, U1 - 1):
        if mask is not None and not all(mask[t, u] for (t, u, _) in arcs):
            continue
        lps.append(sum(px[t, u] if k == "y" else py[t, u] for (t, u, k) in arcs))
    if not lps:
        return NEG_INF
    return float(logsumexp(np.array(lps)))


# ------------------------------------------------------------------- full step
def full_step(batch, simple_scale=0.5, pruned_scale=1.0, matched=True, ranges=None,
              with_grads=True):
    """Whole hot path for a padded ``synth.Batch``.

    Per utterance: trivial joiner -> recursion/occupancies -> Eq. 8 -> adjustment
    -> pruned joiner -> pruned recursion -> gradients.  ``ranges`` (N, T-hat)
    overrides the bounds (stage-wise parity uses the oracle's own bounds).
    Returns padded arrays (zeros at padding) mirroring the C-ABI outputs."""
    N, Tm, Um, V, J, S = batch.N, batch.T, batch.U, batch.V, batch.J, batch.S
    res = dict(loss_simple=np.zeros(N), loss_pruned=np.zeros(N),
               px_grad=np.zeros((N, Tm, Um + 1)), py_grad=np.zeros((N, Tm, Um + 1)),
               am_grad=np.zeros((N, Tm, V)), lm_grad=np.zeros((N, Um + 1, V)),
               ranges=np.zeros((N, Tm), np.int64), d_enc=np.zeros((N, Tm, J)),
               d_dec=np.zeros((N, Um + 1, J)), d_w=np.zeros((V, J)), d_b=np.zeros(V),
               status=np.zeros(N, np.int64))
    for n in range(N):
        d = batch.utterance(n)
        T, U = d["T"], d["U"]
        s = simple_loss(d["am"], d["lm"], d["y"], simple_scale, with_grads)
        res["loss_simple"][n] = s["loss"]
        pxg = s["px_grad"].astype(np.float32)
        pyg = s["py_grad"].astype(np.float32)
        res["px_grad"][n, :T, :U + 1] = pxg
        res["py_grad"][n, :T, :U + 1] = pyg
        if with_grads:
            res["am_grad"][n, :T] = s["am_grad"]
            res["lm_grad"][n, :U + 1] = s["lm_grad"]
        if ranges is None:
            p = adjust_bounds(raw_bounds(pxg, pyg, S), T, U, S)
        else:
            p = np.asarray(ranges[n, :T], np.int64)
        if not feasible(T, U, S):
            res["status"][n] |= 1
            res["loss_pruned"][n] = np.inf
            continue
        res["ranges"][n, :T] = p
        res["ranges"][n, T:] = umax(U, S)
        pr = pruned_loss(d["enc"], d["dec"], d["W"], d["b"], d["y"], p, S, pruned_scale,
                         matched, with_grads)
        res["loss_pruned"][n] = pr["loss"]
        if with_grads:
            res["d_enc"][n, :T] = pr["d_enc"]
            res["d_dec"][n, :U + 1] = pr["d_dec"]
            res["d_w"] += pr["d_w"]
            res["d_b"] += pr["d_b"]
    res["loss"] = simple_scale * res["loss_simple"].sum() + pruned_scale * np.where(
        np.isfinite(res["loss_pruned"]), res["loss_pruned"], 0.0).sum()
    return res
