// workspace.h — carving of the caller-provided device workspace (host + device).
// The simple-loss region and the pruned-loss region are disjoint, so one
// workspace can serve rnnt_simple_loss and rnnt_pruned_loss concurrently.
#pragma once
#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime.h>
#include <stdlib.h>
#include <algorithm>

namespace rnnt {

struct Dims {
  int N, T, U, V, J, S;
  int U1() const { return U + 1; }
  // Wavefront geometry of the simple lattice (lattice.cu): W strips (one warp each, on distinct
  // SM sub-partitions) of 32 lanes x R columns; the skewed row pitch is LU = 32 R W, so every lane
  // owns whole columns of every row (no partial lanes, no masks).  0 = unsupported (U+1 > 1024).
  int lat_R() const {
    const int need = (U + 1 + 31) / 32;   // columns per lane if one warp held the row
    if (need <= 2) return need;
    if (need <= 8) return 2;
    if (need <= 16) return 4;
    if (need <= 32) return 8;
    return 0;
  }
  int lat_W() const {
    const int r = lat_R();
    return r ? ((U + 1 + 32 * r - 1) / (32 * r)) : 0;
  }
  int LU() const { return 32 * lat_R() * lat_W(); }
  int K() const { return T + U; }                       // number of anti-diagonals
  long long rows() const { return (long long)N * T * S; }
  int VP64() const { return (V + 63) / 64 * 64; }       // bf16 pitch of the E operands (K-major boxes of 64)
  int UP() const { return (U + 1 + 63) / 64 * 64; }      // bf16 pitch of G~ (t-major, K-major boxes of 64)
  int ntb() const { return (T + 31) / 32; }              // 32-frame blocks of the occupancy column partials
  int ntile() const { return (V + 127) / 128; }        // kVT-wide max-shift tiles
  int VP() const { return (V + 127) / 128 * 128; }      // padded row pitch of P~ (elements)
};

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// d_dec partials of the band reduction (pruned.cu band_chunk_kernel): chunks of kBandCH frames; per
// utterance U + 1 + S ceil(T / kBandCH) rows (chunk c's partial of u at row u + c S).
constexpr int kBandCH = 16;
__host__ __device__ inline long long band_part_rows(int T, int U, int S) {
  return (long long)U + 1 + (long long)S * ((T + kBandCH - 1) / kBandCH);
}
// 512-B column segments (32 float4) of a J-wide row: the band reduction's unit of work per warp
__host__ __device__ inline int band_nseg(int J) { return (J / 4 + 31) / 32; }

// Interpolation weights of the smoothed trivial joiner (Eq. 11): a_lm = lm_only_scale, a_ac =
// am_only_scale; both 0 is the plain trivial joiner.
struct Smooth {
  float a_lm = 0.f, a_ac = 0.f;
  __host__ __device__ bool on() const { return a_lm != 0.f || a_ac != 0.f; }
  __host__ __device__ float w0() const { return 1.f - a_lm - a_ac; }
};

struct SimpleWS {
  float* m_am;    // (N,T)     row max of am
  float* m_lm;    // (N,U+1)   row max of lm
  float2* pxy;    // (N,K+1,LU) skewed {y(t,u), empty(t,u)} * log2e   (k = t+u)
  float* rS;      // (N,K+1,LU) skewed 1/S(t,u) = 1/sum_v exp(am-m_am+lm-m_lm) (valid cells only)
  float* alpha;   // (N,K+1,LU) skewed alpha-hat = alpha*log2e - A_k (fp32, rebased)
  float* beta;    // (N,K+1,LU) skewed beta-hat  = beta*log2e - B_k
  float* Ash;     // (N,K+1,W)  A_k per diagonal and strip (integer-valued)
  float* Bsh;     // (N,K+1,W)  B_k per diagonal and strip
  double* Ltot;   // (N)        L_tot (natural log)
  uint16_t* Eam_hi;  // (N,T,VP64) bf16 hi of e^{am - m_am} (zero rows t >= T_n, zero cols v >= V)
  uint16_t* Eam_lo;  // (N,T,VP64) bf16 lo = bf16(e - hi)
  uint16_t* Elm_hi;  // (N,U+1,VP64)
  uint16_t* Elm_lo;
  uint16_t* Gt_hi;   // (N,T,UP)   bf16 hi/lo of G~ = (y'+empty')/S(t,u) (t-major, zero padded)
  uint16_t* Gt_lo;
  float* amy;        // (N,T,UP)   am[t, y_{u+1}] (gathered by exp_split for the normaliser epilogue)
  float* rowb;       // (N,T)      sum_u empty'(t,u)
  float* colpy;      // (N,ntb,U+1) per-32-frame-block partial sums of y'(t,u) over t
  float* colpb;      // (N,ntb,U+1) ... of empty'(t,u)
  float* rowy;       // (N,T)      sum_u y'(t,u)
  // smoothed trivial joiner (Eq. 11-15), used only when a scale is nonzero
  float* lse_lm;     // (N,U+1)    log sum_v exp lm[u,v]
  float* Lavg;       // (N,VP64)   L_dec^avg(v) = log mean_u softmax(lm[u])(v)   (Eq. 15)
  float* lse_ac;     // (N,T)      log sum_v exp(am[t,v] + L_dec^avg(v))        (Eq. 13 normaliser)
  float* gq;         // (N,VP64)   a_ac g_avg(v) / ((U+1) avg(v)): the L_dec^avg backward factor
  float* Qu;         // (N,U+1)    sum_v softmax(lm[u])(v) gq(v)
};

struct PrunedWS {
  int32_t* rowinfo;  // (R) label y_{u+1} (V if u==U_n), -1 for masked/padded rows
  int2* urange;      // (N,U+1) frames [lo,hi) whose band covers token position u
  float* bias;       // (VP) fp32 copy of b_out, zero padded
  float* bmax;       // (ntile) max of the bias over each 128-column tile
  uint8_t* tlive;    // (ceil(R/128)) 128-row tile holds a live band row
  int* tcounter;     // tile scheduler counter of the persistent joiner forward
  float* gsp;        // (tcounter + 2) the forward's grad_scale: the fp16 dpre rows hold dpre / gs
  int* tscale;       // 0: every row's P~ tiles share one offset m_ref (the joiner backward runs as plain
                     //    GEMMs on P~ with the picks folded in, pruned_combine); else per-tile offsets
                     //    (the backward rescales P~ per (row, tile) in shared memory)
  uint16_t* Pt;      // (R,VP) bf16 exp(z - m_tile), pitch VP
  float* mt;         // (R,ntile) tile maxima of z
  float* lse;        // (R) log-sum-exp of z
  float* px2;        // (R) y_p * log2e (band arcs)
  float* py2;        // (R) empty_p * log2e
  float* ap;         // (R) pruned alpha-hat (log2, rebased per frame)
  float* bp;         // (R) pruned beta-hat
  double* Af;        // (N,T) pruned alpha shift per frame (log2): alpha(t,s) log2e = ap + Af[t]
  double* Bf;        // (N,T) pruned beta shift per frame
  double* Lp;        // (N) L_pruned
  float* gb;         // (R) empty'_p
  float* gl;         // (R) y'_p
  float4* gpk;       // (ntile,R) per (V tile, row): {gs (gb+gl) exp(m_tile - lse), gs gb, gs gl, label bits}
  int* dhlive;       // (R/128 + 1) ids of the live 128-row joiner_dh tiles, then their count
  float* dpre;       // (R,J) dpre = dh (1 - h^2) of every band row (live rows only are written): the pruned
                     //    path stores it as fp16 dpre / gs (the first half of the buffer), the full loss fp32
  bool plain;        // the plain joiner backward may run (tscale == 0 honoured; false: the full loss)
  uint16_t* Hs;      // (R,J) bf16 sc_r h_r, the plain d_w GEMM's B operand for large V (null: formed in smem)
  float* bpart;      // (N, band_part_rows, J) d_dec partials of the band reduction
  float* dWp;        // (splits,V,J) split-K partials of d_w
  float* dbp;        // (splits,V)   split-K partials of d_b
  int splits;
};

// K11 variant: "wide" CTAs (one per SM) hold two V tiles (256 v x 256 j, 512 TMEM columns) so each
// h k-block feeds two MMAs; used for large V (L2 -> SM bound), RNNT_DW_WIDE=0/1 forces it off/on.
inline bool dw_wide(const Dims& d) {
  static const int force = env_int("RNNT_DW_WIDE", -1);
  if (force >= 0) return force == 1;
  return true;   // measured: c2 65.5 vs 68.6 us, c3 339 vs 593, c4 2113 vs 3234 (the 128-v variant with 2D boxes)
}

// Plain-mode d_w operand Hs = bf16(sc h): precomputed by scale_rows_kernel for large V (the d_w mainloop is
// long and shared-memory bound), else formed in the d_w kernel's shared memory (joiner_bwd.cu).
inline bool hs_precomputed(const Dims& d) {
  static const int force = env_int("RNNT_HS_PRE", -1);   // A/B: 1 always precompute, 0 never
  return force >= 0 ? force == 1 : d.V >= 2048;
}

// Split-K factor of the d_w GEMM (K11): about two CTAs per SM over the (V/128) x (J/256)
// output tiles, at least 4 K-blocks of 64 rows per split.
inline int dw_splits(const Dims& d) {
  const long long nkb = (d.rows() + 63) / 64;
  if (dw_wide(d)) {
    // one CTA per SM: the smallest split count whose grid fills whole waves to >= 90 %
    const long long tiles = (long long)((d.ntile() + 1) / 2) * ((d.J + 255) / 256);
    const long long cap = std::max(1LL, std::min(64LL, nkb / 4));
    long long best = 1;
    double beff = 0.0;
    for (long long s = 1; s <= cap; ++s) {
      const long long c = tiles * s;
      const double eff = (double)c / (148.0 * (double)((c + 147) / 148));
      if (c >= 148 && eff >= 0.9) return (int)s;
      if (eff > beff + 1e-9) { beff = eff; best = s; }
    }
    return (int)best;
  }
  const long long tiles = (long long)((d.V + 127) / 128) * ((d.J + 255) / 256);
  long long s = (2 * 148 + tiles - 1) / tiles;
  const long long cap = nkb / 4 > 1 ? nkb / 4 : 1;
  if (s > cap) s = cap;
  if (s > 64) s = 64;
  if (s < 1) s = 1;
  return (int)s;
}

// Returns total bytes; if base != nullptr fills the structs.
inline size_t carve(const Dims& d, void* base, SimpleWS* sw, PrunedWS* pw, bool with_plain = true) {
  size_t off = 0;
  char* b = static_cast<char*>(base);
  auto take = [&](size_t bytes) -> void* {
    void* p = b ? (void*)(b + off) : nullptr;
    off += align_up(bytes);
    return p;
  };
  const size_t N = d.N, T = d.T, U1 = d.U1(), LU = d.LU(), K1 = d.K() + 1;
  const size_t R = (size_t)d.rows(), V = d.V, J = d.J, NT = d.ntile(), VP = d.VP();
  SimpleWS s;
  s.m_am = (float*)take(N * T * 4);
  s.m_lm = (float*)take(N * U1 * 4);
  s.pxy = (float2*)take(N * K1 * LU * 8);
  s.rS = (float*)take(N * K1 * LU * 4);
  s.alpha = (float*)take(N * K1 * LU * 4);
  s.beta = (float*)take(N * K1 * LU * 4);
  s.Ash = (float*)take(N * K1 * (size_t)d.lat_W() * 4);
  s.Bsh = (float*)take(N * K1 * (size_t)d.lat_W() * 4);
  s.Ltot = (double*)take(N * 8);
  const size_t VP64 = d.VP64(), UP = d.UP(), NTB = d.ntb();
  s.Eam_hi = (uint16_t*)take(N * T * VP64 * 2);
  s.Eam_lo = (uint16_t*)take(N * T * VP64 * 2);
  s.Elm_hi = (uint16_t*)take(N * U1 * VP64 * 2);
  s.Elm_lo = (uint16_t*)take(N * U1 * VP64 * 2);
  s.Gt_hi = (uint16_t*)take(N * T * UP * 2);
  s.Gt_lo = (uint16_t*)take(N * T * UP * 2);
  s.amy = (float*)take(N * T * UP * 4);
  s.rowb = (float*)take(N * T * 4);
  s.colpy = (float*)take(N * NTB * U1 * 4);
  s.colpb = (float*)take(N * NTB * U1 * 4);
  s.rowy = (float*)take(N * T * 4);
  s.lse_lm = (float*)take(N * U1 * 4);
  s.Lavg = (float*)take(N * VP64 * 4);
  s.lse_ac = (float*)take(N * T * 4);
  s.gq = (float*)take(N * VP64 * 4);
  s.Qu = (float*)take(N * U1 * 4);
  PrunedWS p;
  p.splits = dw_splits(d);
  p.rowinfo = (int32_t*)take(R * 4);
  p.urange = (int2*)take(N * U1 * 8);
  p.bias = (float*)take(VP * 4);
  p.bmax = (float*)take(NT * 4);
  p.tlive = (uint8_t*)take((R + 127) / 128);
  p.tcounter = (int*)take(16);
  p.tscale = b ? p.tcounter + 1 : nullptr;
  p.gsp = b ? reinterpret_cast<float*>(p.tcounter + 2) : nullptr;
  p.Pt = (uint16_t*)take(R * VP * 2);
  p.mt = (float*)take(R * NT * 4);
  p.lse = (float*)take(R * 4);
  p.px2 = (float*)take(R * 4);
  p.py2 = (float*)take(R * 4);
  p.ap = (float*)take(R * 4);
  p.bp = (float*)take(R * 4);
  p.Af = (double*)take(N * T * 8);
  p.Bf = (double*)take(N * T * 8);
  p.Lp = (double*)take(N * 8);
  p.gb = (float*)take(R * 4);
  p.gl = (float*)take(R * 4);
  p.gpk = (float4*)take(R * NT * 16);
  // joiner_dh: ids of the live 128-row tiles (+ count), and dpre = dh (1 - h^2) per band row, which
  // band_reduce_kernel turns into d_enc / d_dec
  p.dhlive = (int*)take(((R + 127) / 128 + 1) * 4);
  p.dpre = (float*)take(R * J * 4);
  p.plain = with_plain;
  p.Hs = with_plain && hs_precomputed(d) ? (uint16_t*)take(R * J * 2) : nullptr;
  p.bpart = (float*)take((size_t)N * band_part_rows(d.T, d.U, d.S) * J * 4);
  p.dWp = (float*)take((size_t)p.splits * V * J * 4);
  p.dbp = (float*)take((size_t)p.splits * V * 4);
  if (sw) *sw = s;
  if (pw) *pw = p;
  return off + 256;  // slack for base alignment
}

// The full (unpruned) lattice of SURVEY 8(f) f4: the pruned workspace of dims with S = U+1 (every
// (t,u) is a band row), then all-zero bounds and the dpre rows of the generic joiner_dh mode.
struct FullWS {
  int32_t* ranges0;  // (N,T) all zero: the band [0, U] of every frame
  float* dpre;       // (R,J) dpre = dh (1 - h^2) for every (t,u) row
  uint16_t* h;       // (R,J) bf16 joiner input of every (t,u)
};
inline size_t carve_full(const Dims& df, void* base, SimpleWS* sw, PrunedWS* pw, FullWS* fw) {
  const size_t inner = carve(df, base, sw, pw, false);
  size_t off = align_up(inner);
  char* b = static_cast<char*>(base);
  auto take = [&](size_t bytes) -> void* {
    void* q = b ? (void*)(b + off) : nullptr;
    off += align_up(bytes);
    return q;
  };
  FullWS f;
  f.ranges0 = (int32_t*)take((size_t)df.N * df.T * 4);
  f.dpre = pw ? pw->dpre : nullptr;        // the pruned region's dpre rows (R = N T (U+1) here)
  f.h = (uint16_t*)take((size_t)df.rows() * df.J * 2);
  if (fw) *fw = f;
  return off + 256;
}

}  // namespace rnnt
