// simple_tc.cu — the contractions of the simple (trivial-joiner) loss on tcgen05.
//
//   K1 exp_split_kernel   m(row) = max_v x[row,v] (the offsets of Eq. 6, "after first applying
//                         offsets") and E = e^{x - m} split into bf16 hi + lo
//                         (E = hi + lo to 2^-17 relative; D7 "bf16x3")
//   K2 norm (gemm3)       S(t,u) = sum_v E_am[t,v] E_lm[u,v]        (Eq. 6 as a contraction, never
//                         materialising (T,U+1,V)); epilogue: L_norm = log S + m_am + m_lm and the
//                         skewed lattice arcs px2 = y(t,u) log2e, py2 = empty(t,u) log2e (Eq. 1-2,
//                         Eq. 5), 1/S — written diagonal-major through a per-warp smem transpose
//   K5a am_grad (gemm3)   am_grad[t,v] = gs (E_am[t,v] sum_u G~[t,u] E_lm[u,v] - picks)
//   K5b lm_grad (gemm3)   lm_grad[u,v] = gs (E_lm[u,v] sum_t G~[t,u] E_am[t,v] - picks)
//                         with G~ = (y' + empty') / S and the picks sum_u y'[v = y_{u+1}] +
//                         [v = 0] sum_u empty' (chain rule through Eq. 5-6)
// gemm3: one 128 x BN output tile per CTA, fp32 accumulator in TMEM, bf16x3 products
// hi*hi + hi*lo + lo*hi issued as three tcgen05.mma.kind::f16 per K slice.  Operands come from
// per-utterance 3-D TMA tensor maps (a box never spills into the next utterance: OOB reads 0).
// Warp 4: TMEM allocator, lane 0 TMA producer, lane 1 MMA issuer; warps 0-3: prologue (per-tile
// tables in smem, overlapping the mainloop) and epilogue (TMEM lane = tile row = thread).
#include <algorithm>

#include "common.cuh"
#include "launch.h"
#include "tc.cuh"
#include "tmap.h"
#include "workspace.h"

namespace rnnt {

// ------------------------------------------------------------------ K1
// One warp per row of am (which = 0, rows t of T) or lm (which = 1, rows u of U+1).  am rows also
// gather amy[t,u] = am[t, y_{u+1}] (the label logit the normaliser epilogue needs, read here while
// the row is in L1).
__device__ __forceinline__ void exp_split_rows(const float* __restrict__ x, const int64_t* __restrict__ sym,
                                               const int64_t* __restrict__ bnd, int N, int rows_per_n, int U, int V,
                                               int VP, int which, float* __restrict__ m, uint16_t* __restrict__ hi,
                                               uint16_t* __restrict__ lo, float* __restrict__ amy, int UPa,
                                               float* __restrict__ lse, int blk) {
  const long long row = (long long)blk * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= (long long)N * rows_per_n) return;
  const int n = (int)(row / rows_per_n), r = (int)(row % rows_per_n);
  const int Un = utt_U(bnd, n);
  const int lim = which == 0 ? utt_T(bnd, n) : Un + 1;
  uint32_t* H = reinterpret_cast<uint32_t*>(hi + row * (long long)VP);
  uint32_t* L = reinterpret_cast<uint32_t*>(lo + row * (long long)VP);
  if (r >= lim) {   // padded row: zero operand, never read otherwise
    for (int v2 = lane; v2 < VP / 2; v2 += 32) { H[v2] = 0u; L[v2] = 0u; }
    if (lane == 0) m[row] = 0.f;
    if (lse && lane == 0) lse[row] = 0.f;
    return;
  }
  const float* p = x + row * (long long)V;
  float mx = neg_inf_f();
  float esum = 0.f;
  if ((V & 3) == 0) {
    // float4 rows (V % 4 == 0: every row starts 16-B aligned), four loads in flight per lane in both
    // passes (the second re-reads the row from L1/L2); same arithmetic as the scalar path below
    const float4* p4 = reinterpret_cast<const float4*>(p);
    const int V4 = V >> 2, VP4 = VP >> 2;
    for (int j0 = lane; j0 < V4; j0 += 128) {
      float4 t[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = j0 + 32 * k;
        t[k] = j < V4 ? __ldg(p4 + j) : make_float4(neg_inf_f(), neg_inf_f(), neg_inf_f(), neg_inf_f());
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) mx = fmaxf(mx, fmaxf(fmaxf(t[k].x, t[k].y), fmaxf(t[k].z, t[k].w)));
    }
    mx = warp_max(mx);
    if (lane == 0) m[row] = mx;
    uint2* H2 = reinterpret_cast<uint2*>(H);
    uint2* L2 = reinterpret_cast<uint2*>(L);
    for (int j0 = lane; j0 < VP4; j0 += 128) {
      float4 t[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = j0 + 32 * k;
        t[k] = j < V4 ? __ldg(p4 + j) : make_float4(neg_inf_f(), neg_inf_f(), neg_inf_f(), neg_inf_f());
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = j0 + 32 * k;
        if (j < VP4) {
          const float e0 = __expf(t[k].x - mx), e1 = __expf(t[k].y - mx);
          const float e2 = __expf(t[k].z - mx), e3 = __expf(t[k].w - mx);
          esum += (e0 + e1) + (e2 + e3);
          const __nv_bfloat162 h01 = __floats2bfloat162_rn(e0, e1), h23 = __floats2bfloat162_rn(e2, e3);
          const __nv_bfloat162 l01 = __floats2bfloat162_rn(e0 - __low2float(h01), e1 - __high2float(h01));
          const __nv_bfloat162 l23 = __floats2bfloat162_rn(e2 - __low2float(h23), e3 - __high2float(h23));
          H2[j] = make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
          L2[j] = make_uint2(*reinterpret_cast<const uint32_t*>(&l01), *reinterpret_cast<const uint32_t*>(&l23));
        }
      }
    }
  } else {
    for (int v = lane; v < V; v += 32) mx = fmaxf(mx, p[v]);
    mx = warp_max(mx);
    if (lane == 0) m[row] = mx;
    for (int v2 = lane; v2 < VP / 2; v2 += 32) {
      const int v = 2 * v2;
      const float e0 = v < V ? __expf(p[v] - mx) : 0.f;
      const float e1 = v + 1 < V ? __expf(p[v + 1] - mx) : 0.f;
      esum += e0 + e1;
      const __nv_bfloat162 h = __floats2bfloat162_rn(e0, e1);
      const __nv_bfloat162 l = __floats2bfloat162_rn(e0 - __low2float(h), e1 - __high2float(h));
      H[v2] = *reinterpret_cast<const uint32_t*>(&h);
      L[v2] = *reinterpret_cast<const uint32_t*>(&l);
    }
  }
  if (lse) {   // lm rows: log sum_v exp lm[u,v] (the LM-only log-softmax of Eq. 14)
    esum = warp_sum(esum);
    if (lane == 0) lse[row] = mx + __logf(esum);
  }
  if (which == 0) {
    float* ay = amy + ((size_t)n * rows_per_n + r) * UPa;
    for (int u0 = lane; u0 <= Un; u0 += 128) {     // 4 labels, then 4 gathers, in flight per lane
      long long y[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int u = u0 + 32 * k;
        y[k] = u < Un ? sym[(size_t)n * U + u] : 0;
        y[k] = y[k] < 0 ? 0 : (y[k] >= V ? V - 1 : y[k]);   // address safety; bad symbols flagged in status
      }
      float val[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) val[k] = u0 + 32 * k < Un ? p[y[k]] : 0.f;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (u0 + 32 * k <= Un) ay[u0 + 32 * k] = val[k];
    }
  }
}

// Large V (V % 4 == 0, 2048 < V <= 4 256 PER): one 256-thread block per row, the row held in registers
// (PER float4 per thread) between the max and the exp pass -- the warp-per-row form re-reads every row
// for its second pass, which at V = 8000 (32 KB rows, 8 rows per block) misses L2 (c4: 0.54 of HBM).
// Same per-element arithmetic; the row sums for lse_lm are reduced in a different order.
template <int PER>
__device__ __forceinline__ void exp_split_row_block(const float* __restrict__ x, const int64_t* __restrict__ sym,
                                                    const int64_t* __restrict__ bnd, int rows_per_n, int U, int V,
                                                    int VP, int which, float* __restrict__ m, uint16_t* __restrict__ hi,
                                                    uint16_t* __restrict__ lo, float* __restrict__ amy, int UPa,
                                                    float* __restrict__ lse, long long row) {
  __shared__ float red[8];
  __shared__ float bmx;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = (int)(row / rows_per_n), r = (int)(row % rows_per_n);
  const int Un = utt_U(bnd, n);
  const int lim = which == 0 ? utt_T(bnd, n) : Un + 1;
  uint2* H2 = reinterpret_cast<uint2*>(hi + row * (long long)VP);
  uint2* L2 = reinterpret_cast<uint2*>(lo + row * (long long)VP);
  const int V4 = V >> 2, VP4 = VP >> 2;
  if (r >= lim) {   // padded row: zero operand, never read otherwise
    for (int j = tid; j < VP4; j += 256) { H2[j] = make_uint2(0u, 0u); L2[j] = make_uint2(0u, 0u); }
    if (tid == 0) {
      m[row] = 0.f;
      if (lse) lse[row] = 0.f;
    }
    return;
  }
  const float* p = x + row * (long long)V;
  const float4* p4 = reinterpret_cast<const float4*>(p);
  float4 t[PER];
  float mx = neg_inf_f();
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int j = tid + 256 * k;
    t[k] = j < V4 ? __ldg(p4 + j) : make_float4(neg_inf_f(), neg_inf_f(), neg_inf_f(), neg_inf_f());
    mx = fmaxf(mx, fmaxf(fmaxf(t[k].x, t[k].y), fmaxf(t[k].z, t[k].w)));
  }
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  if (tid == 0) {
    float v = red[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) v = fmaxf(v, red[w]);
    bmx = v;
    m[row] = v;
  }
  __syncthreads();
  mx = bmx;
  float esum = 0.f;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int j = tid + 256 * k;
    if (j < VP4) {
      const float e0 = __expf(t[k].x - mx), e1 = __expf(t[k].y - mx);
      const float e2 = __expf(t[k].z - mx), e3 = __expf(t[k].w - mx);
      esum += (e0 + e1) + (e2 + e3);
      const __nv_bfloat162 h01 = __floats2bfloat162_rn(e0, e1), h23 = __floats2bfloat162_rn(e2, e3);
      const __nv_bfloat162 l01 = __floats2bfloat162_rn(e0 - __low2float(h01), e1 - __high2float(h01));
      const __nv_bfloat162 l23 = __floats2bfloat162_rn(e2 - __low2float(h23), e3 - __high2float(h23));
      H2[j] = make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
      L2[j] = make_uint2(*reinterpret_cast<const uint32_t*>(&l01), *reinterpret_cast<const uint32_t*>(&l23));
    }
  }
  for (int j = VP4 > 256 * PER ? 256 * PER + tid : VP4; j < VP4; j += 256) {   // (VP4 <= 256 PER: none)
    H2[j] = make_uint2(0u, 0u);
    L2[j] = make_uint2(0u, 0u);
  }
  if (lse) {   // lm rows: log sum_v exp lm[u,v] (the LM-only log-softmax of Eq. 14)
    esum = warp_sum(esum);
    __syncthreads();                                 // red reused
    if (lane == 0) red[warp] = esum;
    __syncthreads();
    if (tid == 0) {
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) v += red[w];
      lse[row] = mx + __logf(v);
    }
  }
  if (which == 0) {
    float* ay = amy + ((size_t)n * rows_per_n + r) * UPa;
    for (int u = tid; u <= Un; u += 256) {
      long long y = u < Un ? sym[(size_t)n * U + u] : 0;
      y = y < 0 ? 0 : (y >= V ? V - 1 : y);   // address safety; bad symbols flagged in status
      ay[u] = u < Un ? p[y] : 0.f;
    }
  }
}

// One launch for the independent prologue work of the simple loss, dispatched by block index:
// am rows (exp split + amy), lm rows (exp split), skewed-arc sentinels, validation.
struct PrepParams {
  const float *am, *lm;
  const int64_t *sym, *bnd;
  int N, T, U, V, VP, UP, LU, K;
  float *m_am, *m_lm, *amy, *lse_lm;
  uint16_t *eam_hi, *eam_lo, *elm_hi, *elm_lo;
  float2* pxy;
  int32_t* status;
  int nb_am, nb_lm, nb_fill;
  int rowblk;   // 1: one block per am / lm row (exp_split_row_block<8>), else 8 rows per block
};

// ROWBLK: the large-V row form (its 32-float4 register row would otherwise set the register budget, and so
// the occupancy, of the warp-per-row form too: c5 prep 29 -> 34 us)
template <bool ROWBLK>
__global__ void __launch_bounds__(256) simple_prep_kernel(PrepParams p) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  int b = blockIdx.x;
  if (ROWBLK) {
    if (b < p.nb_am) {
      exp_split_row_block<8>(p.am, p.sym, p.bnd, p.T, p.U, p.V, p.VP, 0, p.m_am, p.eam_hi, p.eam_lo, p.amy, p.UP,
                             nullptr, b);
      return;
    }
    b -= p.nb_am;
    if (b < p.nb_lm) {
      exp_split_row_block<8>(p.lm, p.sym, p.bnd, p.U + 1, p.U, p.V, p.VP, 1, p.m_lm, p.elm_hi, p.elm_lo, nullptr, 0,
                             p.lse_lm, b);
      return;
    }
    b -= p.nb_lm;
  } else if (b < p.nb_am) {
    exp_split_rows(p.am, p.sym, p.bnd, p.N, p.T, p.U, p.V, p.VP, 0, p.m_am, p.eam_hi, p.eam_lo, p.amy, p.UP, nullptr,
                   b);
    return;
  } else {
    b -= p.nb_am;
    if (b < p.nb_lm) {
      exp_split_rows(p.lm, p.sym, p.bnd, p.N, p.U + 1, p.U, p.V, p.VP, 1, p.m_lm, p.elm_hi, p.elm_lo, nullptr, 0,
                     p.lse_lm, b);
      return;
    }
    b -= p.nb_lm;
  }
  if (b < p.nb_fill) {
    // kNegBig in every invalid cell of the skewed arcs (lattice.cu conventions): a warp per row (n, k), lanes
    // over u, writing only the columns outside the row's lattice cells [max(0, k - T_n + 1), min(k, U_n)]
    // (one division per warp and row: the per-thread 64-bit divisions of a block-per-8-rows form were
    // 40 % of this kernel's samples at c5)
    const long long row = (long long)b * 8 + (threadIdx.x >> 5);
    if (row < (long long)p.N * (p.K + 1)) {
      const int n = (int)(row / (p.K + 1)), k = (int)(row - (long long)n * (p.K + 1));
      const int Tn = utt_T(p.bnd, n), Un = utt_U(p.bnd, n);
      const int lo = max(0, k - Tn + 1), hi = min(k, Un);   // (empty when lo > hi)
      float2* r = p.pxy + row * p.LU;
      const float2 sent = make_float2(kNegBig, kNegBig);
      for (int u = threadIdx.x & 31; u < p.LU; u += 32)
        if (u < lo || u > hi) r[u] = sent;
    }
    return;
  }
  b -= p.nb_fill;
  // validation of utterance b: symbols in [1, V), zero begins
  const int n = b, Un = utt_U(p.bnd, n);
  int bits = 0;
  if (threadIdx.x == 0 && (p.bnd[4 * n] != 0 || p.bnd[4 * n + 1] != 0)) bits |= kStatusBadBoundary;
  for (int u = threadIdx.x; u < Un && u < p.U; u += blockDim.x) {
    const int64_t y = p.sym[(size_t)n * p.U + u];
    if (y < 1 || y >= p.V) bits |= kStatusBadSymbol;
  }
  bits = __syncthreads_or(bits & kStatusBadSymbol) ? (bits | kStatusBadSymbol) : bits;
  if (threadIdx.x == 0) set_status(p.status, n, bits);
}

// ------------------------------------------------------------------ occupancy sums
// rowb[n,t] = sum_u empty'(t,u); colpy/colpb[n,tb,u] = sum_{t in 32-frame block tb} y'(t,u), empty'(t,u)
__global__ void __launch_bounds__(256) occ_sums_kernel(const float* __restrict__ px_grad,
                                                       const float* __restrict__ py_grad, int T, int U, int ntb,
                                                       float* __restrict__ rowb, float* __restrict__ colpy,
                                                       float* __restrict__ colpb, float* __restrict__ rowy) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  const int tb = blockIdx.x, n = blockIdx.y, U1 = U + 1, t0 = tb * 32;
  const int t1 = min(T, t0 + 32);
  for (int u = threadIdx.x; u < U1; u += blockDim.x) {
    float sy = 0.f, sb = 0.f;
    for (int t = t0; t < t1; ++t) {
      const size_t o = ((size_t)n * T + t) * U1 + u;
      sy += px_grad[o];
      sb += py_grad[o];
    }
    colpy[((size_t)n * ntb + tb) * U1 + u] = sy;
    colpb[((size_t)n * ntb + tb) * U1 + u] = sb;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = t0 + warp; t < t1; t += blockDim.x / 32) {
    float s = 0.f, sy = 0.f;
    for (int u = lane; u < U1; u += 32) {
      s += py_grad[((size_t)n * T + t) * U1 + u];
      sy += px_grad[((size_t)n * T + t) * U1 + u];
    }
    s = warp_sum(s);
    sy = warp_sum(sy);
    if (lane == 0) { rowb[(size_t)n * T + t] = s; rowy[(size_t)n * T + t] = sy; }
  }
}

// ------------------------------------------------------------------ smoothed trivial joiner
// Eq. 13-15 pieces that are not contractions: per utterance the unigram prior
// L_dec^avg(v) and per frame the normaliser of L_acoustic, then in the backward the factor through
// L_dec^avg.  One thread per column v (coalesced rows), or one warp per row.
//   Lavg(v) = log( (1/(U+1)) sum_u exp(lm[u,v] - lse_lm(u)) )
__global__ void __launch_bounds__(256) smooth_avg_kernel(const float* __restrict__ lm, const float* __restrict__ lse_lm,
                                                         const int64_t* __restrict__ bnd, int U, int V, int VP,
                                                         float* __restrict__ Lavg) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  const int n = blockIdx.y, v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= VP) return;
  const int Un = utt_U(bnd, n);
  float s = 0.f;
  if (v < V)
    for (int u = 0; u <= Un; ++u) s += __expf(lm[((size_t)n * (U + 1) + u) * V + v] - lse_lm[(size_t)n * (U + 1) + u]);
  Lavg[(size_t)n * VP + v] = v < V ? __logf(s / (float)(Un + 1)) : neg_inf_f();
}

//   lse_ac(t) = log sum_v exp(am[t,v] + Lavg(v))      (warp per frame)
__global__ void __launch_bounds__(256) smooth_ac_kernel(const float* __restrict__ am, const float* __restrict__ m_am,
                                                        const float* __restrict__ Lavg, const int64_t* __restrict__ bnd,
                                                        int N, int T, int V, int VP, float* __restrict__ lse_ac) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= (long long)N * T) return;
  const int n = (int)(row / T), t = (int)(row - (long long)n * T);
  if (t >= utt_T(bnd, n)) {
    if (lane == 0) lse_ac[row] = 0.f;
    return;
  }
  const float* a = am + row * V;
  const float* L = Lavg + (size_t)n * VP;
  const float mx = m_am[row];
  float s = 0.f;
  for (int v = lane; v < V; v += 32) s += __expf(a[v] - mx + L[v]);
  s = warp_sum(s);
  if (lane == 0) lse_ac[row] = mx + __logf(s);
}

//   g_avg(v) = sum_t (sum_u y' + empty')(t) P_ac(t,v) - sum_u [v = y_{u+1}] sum_t y'(t,u) - [v = 0] sum_{t,u} empty'
//   gq(v) = a_ac g_avg(v) / ((U+1) avg(v)),  P_ac(t,v) = exp(am[t,v] + Lavg(v) - lse_ac(t))
__global__ void __launch_bounds__(256) smooth_gq_kernel(const float* __restrict__ am, const float* __restrict__ Lavg,
                                                        const float* __restrict__ lse_ac, const float* __restrict__ rowy,
                                                        const float* __restrict__ rowb, const float* __restrict__ colpy,
                                                        const int64_t* __restrict__ sym, const int64_t* __restrict__ bnd,
                                                        int T, int U, int V, int VP, int ntb, float a_ac,
                                                        float* __restrict__ gq) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  const int n = blockIdx.y, v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= VP) return;
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  float g = 0.f;
  const float Lv = v < V ? Lavg[(size_t)n * VP + v] : 0.f;
  if (v < V) {
    float btot = 0.f;
    for (int t = 0; t < Tn; ++t) {
      const size_t r = (size_t)n * T + t;
      const float ob = rowb[r];
      g += (rowy[r] + ob) * __expf(am[r * V + v] + Lv - lse_ac[r]);
      btot += ob;
    }
    if (v == 0) g -= btot;
    for (int u = 0; u < Un; ++u)
      if (sym[(size_t)n * U + u] == v) {
        float cy = 0.f;
        for (int tb = 0; tb < ntb; ++tb) cy += colpy[((size_t)n * ntb + tb) * (U + 1) + u];
        g -= cy;
      }
  }
  gq[(size_t)n * VP + v] = v < V ? a_ac * g / ((float)(Un + 1) * __expf(Lv)) : 0.f;
}

//   Q(u) = sum_v softmax(lm[u])(v) gq(v)      (warp per token row)
__global__ void __launch_bounds__(256) smooth_q_kernel(const float* __restrict__ lm, const float* __restrict__ lse_lm,
                                                       const float* __restrict__ gq, const int64_t* __restrict__ bnd,
                                                       int N, int U, int V, int VP, float* __restrict__ Qu) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= (long long)N * (U + 1)) return;
  const int n = (int)(row / (U + 1)), u = (int)(row - (long long)n * (U + 1));
  if (u > utt_U(bnd, n)) {
    if (lane == 0) Qu[row] = 0.f;
    return;
  }
  const float* l = lm + row * V;
  const float* g = gq + (size_t)n * VP;
  const float z = lse_lm[row];
  float s = 0.f;
  for (int v = lane; v < V; v += 32) s += __expf(l[v] - z) * g[v];
  s = warp_sum(s);
  if (lane == 0) Qu[row] = s;
}

// ------------------------------------------------------------------ gemm3 mainloop
namespace sg {
constexpr int BM = 128, BK = 64;
constexpr int EPI_WARPS = 8, THREADS = 32 * (EPI_WARPS + 1);   // warps 0-7 epilogue, warp 8 TMA + MMA
constexpr int A_BYTES = BM * BK * 2;                        // 16 KB per hi | lo
constexpr int AUX_BYTES = 12288;                            // prologue tables (AmProb: up to 1023 label picks)
// per problem P: an N tile of P::kBN columns, P::kStages pipeline stages, P::kMinBlocks CTAs per SM.
// The gradient contractions (one K block per tile at c2 / c3) use 128-column tiles and one stage so that
// two CTAs share an SM (smem ~72 KB, TMEM <= 256 columns each): one CTA's epilogue overlaps the other's
// loads and MMAs.
template <class P> struct Geo {
  static constexpr int B_BYTES = P::kBN * BK * 2;                       // per hi | lo
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int SMEM_BYTES = P::kStages * STAGE_BYTES + AUX_BYTES + 1024 + 256;
  static constexpr uint32_t kCols = (P::kPhases == 2 ? 2 : 1) * P::kBN;   // TMEM columns (power of two)
};
constexpr int SCR = 32 * 33;                                // per-warp 32x32 staging block (floats)
}  // namespace sg

struct Tile {
  int n, m0, n0, nkb0, nkb1;   // k-blocks of phase 0 (bf16x3 product) and phase 1 (hi/lo x exact B)
};
struct Maps {
  CUtensorMap m[6];            // phase 0: A hi, A lo, B hi, B lo; phase 1: A' hi, A' lo
  CUtensorMap b1;              // phase 1: B' (exact)
  CUtensorMap ein, eout;       // epilogue fp32 input tiles (loaded after the mainloop) / output tiles
};
// Epilogue fp32 tiles: chunk c (32 columns x 128 rows, SWIZZLE_128B) at smem + c * EP_BYTES.
constexpr int EP_BYTES = 128 * 32 * 4;
// row r, 16-B chunk q of an epilogue tile
__device__ __forceinline__ float4* ep_at(uint8_t* tile, int r, int q) {
  return reinterpret_cast<float4*>(tile + r * 128 + ((q ^ (r & 7)) << 4));
}

__device__ __forceinline__ uint64_t kdesc(uint32_t base, int k) { return tc::sdesc(base + 32 * k, 16, 1024); }
__device__ __forceinline__ uint64_t mndesc(uint32_t base, int k) { return tc::sdesc(base + 2048 * k, 8192, 1024); }
// all 8 epilogue warps / the 4 warps of epilogue group g (one warp per TMEM lane quadrant)
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ void group_bar(int g) { asm volatile("bar.sync %0, 128;" ::"r"(2 + g) : "memory"); }

// Epilogue context of one thread: group g (0/1) takes the 32-column chunks c with c % 2 == g;
// quadrant q = warp % 4 owns TMEM lanes (tile rows) 32q..32q+31; row = 32q + lane.
struct Epi {
  int warp, lane, g, q, row;
  uint32_t taddr;   // TMEM address of this thread's lane, column 0
};

#ifdef RNNT_DIAGNOSTICS
__device__ unsigned long long* g_timeline = nullptr;   // diagnostics: per-CTA phase timestamps
#else
constexpr unsigned long long* g_timeline = nullptr;     // product build: tracing compiled out
#endif
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// diagnostics: epilogue-internal mark k (4..7) of this CTA, written by thread 0
__device__ __forceinline__ void etrace(int k) {
  if (g_timeline && threadIdx.x == 0) {
    const unsigned cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    g_timeline[(size_t)cta * 8 + k] = gtime();
  }
}

// Phase 0: acc0 (TMEM columns 0..kBN-1) += A_hi B_hi + A_hi B_lo + A_lo B_hi   (bf16x3)
// Phase 1: acc1 (TMEM columns kBN..2kBN-1) += A'_hi B' + A'_lo B'              (B' exact in bf16)
template <class P>
__global__ void __launch_bounds__(sg::THREADS, P::kMinBlocks) gemm3_kernel(const __grid_constant__ Maps mp, P p) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  using namespace sg;
  constexpr int STAGES = P::kStages, STAGE_BYTES = Geo<P>::STAGE_BYTES, B_BYTES = Geo<P>::B_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = tc::align1024(smem_raw);
  uint8_t* aux = smem + STAGES * STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(aux + AUX_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* ep_full = tfull + 1;                              // [8] epilogue input tiles
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ep_full + 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Tile tl = p.tile();
  if (tl.n < 0) return;
  constexpr uint32_t kCols = Geo<P>::kCols;
  const int nk = tl.nkb0 + (P::kPhases == 2 ? tl.nkb1 : 0);

  if (warp == EPI_WARPS && lane == 0) {
    for (int s = 0; s < STAGES; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
    tc::mbar_init(tfull, 1);
    for (int c = 0; c < 8; ++c) tc::mbar_init(&ep_full[c], 1);
    tc::fence_barrier_init();
    for (int i = 0; i < 4 + (P::kPhases == 2 ? 2 : 0); ++i) tc::tma_prefetch(&mp.m[i]);
    if (P::kPhases == 2) tc::tma_prefetch(&mp.b1);
  }
  if (warp == EPI_WARPS) tc::tmem_alloc(tmem_slot, kCols);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = *tmem_slot;

  unsigned long long* tlog = nullptr;
  if (g_timeline && threadIdx.x == 0) {
    const unsigned cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    tlog = g_timeline + (size_t)cta * 8;   // [0..3] kernel phases, [4..7] epilogue-internal marks (etrace)
    tlog[0] = gtime();
  }
  if (warp < EPI_WARPS) {
    Epi e;
    e.warp = warp; e.lane = lane; e.g = warp >> 2; e.q = warp & 3; e.row = 32 * e.q + lane;
    e.taddr = tbase + ((uint32_t)(32 * e.q) << 16);
    p.prologue(aux, tl);
    if (tlog) tlog[1] = gtime();
    if (nk > 0) {
      tc::mbar_wait(tfull, 0);
      tc::fence_after_sync();
    }
    if (tlog) tlog[2] = gtime();
    p.epilogue(smem, aux, tl, e, ep_full, mp);
    if (tlog) tlog[3] = gtime();
  } else if (lane == 0 && nk > 0) {
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nk; ++i) {
      const int phase = i < tl.nkb0 ? 0 : 1, kb = phase == 0 ? i : i - tl.nkb0;
      tc::mbar_wait(&empty[s], ph ^ 1);
      tc::mbar_arrive_expect_tx(&full[s], p.bytes(phase));
      p.load(smem + s * STAGE_BYTES, phase, kb, tl, &full[s], mp);
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
    // epilogue input tiles into the (now idle) stage buffers, as soon as the MMAs are done
    const int nep = p.epi_chunks(tl);
    if (nep > 0) {
      tc::mbar_wait(tfull, 0);
      for (int c = 0; c < nep; ++c) {
        tc::mbar_arrive_expect_tx(&ep_full[c], EP_BYTES);
        p.epi_load(c, smem + c * EP_BYTES, &ep_full[c], tl, mp);
      }
    }
  } else if (lane == 1 && nk > 0) {
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nk; ++i) {
      const int phase = i < tl.nkb0 ? 0 : 1, kb = phase == 0 ? i : i - tl.nkb0;
      const uint32_t idesc = p.idesc(phase);
      tc::mbar_wait(&full[s], ph);
      tc::fence_after_sync();
      const uint32_t ah = tc::smem_u32(smem + s * STAGE_BYTES), al = ah + A_BYTES;
      const uint32_t bh = ah + 2 * A_BYTES, bl = bh + B_BYTES;
#pragma unroll
      for (int k = 0; k < BK / 16; ++k) {
        const uint64_t dah = P::kA_MN ? mndesc(ah, k) : kdesc(ah, k);
        const uint64_t dal = P::kA_MN ? mndesc(al, k) : kdesc(al, k);
        const uint64_t dbh = P::kB_MN ? mndesc(bh, k) : kdesc(bh, k);
        if (phase == 0) {
          const uint64_t dbl = P::kB_MN ? mndesc(bl, k) : kdesc(bl, k);
          tc::mma_bf16(tbase, dah, dbh, idesc, (kb | k) != 0);   // hi * hi
          tc::mma_bf16(tbase, dah, dbl, idesc, 1);               // hi * lo
          tc::mma_bf16(tbase, dal, dbh, idesc, 1);               // lo * hi
        } else {
          tc::mma_bf16(tbase + P::kBN, dah, dbh, idesc, (kb | k) != 0);
          tc::mma_bf16(tbase + P::kBN, dal, dbh, idesc, 1);
        }
      }
      tc::mma_commit(&empty[s]);
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
    tc::mma_commit(tfull);
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == EPI_WARPS) tc::tmem_dealloc(tbase, kCols);
}

// Coalesced warp I/O of a 32-row x 32-column fp32 block through the per-warp staging buffer:
// row i of the block is rows0 + i (valid if i < nrows), columns c0 + lane (valid if < ncols).
__device__ __forceinline__ void warp_load_block(float (*buf)[33], const float* src, size_t ld, int nrows, int ncols,
                                                int lane) {
#pragma unroll 8
  for (int i = 0; i < 32; ++i) buf[i][lane] = (i < nrows && lane < ncols) ? src[(size_t)i * ld + lane] : 0.f;
  __syncwarp();
}
__device__ __forceinline__ void warp_store_block(const float (*buf)[33], float* dst, size_t ld, int nrows, int ncols,
                                                 int lane) {
  __syncwarp();
#pragma unroll 8
  for (int i = 0; i < 32; ++i)
    if (i < nrows && lane < ncols) dst[(size_t)i * ld + lane] = buf[i][lane];
  __syncwarp();
}

// ------------------------------------------------------------------ K2: normaliser + lattice arcs
// 128 x 128 tiles: twice the CTAs of 128 x 256 for the latency-bound epilogue (c5 44.9 -> 38.9 us; the
// epilogue's 8 warps x 12.4 KB transpose scratch lives in the 2 x 64 KB of stages, so 1 CTA per SM)
#ifndef RNNT_NORM_BN
#define RNNT_NORM_BN 128
#define RNNT_NORM_STAGES 2
#define RNNT_NORM_MINB 1
#endif
// BNT = 256 for large V (c4: the mainloop, not the epilogue, dominates; the am operand tile is then read
// once per utterance instead of once per 128 columns of u)
template <int BNT>
struct NormProbT {
  static constexpr bool kA_MN = false, kB_MN = false;
  // 128-column tiles: three 64 KB stages (the mainloop is bound by the load round trip per stage: two stages ran
  // 0.75-0.87 us per k-block at c5 / c3); 256-column tiles (96 KB stages): two
  // (64-column tiles, U + 1 <= 64 as at c3: four 48 KB stages)
  static constexpr int kPhases = 1, kBN = BNT,
                       kStages = BNT <= 64 ? RNNT_NORM_STAGES + 2 : (BNT <= 128 ? RNNT_NORM_STAGES + 1 : RNNT_NORM_STAGES),
                       kMinBlocks = RNNT_NORM_MINB;
  const float *lm, *m_am, *m_lm;
  const int64_t *sym, *bnd;
  int T, U, V, LU, K, BN, nkb, UPa;
  float2* pxy;     // (N,K+1,LU) skewed {y, empty} * log2e
  float* rS;       // (N,K+1,LU) skewed 1/S(t,u) (valid cells only)
  int32_t* status;
  const float *am, *amy;
  Smooth sm;                                   // Eq. 11 interpolation (both 0: plain trivial joiner)
  const float *lse_lm, *Lavg, *lse_ac;         // smoothing tables (workspace.h)
  int VPl;                                     // pitch of Lavg

  __device__ Tile tile() const {
    Tile t{(int)blockIdx.z, (int)blockIdx.x * sg::BM, (int)blockIdx.y * BN, nkb, 0};
    if (t.m0 >= utt_T(bnd, t.n) || t.n0 > utt_U(bnd, t.n)) t.n = -1;
    return t;
  }
  __device__ uint32_t bytes(int) const { return 2 * sg::A_BYTES + 2 * BN * sg::BK * 2; }
  __device__ uint32_t idesc(int) const { return tc::idesc_bf16(sg::BM, BN, false, false); }
  __device__ void load(uint8_t* st, int, int kb, const Tile& t, uint64_t* bar, const Maps& mp) const {
    tc::tma_load_3d(st, &mp.m[0], bar, kb * sg::BK, t.m0, t.n);
    tc::tma_load_3d(st + sg::A_BYTES, &mp.m[1], bar, kb * sg::BK, t.m0, t.n);
    tc::tma_load_3d(st + 2 * sg::A_BYTES, &mp.m[2], bar, kb * sg::BK, t.n0, t.n);
    tc::tma_load_3d(st + 2 * sg::A_BYTES + sg::Geo<NormProbT>::B_BYTES, &mp.m[3], bar, kb * sg::BK, t.n0, t.n);
  }
  __device__ int epi_chunks(const Tile&) const { return 0; }
  __device__ void epi_load(int, uint8_t*, uint64_t*, const Tile&, const Maps&) const {}
  // per-column tables of the tile: lm[u, y_{u+1}], lm[u, 0], m_lm[u]
  __device__ void prologue(uint8_t* aux, const Tile& t) const {
    float* lmy = reinterpret_cast<float*>(aux);
    float* lm0 = lmy + 256;
    float* mlm = lm0 + 256;
    float* lz = mlm + 256;      // smoothing: lse_lm(u)
    float* lyv = lz + 256;      // smoothing: Lavg(y_{u+1})
    const int Un = utt_U(bnd, t.n);
    for (int j = threadIdx.x; j < BN; j += 32 * sg::EPI_WARPS) {
      const int u = t.n0 + j;
      float a = 0.f, b = 0.f, c = 0.f, z = 0.f, w = 0.f;
      if (u <= Un) {
        const float* l = lm + ((size_t)t.n * (U + 1) + u) * V;
        if (u < Un) {
          long long yy = sym[(size_t)t.n * U + u];
          yy = yy < 0 ? 0 : (yy >= V ? V - 1 : yy);     // address safety; bad symbols flagged in status
          a = l[yy];
          if (sm.on()) w = Lavg[(size_t)t.n * VPl + yy];
        }
        b = l[0];
        c = m_lm[(size_t)t.n * (U + 1) + u];
        if (sm.on()) z = lse_lm[(size_t)t.n * (U + 1) + u];
      }
      lmy[j] = a; lm0[j] = b; mlm[j] = c; lz[j] = z; lyv[j] = w;
    }
    // the rows' {m_am(t), am[t, 0]} and the utterance's lengths for the epilogue, loaded while the mainloop runs
    // (as the epilogue's first statements they were two exposed global round trips after the last MMA)
    if (threadIdx.x < sg::BM) {
      const int trow = t.m0 + threadIdx.x;
      float2 r = make_float2(0.f, 0.f);
      if (trow < utt_T(bnd, t.n)) {
        const size_t arow = (size_t)t.n * T + trow;
        r = make_float2(m_am[arow], am[arow * V]);
      }
      reinterpret_cast<float2*>(aux + 5120)[threadIdx.x] = r;
    }
    if (threadIdx.x == 0) {
      reinterpret_cast<int*>(aux + 6144)[0] = utt_T(bnd, t.n);
      reinterpret_cast<int*>(aux + 6144)[1] = Un;
    }
    epi_bar();
  }
  __device__ void epilogue(uint8_t* smem, uint8_t* aux, const Tile& t, const Epi& e, uint64_t*, const Maps&) const {
    const float* lmy = reinterpret_cast<const float*>(aux);
    const float* lm0 = lmy + 256;
    const float* mlm = lm0 + 256;
    const float* lz = mlm + 256;
    const float* lyv = lz + 256;
    const int Tn = reinterpret_cast<const int*>(aux + 6144)[0], Un = reinterpret_cast<const int*>(aux + 6144)[1];
    const int trow = t.m0 + e.row;
    const bool rowok = trow < Tn;
    const int t0w = t.m0 + 32 * e.q;
    // per-warp 32 x 32 staging blocks with a pitch of 35 elements: the row-wise writes bxy[lane][j] and the
    // anti-diagonal reads bxy[i - lane][lane] are both (at most 2-way) bank-conflict free (a pitch of 33 put
    // every lane of a diagonal read on the same bank: 32-way)
    constexpr int PB = 35;
    static_assert(sg::EPI_WARPS * 32 * PB * 12 <= kStages * sg::Geo<NormProbT>::STAGE_BYTES, "staging fits the stages");
    float2 (*bxy)[PB] = reinterpret_cast<float2 (*)[PB]>(smem + e.warp * 32 * PB * 8);
    float (*brs)[PB] = reinterpret_cast<float (*)[PB]>(smem + sg::EPI_WARPS * 32 * PB * 8 + e.warp * 32 * PB * 4);
    const size_t arow = (size_t)t.n * T + (rowok ? trow : 0);
    const float2 rsc = reinterpret_cast<const float2*>(aux + 5120)[e.row];   // (prologue)
    const float mam = rsc.x, am0 = rsc.y;
    const float* ayr = amy + arow * UPa;
    const size_t nbase = (size_t)t.n * (K + 1);
    const bool smooth = sm.on();
    const float w0 = sm.w0();
    const float lac = (smooth && rowok) ? lse_ac[arow] : 0.f;        // normaliser of L_acoustic(t,.)
    const float L0 = smooth ? Lavg[(size_t)t.n * VPl] : 0.f;        // L_dec^avg(0)
    bool under = false;
    const int nch = (min(BN, Un + 1 - t.n0) + 31) / 32;   // 32-column chunks with at least one u <= U_n
    for (int c = e.g; c < nch; c += 2) {
      const int c0 = 32 * c, u0 = t.n0 + c0;
      float acc[32], ay[32];
      // the row's am[t, y_{u+1}] loads are issued first so their latency overlaps the TMEM load's
      if (rowok) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 v = reinterpret_cast<const float4*>(ayr + u0)[q];
          ay[4 * q] = v.x; ay[4 * q + 1] = v.y; ay[4 * q + 2] = v.z; ay[4 * q + 3] = v.w;
        }
      }
      tc::tmem_ld32(e.taddr + c0, acc);
      if (c == e.g) etrace(4);
      // branch-free per cell: every cell is computed (invalid ones from S = 1) and selected; the
      // smoothing term (a warp-uniform switch) is applied in a second, separate loop
      // (the chunk's column tables into registers first, as 16-B loads: read cell by cell between the staging
      //  stores of the loop below, which they may alias as far as the compiler knows, they could not be
      //  hoisted and the cells ran as a chain of shared-memory + MUFU latencies, 2.3 us per chunk)
      float tm[32], ty[32], t0[32];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 a = reinterpret_cast<const float4*>(mlm + c0)[q], b = reinterpret_cast<const float4*>(lmy + c0)[q],
                     d = reinterpret_cast<const float4*>(lm0 + c0)[q];
        tm[4 * q] = a.x; tm[4 * q + 1] = a.y; tm[4 * q + 2] = a.z; tm[4 * q + 3] = a.w;
        ty[4 * q] = b.x; ty[4 * q + 1] = b.y; ty[4 * q + 2] = b.z; ty[4 * q + 3] = b.w;
        t0[4 * q] = d.x; t0[4 * q + 1] = d.y; t0[4 * q + 2] = d.z; t0[4 * q + 3] = d.w;
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int u = u0 + j;
        const bool valid = rowok && u <= Un;
        const float S = valid ? acc[j] : 1.f;
        under |= !(S > 0.f);
        // base-2 throughout: Lnorm2 = log2 S + (m_am + m_lm) log2e = L_normalizer(t,u) log2e, Eq. 6
        const float Ln2 = lg2_approx(S) + (mam + tm[j]) * RNNT_LOG2E_F;
        const float px0 = fmaf(ay[j] + ty[j], RNNT_LOG2E_F, -Ln2);   // y(t,u) log2e, Eq. 1 + 5
        const float py0 = fmaf(am0 + t0[j], RNNT_LOG2E_F, -Ln2);     // empty(t,u) log2e, Eq. 2 + 5
        // y only below U_n; out of the last frame only the terminal blank exists
        const float px = (valid && u < Un) ? px0 : kNegBig;
        const float py = (valid && !(trow == Tn - 1 && u < Un)) ? py0 : kNegBig;
        bxy[e.lane][j] = make_float2(px, py);
        brs[e.lane][j] = valid ? rcp_approx(S) : 0.f;
      }
      if (smooth) {
        // Eq. 11: w0 L_trivial + a_lm L_lm (Eq. 14) + a_ac L_acoustic (Eq. 13)
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float2 xy = bxy[e.lane][j];
          if (xy.x > -1e29f)
            xy.x = fmaf(w0, xy.x, RNNT_LOG2E_F * (sm.a_lm * (lmy[c0 + j] - lz[c0 + j]) +
                                                  sm.a_ac * (ay[j] + lyv[c0 + j] - lac)));
          if (xy.y > -1e29f)
            xy.y = fmaf(w0, xy.y, RNNT_LOG2E_F * (sm.a_lm * (lm0[c0 + j] - lz[c0 + j]) + sm.a_ac * (am0 + L0 - lac)));
          bxy[e.lane][j] = xy;
        }
      }
      __syncwarp();
      if (c == e.g) etrace(5);
      // diagonal-major write of the arcs and of 1/S: for diagonal k = t0w + u0 + d, lane l holds
      // column u0 + l (t = k - u)
      // iteration i: lanes l <= i write diagonal t0w + u0 + i, lanes l > i diagonal t0w + u0 + i + 32
      // (two contiguous runs per store), so every lane writes a cell in each of 32 iterations
      const int u = u0 + e.lane;
      const size_t o0 = (nbase + t0w + u) * LU + u;   // cell (t0w, u); row t0w + tl_ is tl_ diagonals further
      if (u <= Un)
        for (int i = 0; i < 32; ++i) {
          const int tl_ = e.lane <= i ? i - e.lane : i + 32 - e.lane;
          if (t0w + tl_ < Tn) {
            const size_t o = o0 + (size_t)(tl_ * LU);
            pxy[o] = bxy[tl_][e.lane];
            rS[o] = brs[tl_][e.lane];
          }
        }
      __syncwarp();
      if (c == e.g) etrace(6);
    }
    etrace(7);
    if (under) set_status(status, t.n, kStatusUnderflow);
  }
};

// ------------------------------------------------------------------ K5a: am_grad
// The label picks -sum_u y'(t,u) [v = y_{u+1}] are applied in the epilogue: the prologue lists the (u,
// column) pairs whose label falls in the tile (about U kBN / V of them) and each row adds its fp32 y'(t,u)
// (px_grad) at those columns -- no second contraction against a one-hot matrix.
struct AmProb {
  static constexpr bool kA_MN = false, kB_MN = true;
  static constexpr int kPhases = 1, kBN = 128, kStages = 1, kMinBlocks = 2;
  static constexpr int kNC = kBN / 32;      // 32-column epilogue chunks per tile
  static constexpr int kMaxPicks = 1024;    // (u, column) pairs listed in aux (U <= 1023)
  static constexpr int kRowOff = 256 + kMaxPicks * 8;   // aux: per-row {m_am, rowb} after the pick list
  const float *am, *m_am, *rowb;
  const int64_t* bnd;
  int T, U, V;
  float gs;
  float* am_grad;
  bool tma_io;   // V % 4 == 0: fp32 rows are 16-B aligned, tiles move by TMA
  Smooth sm;
  const float *Lavg, *lse_ac, *rowy;
  int VPl;
  const float* px_grad;     // (N, T, U+1) y'
  const int64_t* sym;
  // d(-L)/d am[t,v] / gs = w0 E G~E_lm - (w0 + a_ac) picks + a_ac occ(t) P_ac(t,v)  (Eq. 11-13 chain rule)
  __device__ __forceinline__ float grad(float x, float mam, float a0, float pick, float occ, float Lv, float lac) const {
    float g = sm.w0() * __expf(x - mam) * a0 - (sm.w0() + sm.a_ac) * pick;
    if (sm.a_ac != 0.f) g = fmaf(sm.a_ac * occ, __expf(x + Lv - lac), g);
    return gs * g;
  }

  __device__ Tile tile() const {
    Tile t{(int)blockIdx.z, (int)blockIdx.x * sg::BM, (int)blockIdx.y * kBN, 0, 0};
    const int Tn = utt_T(bnd, t.n), Un = utt_U(bnd, t.n);
    t.nkb0 = (t.m0 < Tn) ? (Un + 1 + sg::BK - 1) / sg::BK : 0;
    return t;
  }
  __device__ uint32_t bytes(int) const { return 2 * sg::A_BYTES + 2 * sg::Geo<AmProb>::B_BYTES; }
  __device__ uint32_t idesc(int) const { return tc::idesc_bf16(sg::BM, kBN, false, true); }
  // A = G~ (hi, lo; K-major over u), B = E_lm (hi, lo; MN-major)
  __device__ void load(uint8_t* st, int, int kb, const Tile& t, uint64_t* bar, const Maps& mp) const {
    tc::tma_load_3d(st, &mp.m[0], bar, kb * sg::BK, t.m0, t.n);
    tc::tma_load_3d(st + sg::A_BYTES, &mp.m[1], bar, kb * sg::BK, t.m0, t.n);
#pragma unroll
    for (int i = 0; i < kBN / 64; ++i) {
      tc::tma_load_3d(st + 2 * sg::A_BYTES + i * 8192, &mp.m[2], bar, t.n0 + 64 * i, kb * sg::BK, t.n);
      tc::tma_load_3d(st + 2 * sg::A_BYTES + sg::Geo<AmProb>::B_BYTES + i * 8192, &mp.m[3], bar, t.n0 + 64 * i,
                      kb * sg::BK, t.n);
    }
  }
  __device__ int epi_chunks(const Tile& t) const { return (tma_io && t.nkb0 > 0) ? min(kNC, (V - t.n0 + 31) / 32) : 0; }
  __device__ void epi_load(int c, uint8_t* dst, uint64_t* bar, const Tile& t, const Maps& mp) const {
    tc::tma_load_3d(dst, &mp.ein, bar, t.n0 + 32 * c, t.m0, t.n);
  }
  // aux: ints [0..4] where each 32-column chunk's picks start in the list ([4] = their total), ints [8..40) the
  // per-warp per-chunk counts of the scan; at aux + 256 the (u, column - n0) pairs of the labels falling in this
  // tile, grouped by chunk and in ascending u inside a chunk (ballot / warp-count scans: a deterministic order,
  // so duplicate labels always add in the same order).  Grouping by chunk lets the epilogue of a chunk walk only
  // its own picks (c5: ~5 of the tile's ~20; walking all of them cost 4 us per chunk, mostly y' load latency).
  __device__ void prologue(uint8_t* aux, const Tile& t) const {
    int* off = reinterpret_cast<int*>(aux);
    int* wc = off + 8;                                    // [EPI_WARPS][kNC]
    int2* pk = reinterpret_cast<int2*>(aux + 256);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int Un = utt_U(bnd, t.n);
    // the rows' scalars {m_am, sum_u empty'} for the epilogue, loaded while the operands are in flight (as the
    // epilogue's first statements they were an exposed L2 / HBM round trip after the MMAs): aux + kRowOff
    float2 rsc = make_float2(0.f, 0.f);
    if (threadIdx.x < sg::BM && t.m0 + (int)threadIdx.x < utt_T(bnd, t.n)) {
      const size_t row = (size_t)t.n * T + t.m0 + threadIdx.x;
      rsc = make_float2(m_am[row], rowb[row]);
    }
    auto label = [&](int u, bool& hit, int& col) {
      hit = false;
      col = 0;
      if (u < Un) {
        const long long y = sym[(size_t)t.n * U + u];
        hit = y >= t.n0 && y < t.n0 + kBN && y < V;
        col = (int)(y - t.n0);
      }
    };
    // pass 1: picks per chunk
    int cnt[kNC];
#pragma unroll
    for (int c = 0; c < kNC; ++c) cnt[c] = 0;
    for (int u0 = 0; u0 < Un; u0 += 32 * sg::EPI_WARPS) {
      bool hit;
      int col;
      label(u0 + (int)threadIdx.x, hit, col);
#pragma unroll
      for (int c = 0; c < kNC; ++c) cnt[c] += __popc(__ballot_sync(0xffffffffu, hit && (col >> 5) == c));
    }
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < kNC; ++c) wc[warp * kNC + c] = cnt[c];
    }
    epi_bar();
    int base[kNC + 1];
    {
      int run = 0;
#pragma unroll
      for (int c = 0; c < kNC; ++c) {
        base[c] = run;
        for (int w = 0; w < sg::EPI_WARPS; ++w) run += wc[w * kNC + c];
      }
      base[kNC] = run;
    }
    epi_bar();                                            // (wc is rewritten below)
    if (threadIdx.x == 0) {
#pragma unroll
      for (int c = 0; c <= kNC; ++c) off[c] = min(base[c], kMaxPicks);
    }
    // pass 2: placement
    for (int u0 = 0; u0 < Un; u0 += 32 * sg::EPI_WARPS) {
      const int u = u0 + (int)threadIdx.x;
      bool hit;
      int col;
      label(u, hit, col);
      unsigned bl[kNC];
#pragma unroll
      for (int c = 0; c < kNC; ++c) {
        bl[c] = __ballot_sync(0xffffffffu, hit && (col >> 5) == c);
        if (lane == 0) wc[warp * kNC + c] = __popc(bl[c]);
      }
      epi_bar();
#pragma unroll
      for (int c = 0; c < kNC; ++c) {
        int o = base[c], tot = 0;
        for (int w = 0; w < sg::EPI_WARPS; ++w) {
          const int x = wc[w * kNC + c];
          if (w < warp) o += x;
          tot += x;
        }
        const int i = o + __popc(bl[c] & ((1u << lane) - 1u));
        if (hit && (col >> 5) == c && i < kMaxPicks) pk[i] = make_int2(u, col);
        base[c] += tot;
      }
      epi_bar();
    }
    if (threadIdx.x < sg::BM) reinterpret_cast<float2*>(aux + kRowOff)[threadIdx.x] = rsc;
    if (threadIdx.x == 0) off[5] = utt_T(bnd, t.n);       // (the epilogue's T_n: no boundary load after the MMAs)
    epi_bar();
  }
  // the picks of row trow for the 32 columns of chunk c (fp32 y' from px_grad)
  __device__ __forceinline__ void picks(const uint8_t* aux, int c, int trow, bool live, const Tile& t,
                                        float (&a1)[32]) const {
#pragma unroll
    for (int j = 0; j < 32; ++j) a1[j] = 0.f;
    if (!live) return;
    const int* off = reinterpret_cast<const int*>(aux);
    const int i0 = off[c], i1 = off[c + 1];
    const int2* pk = reinterpret_cast<const int2*>(aux + 256);
    const float* yr = px_grad + ((size_t)t.n * T + trow) * (U + 1);
#pragma unroll 2
    for (int i = i0; i < i1; ++i) {
      const int2 q = pk[i];
      const int jj = q.y - 32 * c;
      const float yv = yr[q.x];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j == jj) a1[j] += yv;
    }
  }
  __device__ void epilogue(uint8_t* smem, uint8_t* aux, const Tile& t, const Epi& e, uint64_t* ep_full,
                           const Maps& mp) const {
    const int Tn = reinterpret_cast<const int*>(aux)[5];   // (prologue)
    const int trow = t.m0 + e.row;
    const bool live = trow < Tn;
    const int nep = epi_chunks(t);
    if (nep > 0) {
      // d(-L_simple)/d am = E_am (G~ E_lm) - y' [v = y_{u+1}] - [v=0] sum_u empty'   (times gs), tile in place
      const size_t row = (size_t)t.n * T + (live ? trow : 0);
      const float2 rsc = reinterpret_cast<const float2*>(aux + kRowOff)[e.row];   // (prologue)
      const float mam = rsc.x, rb = rsc.y;
      const float occ = (live && sm.on()) ? rb + rowy[row] : 0.f;
      const float lac = (live && sm.on()) ? lse_ac[row] : 0.f;
      const float* Lr = Lavg + (size_t)t.n * VPl;
      for (int c = e.g; c < nep; c += 2) {
        const int vc = t.n0 + 32 * c;
        uint8_t* tile = smem + c * EP_BYTES;
        if (!sm.on()) {
          // The plain trivial joiner (w0 = 1, no smoothing terms): gs e^(x - m_am) a0 for the whole chunk (~6
          // instructions per element; the general form below, with its per-element smoothing selects, is ~30
          // and made the epilogue issue-bound: 2.3 us per chunk at 4 warps per scheduler), then the row's picks
          // subtracted in place in the staged tile.  The y' values of the chunk's picks are loaded eight at a
          // time, the first batch before the accumulator / input-tile waits (as dependent loads walked one by
          // one they were 3.6 us per chunk at c5).
          const int* off = reinterpret_cast<const int*>(aux);
          const int2* pk = reinterpret_cast<const int2*>(aux + 256);
          const int i0 = live ? off[c] : 0, i1 = live ? off[c + 1] : 0;
          const float* yr = px_grad + ((size_t)t.n * T + (live ? trow : 0)) * (U + 1);
          float yv[8];
          int jj[8];
          auto load8 = [&](int i) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const bool ok = i + k < i1;
              const int2 q = ok ? pk[i + k] : make_int2(0, -1);
              jj[k] = ok ? q.y - 32 * c : -1;
              yv[k] = ok ? yr[q.x] : 0.f;
            }
          };
          auto apply8 = [&]() {
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (jj[k] >= 0) reinterpret_cast<float*>(ep_at(tile, e.row, jj[k] >> 2))[jj[k] & 3] -= gs * yv[k];
          };
          load8(i0);
          float a0[32];
          if (c == e.g) etrace(4);
          tc::tmem_ld32(e.taddr + 32 * c, a0);
          tc::mbar_wait(&ep_full[c], 0);
          if (c == e.g) etrace(5);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float4* pq = ep_at(tile, e.row, q);
            const float4 x = *pq;
            const float xs[4] = {x.x, x.y, x.z, x.w};
            float o[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) o[i] = gs * (__expf(xs[i] - mam) * a0[4 * q + i]);
            *pq = live ? make_float4(o[0], o[1], o[2], o[3]) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
          if (live) {
            apply8();
            for (int i = i0 + 8; i < i1; i += 8) {
              load8(i);
              apply8();
            }
            if (vc == 0) reinterpret_cast<float*>(ep_at(tile, e.row, 0))[0] -= gs * rb;
          }
        } else {
        float a0[32], a1[32];
        picks(aux, c, trow, live, t, a1);
        tc::tmem_ld32(e.taddr + 32 * c, a0);
        tc::mbar_wait(&ep_full[c], 0);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4* pq = ep_at(tile, e.row, q);
          const float4 x = *pq;
          const float xs[4] = {x.x, x.y, x.z, x.w};
          float o[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int j = 4 * q + i;
            const float pick = a1[j] + ((vc + j == 0) ? rb : 0.f);
            o[i] = live ? grad(xs[i], mam, a0[j], pick, occ, sm.on() ? Lr[vc + j] : 0.f, lac) : 0.f;
          }
          *pq = make_float4(o[0], o[1], o[2], o[3]);
        }
        }
        tc::fence_proxy_async();
        group_bar(e.g);
        if (e.row == 0) {
          tc::tma_store_3d(&mp.eout, tile, vc, t.m0, t.n);
          tc::bulk_commit();
        }
        if (c == 0) etrace(6);
      }
      etrace(7);
      if (e.row == 0) tc::bulk_wait_read0();
      return;
    }
    if (tma_io && t.nkb0 == 0) {
      // a tile of padded frames only (t >= T_n): its rows are exactly 0 -- a warp per row, one float4 store
      // per lane (V % 4 == 0: 16-B aligned rows), instead of the staged generic path (traced at 9 us per such
      // tile, as long as a live one; 39 % of the tiles at c3, 25 % at c5)
      const int r1 = min(T, t.m0 + sg::BM), nc4 = min(kBN, V - t.n0) >> 2;
      for (int r = t.m0 + e.warp; r < r1; r += sg::EPI_WARPS) {
        float4* dst = reinterpret_cast<float4*>(am_grad + ((size_t)t.n * T + r) * V + t.n0);
        if (e.lane < nc4) dst[e.lane] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      return;
    }
    // generic path (V % 4 != 0): coalesced warp I/O through smem
    const int t0w = t.m0 + 32 * e.q;
    if (t0w >= T) return;                               // whole warp beyond the padded rows
    const size_t row0 = (size_t)t.n * T + t0w;
    const float mam = live ? m_am[row0 + e.lane] : 0.f;
    const float rb = live ? rowb[row0 + e.lane] : 0.f;
    const float occ = (live && sm.on()) ? rb + rowy[row0 + e.lane] : 0.f;
    const float lac = (live && sm.on()) ? lse_ac[row0 + e.lane] : 0.f;
    const float* Lr = Lavg + (size_t)t.n * VPl;
    float (*buf)[33] = reinterpret_cast<float (*)[33]>(smem + e.warp * sg::SCR * 4);
    const int nin = min(32, Tn - t0w), nout = min(32, T - t0w);
    for (int c = e.g; c < kNC; c += 2) {
      const int vc = t.n0 + 32 * c;
      if (vc >= V) break;
      float a0[32], a1[32];
      picks(aux, c, t0w + e.lane, live, t, a1);
      if (t.nkb0 > 0) {
        tc::tmem_ld32(e.taddr + 32 * c, a0);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) a0[j] = 0.f;
      }
      const int nc = min(32, V - vc);
      warp_load_block(buf, am + row0 * V + vc, V, nin, nc, e.lane);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float pick = a1[j] + ((vc + j == 0) ? rb : 0.f);
        buf[e.lane][j] = live ? grad(buf[e.lane][j], mam, a0[j], pick, occ, (sm.on() && vc + j < V) ? Lr[vc + j] : 0.f, lac)
                              : 0.f;
      }
      warp_store_block(buf, am_grad + row0 * V + vc, V, nout, nc, e.lane);
    }
  }
};

// ------------------------------------------------------------------ K5b: lm_grad
struct LmProb {
  static constexpr bool kA_MN = true, kB_MN = true;
  static constexpr int kPhases = 1, kBN = 128, kStages = 1, kMinBlocks = 2;
  static constexpr int kNC = kBN / 32;
  const float *lm, *m_lm, *colpy, *colpb;
  const int64_t *sym, *bnd;
  int T, U, V, ntb;
  float gs;
  float* lm_grad;
  bool tma_io;
  Smooth sm;
  const float *lse_lm, *gq, *Qu;
  int VPl;
  // d(-L)/d lm[u,v] / gs = w0 E G~^T E_am - (w0 + a_lm) picks + a_lm occ(u) P_lm + P_lm (gq(v) - Q(u))
  __device__ __forceinline__ float grad(float x, float mlm, float acc, float pick, float occ, float lz, float g,
                                        float Q) const {
    float r = sm.w0() * __expf(x - mlm) * acc - (sm.w0() + sm.a_lm) * pick;
    if (sm.on()) r = fmaf(__expf(x - lz), sm.a_lm * occ + g - Q, r);
    return gs * r;
  }

  __device__ Tile tile() const {
    Tile t{(int)blockIdx.z, (int)blockIdx.x * sg::BM, (int)blockIdx.y * kBN, 0, 0};
    const int Tn = utt_T(bnd, t.n), Un = utt_U(bnd, t.n);
    t.nkb0 = (t.m0 <= Un) ? (Tn + sg::BK - 1) / sg::BK : 0;
    return t;
  }
  __device__ uint32_t bytes(int) const { return 2 * sg::A_BYTES + 2 * sg::Geo<LmProb>::B_BYTES; }
  __device__ uint32_t idesc(int) const { return tc::idesc_bf16(sg::BM, kBN, true, true); }
  __device__ void load(uint8_t* st, int, int kb, const Tile& t, uint64_t* bar, const Maps& mp) const {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      tc::tma_load_3d(st + i * 8192, &mp.m[0], bar, t.m0 + 64 * i, kb * sg::BK, t.n);
      tc::tma_load_3d(st + sg::A_BYTES + i * 8192, &mp.m[1], bar, t.m0 + 64 * i, kb * sg::BK, t.n);
    }
#pragma unroll
    for (int i = 0; i < kBN / 64; ++i) {
      tc::tma_load_3d(st + 2 * sg::A_BYTES + i * 8192, &mp.m[2], bar, t.n0 + 64 * i, kb * sg::BK, t.n);
      tc::tma_load_3d(st + 2 * sg::A_BYTES + sg::Geo<LmProb>::B_BYTES + i * 8192, &mp.m[3], bar, t.n0 + 64 * i,
                      kb * sg::BK, t.n);
    }
  }
  __device__ int epi_chunks(const Tile& t) const { return (tma_io && t.nkb0 > 0) ? min(kNC, (V - t.n0 + 31) / 32) : 0; }
  __device__ void epi_load(int c, uint8_t* dst, uint64_t* bar, const Tile& t, const Maps& mp) const {
    tc::tma_load_3d(dst, &mp.ein, bar, t.n0 + 32 * c, t.m0, t.n);
  }
  // the rows' scalars {sum_t y', sum_t empty', m_lm, label} for the epilogue, loaded while the operands are in
  // flight (2 ntb + 2 loads per row that were an exposed round trip after the MMAs): aux[128] float4
  __device__ void prologue(uint8_t* aux, const Tile& t) const {
    const int Un = utt_U(bnd, t.n), U1 = U + 1;
    if (threadIdx.x < sg::BM) {
      const int urow = t.m0 + threadIdx.x;
      float csy = 0.f, csb = 0.f, mlm = 0.f;
      int y = -1;
      if (urow <= Un) {
        for (int tb = 0; tb < ntb; ++tb) {
          csy += colpy[((size_t)t.n * ntb + tb) * U1 + urow];
          csb += colpb[((size_t)t.n * ntb + tb) * U1 + urow];
        }
        if (urow < Un) y = (int)sym[(size_t)t.n * U + urow];
        mlm = m_lm[(size_t)t.n * U1 + urow];
      }
      reinterpret_cast<float4*>(aux)[threadIdx.x] = make_float4(csy, csb, mlm, __int_as_float(y));
    }
    if (threadIdx.x == 0) *reinterpret_cast<int*>(aux + 2048) = Un;
    epi_bar();
  }
  __device__ void epilogue(uint8_t* smem, uint8_t* aux, const Tile& t, const Epi& e, uint64_t* ep_full,
                           const Maps& mp) const {
    const int Un = *reinterpret_cast<const int*>(aux + 2048), U1 = U + 1;   // (prologue)
    if (tma_io && t.nkb0 == 0) {
      // a tile of padded token positions only (u > U_n): exact zeros, a warp per row (see AmProb)
      const int r1 = min(U1, t.m0 + sg::BM), nc4 = min(kBN, V - t.n0) >> 2;
      for (int r = t.m0 + e.warp; r < r1; r += sg::EPI_WARPS) {
        float4* dst = reinterpret_cast<float4*>(lm_grad + ((size_t)t.n * U1 + r) * V + t.n0);
        if (e.lane < nc4) dst[e.lane] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      return;
    }
    const int urow = t.m0 + e.row;
    const bool live = urow <= Un;
    const float4 rsc = reinterpret_cast<const float4*>(aux)[e.row];   // (prologue)
    const float csy = rsc.x, csb = rsc.y;
    const int y = __float_as_int(rsc.w);
    const float lz = (live && sm.on()) ? lse_lm[(size_t)t.n * U1 + urow] : 0.f;
    const float Q = (live && sm.on()) ? Qu[(size_t)t.n * U1 + urow] : 0.f;
    const float* gr = gq + (size_t)t.n * VPl;
    const int nep = epi_chunks(t);
    if (nep > 0) {
      const float mlm = rsc.z;
      for (int c = e.g; c < nep; c += 2) {
        const int vc = t.n0 + 32 * c;
        float acc[32];
        tc::tmem_ld32(e.taddr + 32 * c, acc);
        tc::mbar_wait(&ep_full[c], 0);
        uint8_t* tile = smem + c * EP_BYTES;
        if (!sm.on()) {
          // the plain trivial joiner: gs e^(x - m_lm) acc everywhere, then the row's two picks (its label column
          // and the blank column) subtracted in place -- see AmProb
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float4* pq = ep_at(tile, e.row, q);
            const float4 x = *pq;
            const float xs[4] = {x.x, x.y, x.z, x.w};
            float o[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) o[i] = gs * (__expf(xs[i] - mlm) * acc[4 * q + i]);
            *pq = live ? make_float4(o[0], o[1], o[2], o[3]) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
          if (live) {
            const int jy = y - vc;
            if ((unsigned)jy < 32u) reinterpret_cast<float*>(ep_at(tile, e.row, jy >> 2))[jy & 3] -= gs * csy;
            if (vc == 0) reinterpret_cast<float*>(ep_at(tile, e.row, 0))[0] -= gs * csb;
          }
        } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4* pq = ep_at(tile, e.row, q);
          const float4 x = *pq;
          const float xs[4] = {x.x, x.y, x.z, x.w};
          float o[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int j = 4 * q + i, v = vc + j;
            const float pick = (v == y ? csy : 0.f) + (v == 0 ? csb : 0.f);
            o[i] = live ? grad(xs[i], mlm, acc[j], pick, csy + csb, lz, sm.on() ? gr[v] : 0.f, Q) : 0.f;
          }
          *pq = make_float4(o[0], o[1], o[2], o[3]);
        }
        }
        tc::fence_proxy_async();
        group_bar(e.g);
        if (e.row == 0) {
          tc::tma_store_3d(&mp.eout, tile, vc, t.m0, t.n);
          tc::bulk_commit();
        }
      }
      if (e.row == 0) tc::bulk_wait_read0();
      return;
    }
    const int u0w = t.m0 + 32 * e.q;
    if (u0w >= U1) return;                               // whole warp beyond the padded rows
    const size_t row0 = (size_t)t.n * U1 + u0w;
    const float mlm = live ? m_lm[row0 + e.lane] : 0.f;
    float (*buf)[33] = reinterpret_cast<float (*)[33]>(smem + e.warp * sg::SCR * 4);
    const int nin = min(32, Un + 1 - u0w), nout = min(32, U1 - u0w);
    for (int c = e.g; c < kNC; c += 2) {
      const int vc = t.n0 + 32 * c;
      if (vc >= V) break;
      float acc[32];
      if (t.nkb0 > 0) {
        tc::tmem_ld32(e.taddr + 32 * c, acc);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = 0.f;
      }
      const int nc = min(32, V - vc);
      warp_load_block(buf, lm + row0 * V + vc, V, nin, nc, e.lane);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int v = vc + j;
        const float pick = (v == y ? csy : 0.f) + (v == 0 ? csb : 0.f);
        buf[e.lane][j] = live ? grad(buf[e.lane][j], mlm, acc[j], pick, csy + csb, lz, (sm.on() && v < V) ? gr[v] : 0.f, Q)
                              : 0.f;
      }
      warp_store_block(buf, lm_grad + row0 * V + vc, V, nout, nc, e.lane);
    }
  }
};

// ------------------------------------------------------------------ host
template <class P>
static cudaError_t launch_gemm3(const P& p, dim3 grid, const Maps& mp, int kid, cudaStream_t st) {
  smem_optin(gemm3_kernel<P>, sg::Geo<P>::SMEM_BYTES);
  if (grid.x == 0 || grid.y == 0 || grid.z == 0) return cudaSuccess;
  RNNT_LAUNCH(kid, st, launch_pdl(gemm3_kernel<P>, grid, sg::THREADS, sg::Geo<P>::SMEM_BYTES, st, mp, p));
  return cudaGetLastError();
}

static bool tm3(CUtensorMap* m, const uint16_t* base, int pitch, int rows, int N, int box_rows) {
  return make_tmap_bf16_3d(m, base, (uint64_t)pitch, (uint64_t)rows, (uint64_t)N, (uint64_t)pitch * 2,
                           (uint64_t)pitch * rows * 2, 64, (uint32_t)box_rows);
}

#ifdef RNNT_DIAGNOSTICS
void set_timeline(void* buf) { cudaMemcpyToSymbol(g_timeline, &buf, sizeof(buf)); }
#endif

cudaError_t simple_prep_launch(const Dims& d, const SimpleWS& w, const float* am, const float* lm, const int64_t* sym,
                               const int64_t* bnd, int32_t* status, cudaStream_t st) {
  PrepParams p;
  p.am = am; p.lm = lm; p.sym = sym; p.bnd = bnd;
  p.N = d.N; p.T = d.T; p.U = d.U; p.V = d.V; p.VP = d.VP64(); p.UP = d.UP(); p.LU = d.LU(); p.K = d.K();
  p.m_am = w.m_am; p.m_lm = w.m_lm; p.amy = w.amy; p.lse_lm = w.lse_lm;
  p.eam_hi = w.Eam_hi; p.eam_lo = w.Eam_lo; p.elm_hi = w.Elm_hi; p.elm_lo = w.Elm_lo;
  p.pxy = w.pxy; p.status = status;
  p.rowblk = (d.V % 4 == 0 && d.V > 2048 && d.VP64() <= 4 * 256 * 8) ? 1 : 0;
  p.nb_am = (int)(p.rowblk ? (long long)d.N * d.T : ((long long)d.N * d.T + 7) / 8);
  p.nb_lm = (int)(p.rowblk ? (long long)d.N * d.U1() : ((long long)d.N * d.U1() + 7) / 8);
  p.nb_fill = (int)(((long long)d.N * (d.K() + 1) + 7) / 8);
  const unsigned grid = (unsigned)(p.nb_am + p.nb_lm + p.nb_fill + d.N);
  if (p.rowblk) RNNT_LAUNCH(KID_ROWMAX_AM, st, launch_pdl(simple_prep_kernel<true>, grid, 256, 0, st, p));
  else RNNT_LAUNCH(KID_ROWMAX_AM, st, launch_pdl(simple_prep_kernel<false>, grid, 256, 0, st, p));
  return cudaGetLastError();
}

template <class NP>
static cudaError_t launch_norm(const Dims& d, const SimpleWS& w, const float* am, const float* lm, const int64_t* sym,
                               const int64_t* bnd, int32_t* status, Smooth sm, cudaStream_t st) {
  const int BN = std::min(NP::kBN, (d.U1() + 15) / 16 * 16);
  Maps mp;
  if (!tm3(&mp.m[0], w.Eam_hi, d.VP64(), d.T, d.N, sg::BM) || !tm3(&mp.m[1], w.Eam_lo, d.VP64(), d.T, d.N, sg::BM) ||
      !tm3(&mp.m[2], w.Elm_hi, d.VP64(), d.U1(), d.N, BN) || !tm3(&mp.m[3], w.Elm_lo, d.VP64(), d.U1(), d.N, BN))
    return cudaErrorInvalidValue;
  NP p{lm, w.m_am, w.m_lm, sym, bnd, d.T, d.U, d.V, d.LU(), d.K(), BN, d.VP64() / 64, d.UP(),
             w.pxy, w.rS, status, am, w.amy, sm, w.lse_lm, w.Lavg, w.lse_ac, d.VP64()};
  dim3 grid((d.T + sg::BM - 1) / sg::BM, (d.U1() + BN - 1) / BN, d.N);
  return launch_gemm3(p, grid, mp, KID_NORM, st);
}

cudaError_t norm_gemm_launch(const Dims& d, const SimpleWS& w, const float* am, const float* lm, const int64_t* sym,
                             const int64_t* bnd, int32_t* status, Smooth sm, cudaStream_t st) {
  if (sm.on()) {
    // the smoothed joiner's utterance prior L_dec^avg and the L_acoustic normalisers (Eq. 13, 15)
    RNNT_LAUNCH(KID_SMOOTH_AVG, st, launch_pdl(smooth_avg_kernel, dim3((d.VP64() + 255) / 256, d.N), 256, 0, st, 
        lm, w.lse_lm, bnd, d.U, d.V, d.VP64(), w.Lavg));
    RNNT_LAUNCH(KID_SMOOTH_AC, st, launch_pdl(smooth_ac_kernel, (unsigned)(((long long)d.N * d.T + 7) / 8), 256, 0, st, 
        am, w.m_am, w.Lavg, bnd, d.N, d.T, d.V, d.VP64(), w.lse_ac));
  }
  // 128 x 256 tiles for large V (mainloop-bound: fewer, longer tiles); 128 x 128 otherwise (epilogue-bound)
  if (d.VP64() >= 2048 && d.U1() > 128)
    return launch_norm<NormProbT<256>>(d, w, am, lm, sym, bnd, status, sm, st);
  if (d.U1() <= 64) return launch_norm<NormProbT<64>>(d, w, am, lm, sym, bnd, status, sm, st);
  return launch_norm<NormProbT<RNNT_NORM_BN>>(d, w, am, lm, sym, bnd, status, sm, st);
}

cudaError_t simple_grads_launch(const Dims& d, const SimpleWS& w, const float* am, const float* lm,
                                const float* px_grad, const float* py_grad, const int64_t* sym, const int64_t* bnd,
                                float gs, float* am_grad, float* lm_grad, Smooth sm, cudaStream_t st) {
  if (!am_grad && !lm_grad) return cudaSuccess;
  RNNT_LAUNCH(KID_OCCSUMS, st, launch_pdl(occ_sums_kernel, dim3(d.ntb(), d.N), 256, 0, st, px_grad, py_grad, d.T, d.U, d.ntb(),
                                                                                   w.rowb, w.colpy, w.colpb, w.rowy));
  cudaError_t e;
  if (sm.on() && lm_grad) {
    // backward through L_dec^avg (Eq. 15): gq(v), then Q(u) = sum_v softmax(lm[u])(v) gq(v)
    RNNT_LAUNCH(KID_SMOOTH_GQ, st, launch_pdl(smooth_gq_kernel, dim3((d.VP64() + 255) / 256, d.N), 256, 0, st, 
        am, w.Lavg, w.lse_ac, w.rowy, w.rowb, w.colpy, sym, bnd, d.T, d.U, d.V, d.VP64(), d.ntb(), sm.a_ac, w.gq));
    RNNT_LAUNCH(KID_SMOOTH_Q, st, launch_pdl(smooth_q_kernel, (unsigned)(((long long)d.N * d.U1() + 7) / 8), 256, 0, st, 
        lm, w.lse_lm, w.gq, bnd, d.N, d.U, d.V, d.VP64(), w.Qu));
  }
  auto am_part = [&]() -> cudaError_t {
    cudaError_t e2 = cudaSuccess;
    if (am_grad) {
      Maps mp;
      if (!tm3(&mp.m[0], w.Gt_hi, d.UP(), d.T, d.N, sg::BM) || !tm3(&mp.m[1], w.Gt_lo, d.UP(), d.T, d.N, sg::BM) ||
          !tm3(&mp.m[2], w.Elm_hi, d.VP64(), d.U1(), d.N, 64) || !tm3(&mp.m[3], w.Elm_lo, d.VP64(), d.U1(), d.N, 64))
        return cudaErrorInvalidValue;
      const bool io = d.V % 4 == 0;
      if (io && (!make_tmap_f32_3d(&mp.ein, am, d.V, d.T, d.N, (uint64_t)d.V * 4, (uint64_t)d.V * d.T * 4, 32, sg::BM) ||
                 !make_tmap_f32_3d(&mp.eout, am_grad, d.V, d.T, d.N, (uint64_t)d.V * 4, (uint64_t)d.V * d.T * 4, 32,
                                   sg::BM)))
        return cudaErrorInvalidValue;
      AmProb p{am, w.m_am, w.rowb, bnd, d.T, d.U, d.V, gs, am_grad, io, sm, w.Lavg, w.lse_ac, w.rowy, d.VP64(), px_grad,
               sym};
      dim3 grid((d.T + sg::BM - 1) / sg::BM, (d.V + AmProb::kBN - 1) / AmProb::kBN, d.N);
      if ((e2 = launch_gemm3(p, grid, mp, KID_AMGRAD, st)) != cudaSuccess) return e2;
    }
    return e2;
  };
  auto lm_part = [&]() -> cudaError_t {
    cudaError_t e2 = cudaSuccess;
    if (lm_grad) {
      Maps mp;
      if (!tm3(&mp.m[0], w.Gt_hi, d.UP(), d.T, d.N, 64) || !tm3(&mp.m[1], w.Gt_lo, d.UP(), d.T, d.N, 64) ||
          !tm3(&mp.m[2], w.Eam_hi, d.VP64(), d.T, d.N, 64) || !tm3(&mp.m[3], w.Eam_lo, d.VP64(), d.T, d.N, 64))
        return cudaErrorInvalidValue;
      const bool io = d.V % 4 == 0;
      if (io && (!make_tmap_f32_3d(&mp.ein, lm, d.V, d.U1(), d.N, (uint64_t)d.V * 4, (uint64_t)d.V * d.U1() * 4, 32,
                                   sg::BM) ||
                 !make_tmap_f32_3d(&mp.eout, lm_grad, d.V, d.U1(), d.N, (uint64_t)d.V * 4, (uint64_t)d.V * d.U1() * 4,
                                   32, sg::BM)))
        return cudaErrorInvalidValue;
      LmProb p{lm, w.m_lm, w.colpy, w.colpb, sym, bnd, d.T, d.U, d.V, d.ntb(), gs, lm_grad, io, sm, w.lse_lm, w.gq, w.Qu,
               d.VP64()};
      dim3 grid((d.U1() + sg::BM - 1) / sg::BM, (d.V + LmProb::kBN - 1) / LmProb::kBN, d.N);
      if ((e2 = launch_gemm3(p, grid, mp, KID_LMGRAD, st)) != cudaSuccess) return e2;
    }
    return e2;
  };
  // order on the side stream: the (smaller) lm gradient first finishes while the bounds and the gather run,
  // so the joiner forward starts right after rowinfo instead of waiting for SMs (RNNT_LM_FIRST=0: am first)
  static const int lm_first = env_int("RNNT_LM_FIRST", 1);   // measured: c5 0.4259 vs 0.4343 ms
  if (lm_first) {
    if ((e = lm_part()) != cudaSuccess) return e;
    if ((e = am_part()) != cudaSuccess) return e;
  } else {
    if ((e = am_part()) != cudaSuccess) return e;
    if ((e = lm_part()) != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace rnnt
