// pruned.cu — stages 3-4: gather on the band, full joiner with fused
// log-softmax / pick / logit gradient (function merging), pruned recursion
// (P:253-256), joiner gradients.
//
// Kernels
//   K7  prune_kernel          h = bf16(tanh(enc[t] + dec[p_t+s])), masked rows 0
//   K7b rowinfo_kernel        per band row: label y_{u+1} (V at u=U_n), -1 if masked/padded
//   K8  ZGemm + softmax_rows  z = W h + b; lse, picks, P~ = bf16(exp(z - m_tile)), m_tile
//   K9  pruned_alpha/beta     banded wavefront, one lane per slot s, frames advance per lane
//   K9c pruned_combine        g_b = empty'_p, g_l = y'_p per row; sc = gs (g_b+g_l) e^{m_tile-lse}
//   K10 DhGemm + reduce       dpre = (W^T dz) (1-h^2); d_enc = sum_s dpre; d_dec gather-reduce
//   K11 DwGemm (split-K)      d_w = sum dz h^T, d_b = sum dz, deterministic split reduction
#include "common.cuh"
#include "launch.h"
#include "workspace.h"

namespace rnnt {

__device__ __forceinline__ float warp_max_uniform_p(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

cudaError_t joiner_fwd_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, const uint16_t* W,
                              const uint16_t* b, cudaStream_t st);
struct GradSrc {
  const uint16_t* Pt;
  const float4* gpk;
  const int32_t* rowinfo;
  long long R;
  int V, VP, ntile;
};
cudaError_t joiner_dh_launch(const Dims& d, const GradSrc& g, const uint16_t* h, const uint16_t* W,
                             const int32_t* ranges, const int2* urange, const int64_t* bnd, float* d_enc,
                             float* d_dec, float* part, cudaStream_t st);
cudaError_t joiner_dw_launch(const Dims& d, const GradSrc& g, const uint16_t* h, float* dWp, float* dbp,
                             int splits, cudaStream_t st);

// ------------------------------------------------------------------ K7 prune
// One CTA per frame (n, t); threads over (slot s, 8-column group) of its S band rows: 16 B of
// bf16 out per thread (enc[t] is read once per frame and reused from L1 across the S rows).
__global__ void __launch_bounds__(256) prune_kernel(const float* __restrict__ enc, const float* __restrict__ dec,
                                                    const int32_t* __restrict__ ranges, const int64_t* __restrict__ bnd,
                                                    int T, int U, int J, int S, uint16_t* __restrict__ h) {
  const int nt = blockIdx.x;
  const int n = nt / T, t = nt - n * T;
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  const int J8 = J / 8;
  const int p = t < Tn ? ranges[(size_t)n * T + t] : 0;
  const float* e = enc + (size_t)nt * J;
  for (int idx = threadIdx.x; idx < S * J8; idx += blockDim.x) {
    const int s = idx / J8, j0 = (idx - s * J8) * 8;
    const int u = p + s;
    uint4 out = make_uint4(0, 0, 0, 0);
    if (t < Tn && u <= Un) {
      const float* d = dec + ((size_t)n * (U + 1) + u) * J + j0;
      const float4 e0 = *reinterpret_cast<const float4*>(e + j0), e1 = *reinterpret_cast<const float4*>(e + j0 + 4);
      const float4 d0 = *reinterpret_cast<const float4*>(d), d1 = *reinterpret_cast<const float4*>(d + 4);
      const float x[8] = {e0.x + d0.x, e0.y + d0.y, e0.z + d0.z, e0.w + d0.w,
                          e1.x + d1.x, e1.y + d1.y, e1.z + d1.z, e1.w + d1.w};
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t lo = f_to_bf16_bits_rn(tanh_fast(x[2 * q]));
        const uint32_t hi = f_to_bf16_bits_rn(tanh_fast(x[2 * q + 1]));
        w[q] = lo | (hi << 16);
      }
      out = make_uint4(w[0], w[1], w[2], w[3]);
    }
    *reinterpret_cast<uint4*>(h + ((size_t)nt * S + s) * J + j0) = out;
  }
}

// blocks [0, nb_rows): per band row label info (and the frames covering each u); the last block
// pads the bias to fp32 (VP columns, zero beyond V) for the joiner epilogue.
__global__ void rowinfo_kernel(const int32_t* __restrict__ ranges, const int64_t* __restrict__ sym,
                               const int64_t* __restrict__ bnd, int N, int T, int U, int V, int S,
                               int32_t* __restrict__ rowinfo, int2* __restrict__ urange,
                               const uint16_t* __restrict__ bias_bf16, int VP, float* __restrict__ bias,
                               float* __restrict__ bmax, uint8_t* __restrict__ tlive, int* __restrict__ tcounter) {
  if (blockIdx.x == gridDim.x - 1) {
    if (threadIdx.x == 0) *tcounter = 0;
    for (int v = threadIdx.x; v < VP; v += blockDim.x) bias[v] = v < V ? bf16_bits_to_f(bias_bf16[v]) : 0.f;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int tl = warp; tl < VP / 128; tl += blockDim.x / 32) {   // bias max per 128-column tile
      float m = neg_inf_f();
      for (int j = lane; j < 128; j += 32)
        if (tl * 128 + j < V) m = fmaxf(m, bias[tl * 128 + j]);
      m = warp_max(m);
      if (lane == 0) bmax[tl] = m;
    }
    return;
  }
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long R = (long long)N * T * S;
  int info = -1;
  if (r < R) {
    const int s = (int)(r % S);
    const long long nt = r / S;
    const int t = (int)(nt % T), n = (int)(nt / T);
    const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
    const bool feasible = (long long)Un <= (long long)Tn * (S - 1);
    if (t < Tn && feasible) {
      const int32_t* p = ranges + (size_t)n * T;
      const int u = p[t] + s;
      if (u < Un) {
        long long y = sym[(size_t)n * U + u];
        info = (y >= 1 && y < V) ? (int)y : V;
      } else if (u == Un) {
        info = V;  // no label arc at u = U_n (y(t,U) = -inf)
      }
      if (s == 0) {
        // Frames covering token position u form the contiguous range [lo(u), hi(u)) (p monotone,
        // Eq. 9).  Frame t is the first cover of u in (p_{t-1}+S-1, p_t+S-1] and the last cover of
        // u in [p_t, p_{t+1}-1]; over t these intervals partition [0, U_n], so each entry is
        // written once.
        int2* ur = urange + (size_t)n * (U + 1);
        const int a0 = (t == 0) ? 0 : p[t - 1] + S;
        const int a1 = min(p[t] + S - 1, Un);
        for (int uu = a0; uu <= a1; ++uu) ur[uu].x = t;
        const int b1 = (t == Tn - 1) ? Un : p[t + 1] - 1;
        for (int uu = p[t]; uu <= b1; ++uu) ur[uu].y = t + 1;
      }
    }
    rowinfo[r] = info;
  }
  // 128-row tile liveness for the persistent joiner: a 256-thread block holds two whole tiles
  const bool live = info >= 0;
  const bool lo = __syncthreads_or(live && threadIdx.x < 128);
  const bool hi = __syncthreads_or(live && threadIdx.x >= 128);
  if (threadIdx.x == 0 && r < R) tlive[r / 128] = lo ? 1 : 0;
  if (threadIdx.x == 128 && r < R) tlive[r / 128] = hi ? 1 : 0;
}

// ------------------------------------------------------------------ K9 pruned recursion
// Eq. 3 on the band (Fig. 1b lattice).  grid (N, 2): y = 0 alpha, y = 1 beta.
// Lane s of warp 0 owns band slot s; it processes frame t at anti-diagonal k = d_t + s with
// d_t = t + p_t strictly increasing (Eq. 9), so both in-arcs of a cell were produced one step
// earlier: the vertical one by lane s-1 (same frame), the horizontal one by lane s + p_t - p_{t-1}
// (previous frame).  The state is fp32 rebased per anti-diagonal exactly as in lattice.cu
// (A_k = A_{k-2} + max of diagonal k-2, one CREDUX per step); shifts are kept in fp64.
// Arcs (px2 = y_p log2e, py2 = empty_p log2e; kNegBig off the lattice) and p_t are staged in smem.
__device__ __forceinline__ float plae2(float a, float b, float c) {
  const float m = fmaxf(a, b);
  return (m - c) + lg2_approx(1.0f + ex2_approx(-fabsf(a - b)));
}

// Per (anti-diagonal k, slot s) step record, built in a parallel prepass so that the wavefront
// loop only does value arithmetic: arcs {y, empty} and a code word
//   bits 0-15 frame t | 16-21 source lane + 1 of the frame-crossing arc (0: none) | flags below.
constexpr int kPfAct = 1 << 22, kPfMasked = 1 << 23, kPfFirst = 1 << 24, kPfLast = 1 << 25, kPfUeq = 1 << 26,
              kPfUlt = 1 << 27;

__global__ void __launch_bounds__(256) pruned_fb_kernel(
    const float* __restrict__ px2, const float* __restrict__ py2, const int32_t* __restrict__ ranges,
    const int64_t* __restrict__ bnd, int T, int S, int K, float* __restrict__ ap, float* __restrict__ bp,
    float* __restrict__ Aps, float* __restrict__ Bps, double* __restrict__ Lp, float* __restrict__ loss,
    int32_t* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = blockIdx.x;
  const bool fwd = blockIdx.y == 0;
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  const bool feasible = (long long)Un <= (long long)Tn * (S - 1);
  if (!feasible) {
    if (fwd && threadIdx.x == 0) {
      Lp[n] = neg_inf_d();
      loss[n] = __int_as_float(0x7f800000);  // +inf: no band-respecting path (kept visible, D16)
      set_status(status, n, kStatusInfeasible);
    }
    return;
  }
  const size_t rbase = (size_t)n * T * S;
  const int* pr = ranges + (size_t)n * T;
  const int dlast = (Tn - 1) + pr[Tn - 1];          // d_{T-1}
  const int kend = dlast + S - 1;                    // last anti-diagonal holding a band cell
  // smem: records [(kend+1) * S] {float2 arcs, int code}
  float2* rxy = reinterpret_cast<float2*>(smem_raw);
  int* rcode = reinterpret_cast<int*>(rxy + (size_t)(K + 1) * S);
  const int nrec = (kend + 1) * S;
  for (int i = threadIdx.x; i < nrec; i += blockDim.x) rcode[i] = 0;
  __syncthreads();
  for (int i0 = threadIdx.x; i0 < Tn * S; i0 += 4 * blockDim.x) {
    float x[4], y[4];
    int pp[4], pn[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {                 // all loads of the four entries first (MLP)
      const int i = i0 + q * blockDim.x;
      x[q] = 0.f; y[q] = 0.f; pp[q] = 0; pn[q] = 0;
      if (i < Tn * S) {
        const int t = i / S;
        x[q] = px2[rbase + i];
        y[q] = py2[rbase + i];
        pp[q] = pr[t];
        pn[q] = fwd ? (t > 0 ? pr[t - 1] : 0) : (t < Tn - 1 ? pr[t + 1] : 0);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + q * blockDim.x;
      if (i >= Tn * S) break;
      const int t = i / S, sl = i - t * S;
      const int p = pp[q], u = p + sl, k = t + p + sl;
      int src1 = 0;   // source lane + 1 of the arc crossing frames
      if (fwd) {
        if (t > 0) src1 = sl + p - pn[q] + 1;                          // (t-1, u) in frame t-1
      } else if (t < Tn - 1) {
        const int s2 = sl - (pn[q] - p);                               // (t+1, u) in frame t+1
        src1 = s2 >= 0 ? s2 + 1 : 0;
      }
      int code = t | (min(src1, 63) << 16) | kPfAct;
      if (u > Un) code |= kPfMasked;
      if (t == 0) code |= kPfFirst;
      if (t == Tn - 1) code |= kPfLast;
      if (u == Un) code |= kPfUeq;
      if (u < Un) code |= kPfUlt;
      rxy[k * S + sl] = make_float2(x[q], y[q]);
      rcode[k * S + sl] = code;
    }
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int s = threadIdx.x;
  const bool on = s < S;
  float* shift = (fwd ? Aps : Bps) + (size_t)n * (K + 1);
  float* outv = (fwd ? ap : bp) + rbase;
  const float NB = kNegBig;
  float Sh = 0.f;   // shift of the current diagonal: an integer, exact in fp32
  float Mm2 = 0.f, Mm1 = 0.f, cprev = 0.f;

  // Blocks of 8 diagonals: the records of the block are loaded up front, then 8 straight-line steps.
  constexpr int KB = 8;
  if (fwd) {
    float h_out = NB, v_out = NB;
    int k_loss = -1;
    float hl = NB;
    for (int kb = 0; kb <= kend; kb += KB) {
      int cd[KB];
      float2 xy[KB];
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        const int k = kb + j;
        const bool ok = on && k <= kend;
        cd[j] = ok ? rcode[k * S + s] : 0;
        xy[j] = ok ? rxy[k * S + s] : make_float2(NB, NB);
      }
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        const int k = kb + j, code = cd[j];
        const int src = ((code >> 16) & 63) - 1;
        // A_k = round(A_{k-2} + M_{k-2}); a diagonal with no live cell keeps A_k = A_{k-1}
        const float ci = (k >= 2 && Mm2 > -1e29f) ? rintf(Mm2 - cprev) : 0.f;
        const float hin = __shfl_sync(0xffffffffu, h_out, src >= 0 ? src : s);
        const float vin = __shfl_up_sync(0xffffffffu, v_out, 1);
        const float left = (src >= 0 && src < S) ? hin : NB;
        const float below = s > 0 ? vin : NB;
        float a = ((code & kPfFirst) && s == 0) ? -ci : plae2(left, below, ci);
        if (code & kPfMasked) a = NB;                      // masked slot (S > U_n + 1, D10)
        const bool act = (code & kPfAct) != 0;
        const float hn = a + xy[j].y, vn = a + xy[j].x;
        h_out = act ? hn : h_out;
        v_out = act ? vn : v_out;
        if (act) outv[(code & 0xffff) * S + s] = a;
        const float mx = act ? a : NB;
        const bool fin = act && (code & kPfLast) && (code & kPfUeq);
        k_loss = fin ? k : k_loss;
        hl = fin ? hn : hl;
        Sh += ci;
        if (s == 0 && k <= kend) shift[k] = Sh;
        if (k == k_loss && fin) {
          // L_pruned = alpha(T-1,U) + empty(T-1,U) (P:167-168 on the band), in the frame A_k
          const double L = ((double)hl + (double)Sh) * RNNT_LN2;
          Lp[n] = L;
          loss[n] = (float)(-L);
          if (!isfinite(L) || L < -1e20) set_status(status, n, kStatusNonFinite);
        }
        const float Mk = warp_max_uniform_p(mx);
        Mm2 = Mm1;
        Mm1 = Mk;
        cprev = ci;
      }
    }
  } else {
    float b_out = NB;
    for (int kb = kend; kb >= 0; kb -= KB) {
      int cd[KB];
      float2 xy[KB];
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        const int k = kb - j;
        const bool ok = on && k >= 0;
        cd[j] = ok ? rcode[k * S + s] : 0;
        xy[j] = ok ? rxy[k * S + s] : make_float2(NB, NB);
      }
#pragma unroll
      for (int j = 0; j < KB; ++j) {
        const int k = kb - j, i = kend - k, code = cd[j];
        const int src = ((code >> 16) & 63) - 1;
        const float ci = (i >= 2 && Mm2 > -1e29f) ? rintf(Mm2 - cprev) : 0.f;
        const float rin = __shfl_sync(0xffffffffu, b_out, src >= 0 ? src : s);
        const float uin = __shfl_down_sync(0xffffffffu, b_out, 1);
        float right;
        if (code & kPfLast) right = (code & kPfUeq) ? xy[j].y : NB;       // terminal blank (virtual end, beta = 0)
        else right = (src >= 0 && src < S) ? rin + xy[j].y : NB;
        const float up = ((code & kPfUlt) && s + 1 < S) ? uin + xy[j].x : NB;
        float b = plae2(right, up, ci);
        if (code & kPfMasked) b = NB;
        const bool act = (code & kPfAct) != 0;
        b_out = act ? b : b_out;
        if (act) outv[(code & 0xffff) * S + s] = b;
        const float mx = act ? b : NB;
        Sh += ci;
        if (s == 0 && k >= 0) shift[k] = Sh;
        const float Mk = warp_max_uniform_p(mx);
        Mm2 = Mm1;
        Mm1 = Mk;
        cprev = ci;
      }
    }
  }
}

// g_l = y'_p(t,u), g_b = empty'_p(t,u) for u = p_t + s (P:273-281 on the pruned lattice), and
// the per-(row, tile) softmax scale of the logit gradient sc = gs (g_b + g_l) exp(m_tile - lse).
__global__ void pruned_combine_kernel(const float* __restrict__ px2, const float* __restrict__ py2,
                                      const float* __restrict__ ap, const float* __restrict__ bp,
                                      const float* __restrict__ Aps, const float* __restrict__ Bps,
                                      const double* __restrict__ Lp, const int32_t* __restrict__ ranges,
                                      const int32_t* __restrict__ rowinfo, const float* __restrict__ mt,
                                      const float* __restrict__ lse, const int64_t* __restrict__ bnd,
                                      int N, int T, int S, int K, int ntile, float gs, float* __restrict__ gb,
                                      float* __restrict__ gl, float4* __restrict__ gpk) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long R = (long long)N * T * S;
  if (r >= R) return;
  const int s = (int)(r % S);
  const long long nt = r / S;
  const int t = (int)(nt % T), n = (int)(nt / T);
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  float yb = 0.f, bb = 0.f;
  const double L2 = Lp[n] * RNNT_LOG2E;
  const int info = rowinfo[r];
  if (info >= 0 && isfinite(L2)) {
    const int p = ranges[(size_t)n * T + t];
    const int u = p + s, k = t + u;
    const float* A = Aps + (size_t)n * (K + 1);
    const float* B = Bps + (size_t)n * (K + 1);
    const float a = ap[r];
    if (u < Un && s + 1 < S)
      yb = ex2_approx(a + px2[r] + bp[r + 1] + (float)((double)A[k] + (double)B[k + 1] - L2));
    if (t < Tn - 1) {
      const int s2 = u - ranges[(size_t)n * T + t + 1];
      if (s2 >= 0 && s2 < S) bb = ex2_approx(a + py2[r] + bp[r + S + (s2 - s)] + (float)((double)A[k] + (double)B[k + 1] - L2));
    } else if (u == Un) {
      bb = ex2_approx(a + py2[r] + (float)((double)A[k] - L2));
    }
  }
  gb[r] = bb;
  gl[r] = yb;
  // packed per (V tile, row) operand scalars of the joiner backward (joiner_bwd.cu):
  // {gs (g_b + g_l) exp(m_tile - lse), gs g_b, gs g_l, label}; dead rows {0, 0, 0, -1}
  const float l = lse[r];
  for (int tl = 0; tl < ntile; ++tl) {
    float4 q = make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
    if (info >= 0) q = make_float4(gs * (bb + yb) * expf(mt[r * ntile + tl] - l), gs * bb, gs * yb, __int_as_float(info));
    gpk[(size_t)tl * R + r] = q;
  }
}

__global__ void split_reduce_kernel(const float* __restrict__ part, int splits, long long M,
                                    float* __restrict__ out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  float acc = 0.f;
  for (int z = 0; z < splits; ++z) acc += part[(size_t)z * M + i];
  out[i] = acc;
}

// ------------------------------------------------------------------ host drivers
cudaError_t prune_launch(const Dims& d, const float* enc, const float* dec, const int32_t* ranges,
                         const int64_t* bnd, uint16_t* h, cudaStream_t st) {
  RNNT_LAUNCH(KID_PRUNE, st, prune_kernel<<<(unsigned)((long long)d.N * d.T), 256, 0, st>>>(enc, dec, ranges, bnd, d.T, d.U,
                                                                                      d.J, d.S, h));
  return cudaGetLastError();
}

size_t pruned_recursion_smem(const Dims& d) { return (size_t)(d.K() + 1) * d.S * 12; }

// Forward: per-row info, K8 joiner with fused log-softmax, K9 recursion, the occupancies and the
// packed backward scalars.
cudaError_t pruned_fwd_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, const uint16_t* W,
                              const uint16_t* b, const int64_t* sym, const int32_t* ranges, const int64_t* bnd,
                              float gs, float* loss, int32_t* status, cudaStream_t st) {
  cudaError_t e;
  const long long R = d.rows();
  const int nt = d.ntile();
  RNNT_LAUNCH(KID_ROWINFO, st, rowinfo_kernel<<<(unsigned)((R + 255) / 256 + 1), 256, 0, st>>>(
      ranges, sym, bnd, d.N, d.T, d.U, d.V, d.S, w.rowinfo, w.urange, b, d.VP(), w.bias, w.bmax, w.tlive, w.tcounter));
  if ((e = joiner_fwd_launch(d, w, h, W, b, st)) != cudaSuccess) return e;
  {
    const size_t sm = pruned_recursion_smem(d);
    cudaFuncSetAttribute(pruned_fb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    RNNT_LAUNCH(KID_PALPHA, st, pruned_fb_kernel<<<dim3(d.N, 2), 256, sm, st>>>(w.px2, w.py2, ranges, bnd, d.T, d.S, d.K(),
                                                                              w.ap, w.bp, w.Aps, w.Bps, w.Lp, loss,
                                                                              status));
  }
  RNNT_LAUNCH(KID_PCOMBINE, st, pruned_combine_kernel<<<(unsigned)((R + 255) / 256), 256, 0, st>>>(
      w.px2, w.py2, w.ap, w.bp, w.Aps, w.Bps, w.Lp, ranges, w.rowinfo, w.mt, w.lse, bnd, d.N, d.T, d.S, d.K(), nt,
      gs, w.gb, w.gl, w.gpk));
  return cudaGetLastError();
}

// Backward to the joiner input: K10 dh (and dpre), then d_enc / d_dec reductions.
cudaError_t pruned_bwd_input_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, const uint16_t* W,
                                    const int32_t* ranges, const int64_t* bnd, float* d_enc, float* d_dec,
                                    cudaStream_t st) {
  cudaError_t e;
  GradSrc g{w.Pt, w.gpk, w.rowinfo, d.rows(), d.V, d.VP(), d.ntile()};
  if (!d_enc && !d_dec) return cudaSuccess;
  if ((e = joiner_dh_launch(d, g, h, W, ranges, w.urange, bnd, d_enc, d_dec, w.dpart, st)) != cudaSuccess) return e;
  return cudaGetLastError();
}

// Backward to the joiner weights: K11 dW (split-K) + db, deterministic split reduction.
cudaError_t pruned_bwd_weight_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, float* d_w, float* d_b,
                                     cudaStream_t st) {
  cudaError_t e;
  GradSrc g{w.Pt, w.gpk, w.rowinfo, d.rows(), d.V, d.VP(), d.ntile()};
  if ((e = joiner_dw_launch(d, g, h, w.dWp, w.dbp, w.splits, st)) != cudaSuccess) return e;
  const long long M = (long long)d.V * d.J;
  RNNT_LAUNCH(KID_DW_REDUCE, st, split_reduce_kernel<<<(unsigned)((M + 255) / 256), 256, 0, st>>>(w.dWp, w.splits, M, d_w));
  RNNT_LAUNCH(KID_DB_REDUCE, st, split_reduce_kernel<<<(unsigned)((d.V + 255) / 256), 256, 0, st>>>(w.dbp, w.splits, d.V, d_b));
  return cudaGetLastError();
}

cudaError_t pruned_loss_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, const uint16_t* W,
                               const uint16_t* b, const int64_t* sym, const int32_t* ranges,
                               const int64_t* bnd, float gs, float* loss, float* d_enc, float* d_dec,
                               float* d_w, float* d_b, int32_t* status, cudaStream_t st) {
  cudaError_t e;
  if ((e = pruned_fwd_launch(d, w, h, W, b, sym, ranges, bnd, gs, loss, status, st)) != cudaSuccess) return e;
  if ((e = pruned_bwd_input_launch(d, w, h, W, ranges, bnd, d_enc, d_dec, st)) != cudaSuccess) return e;
  return pruned_bwd_weight_launch(d, w, h, d_w, d_b, st);
}

}  // namespace rnnt
