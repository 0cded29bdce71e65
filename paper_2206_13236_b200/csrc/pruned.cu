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

cudaError_t joiner_fwd_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, const uint16_t* W,
                              const uint16_t* b, cudaStream_t st);
struct GradSrc {
  const uint16_t* Pt;
  const float *sc, *gb, *gl;
  const int32_t* rowinfo;
  long long R;
  int V, VP, ntile;
  float gs;
};
cudaError_t joiner_dh_launch(const Dims& d, const GradSrc& g, const uint16_t* h, const uint16_t* W, float* dpre,
                             cudaStream_t st);
cudaError_t joiner_dw_launch(const Dims& d, const GradSrc& g, const uint16_t* h, float* dWp, float* dbp,
                             int splits, cudaStream_t st);

// ------------------------------------------------------------------ K7 prune
// One thread per 8 consecutive j of one band row (16 B of bf16 out).
__global__ void prune_kernel(const float* __restrict__ enc, const float* __restrict__ dec,
                             const int32_t* __restrict__ ranges, const int64_t* __restrict__ bnd,
                             int N, int T, int U, int J, int S, uint16_t* __restrict__ h) {
  const int J8 = J / 8;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long R = (long long)N * T * S;
  if (i >= R * J8) return;
  const long long r = i / J8;
  const int j0 = (int)(i % J8) * 8;
  const int s = (int)(r % S);
  const long long nt = r / S;
  const int t = (int)(nt % T), n = (int)(nt / T);
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  uint4 out = make_uint4(0, 0, 0, 0);
  if (t < Tn) {
    const int u = ranges[(size_t)n * T + t] + s;
    if (u <= Un) {
      const float* e = enc + ((size_t)n * T + t) * J + j0;
      const float* d = dec + ((size_t)n * (U + 1) + u) * J + j0;
      float4 e0 = *reinterpret_cast<const float4*>(e), e1 = *reinterpret_cast<const float4*>(e + 4);
      float4 d0 = *reinterpret_cast<const float4*>(d), d1 = *reinterpret_cast<const float4*>(d + 4);
      float x[8] = {e0.x + d0.x, e0.y + d0.y, e0.z + d0.z, e0.w + d0.w,
                    e1.x + d1.x, e1.y + d1.y, e1.z + d1.z, e1.w + d1.w};
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t lo = f_to_bf16_bits_rn(tanhf(x[2 * q]));
        uint32_t hi = f_to_bf16_bits_rn(tanhf(x[2 * q + 1]));
        w[q] = lo | (hi << 16);
      }
      out = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  *reinterpret_cast<uint4*>(h + r * J + j0) = out;
}

__global__ void rowinfo_kernel(const int32_t* __restrict__ ranges, const int64_t* __restrict__ sym,
                               const int64_t* __restrict__ bnd, int N, int T, int U, int V, int S,
                               int32_t* __restrict__ rowinfo) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (long long)N * T * S) return;
  const int s = (int)(r % S);
  const long long nt = r / S;
  const int t = (int)(nt % T), n = (int)(nt / T);
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  int info = -1;
  if (t < Tn && (long long)Un <= (long long)Tn * (S - 1)) {
    const int u = ranges[(size_t)n * T + t] + s;
    if (u < Un) {
      long long y = sym[(size_t)n * U + u];
      info = (y >= 1 && y < V) ? (int)y : V;
    } else if (u == Un) {
      info = V;  // no label arc at u = U_n (y(t,U) = -inf)
    }
  }
  rowinfo[r] = info;
}

// ------------------------------------------------------------------ K9 pruned recursion
// Lane s of one warp handles band slot s; it processes frame t at step d_t + s with
// d_t = t + p_t (strictly increasing), i.e. the anti-diagonal of node (t, p_t + s).
// Vertical in-arc from lane s-1 (same frame), horizontal in-arc from lane s + (p_t - p_{t-1})
// (previous frame, same u); both produced exactly one step earlier.
__global__ void __launch_bounds__(128) pruned_alpha_kernel(
    const float* __restrict__ px2, const float* __restrict__ py2, const int32_t* __restrict__ ranges,
    const int64_t* __restrict__ bnd, int T, int S, double* __restrict__ ap, double* __restrict__ Lp,
    float* __restrict__ loss, int32_t* __restrict__ status) {
  extern __shared__ unsigned char smem_raw[];
  const int n = blockIdx.x;
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  int* sp = reinterpret_cast<int*>(smem_raw);
  float* sx = reinterpret_cast<float*>(sp + T);
  float* sy = sx + (size_t)T * S;
  const bool feasible = (long long)Un <= (long long)Tn * (S - 1);
  if (!feasible) {
    if (threadIdx.x == 0) {
      Lp[n] = neg_inf_d();
      loss[n] = __int_as_float(0x7f800000);  // +inf: no band-respecting path (kept visible)
      set_status(status, n, kStatusInfeasible);
    }
    return;
  }
  const size_t rbase = (size_t)n * T * S;
  for (int i = threadIdx.x; i < Tn; i += blockDim.x) sp[i] = ranges[(size_t)n * T + i];
  for (int i = threadIdx.x; i < Tn * S; i += blockDim.x) { sx[i] = px2[rbase + i]; sy[i] = py2[rbase + i]; }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int s = threadIdx.x;
  const double NI = neg_inf_d();
  double h_out = NI, v_out = NI;
  int ts = 0;
  const int kend = (Tn - 1) + sp[Tn - 1] + S - 1;
  for (int k = 0; k <= kend; ++k) {
    const bool act = (s < S) && (ts < Tn) && (ts + sp[ts] + s == k);
    const int t = ts;
    const int p = act ? sp[t] : 0;
    const int src = act && t > 0 ? s + p - sp[t - 1] : s;
    const double hin = __shfl_sync(0xffffffffu, h_out, src < 32 ? src : 31);
    const double vin = __shfl_up_sync(0xffffffffu, v_out, 1);
    if (act) {
      const double left = (t > 0 && src < S) ? hin : NI;
      const double below = s > 0 ? vin : NI;
      const int u = p + s;
      double a = (t == 0 && s == 0) ? 0.0 : logadd2_d(left, below);
      const bool valid = u <= Un;
      if (!valid) a = NI;
      const float px = sx[t * S + s], py = sy[t * S + s];
      h_out = valid ? a + (double)py : NI;
      v_out = (valid && u < Un) ? a + (double)px : NI;
      ap[rbase + (size_t)t * S + s] = a;
      if (t == Tn - 1 && u == Un) {
        const double L = h_out * RNNT_LN2;
        Lp[n] = L;
        loss[n] = (float)(-L);
        if (!isfinite(L)) set_status(status, n, kStatusNonFinite);
      }
      ++ts;
    }
  }
}

// beta in reverse diagonal order: beta(t,u) = LogAdd(beta(t+1,u)+empty(t,u), beta(t,u+1)+y(t,u)).
__global__ void __launch_bounds__(128) pruned_beta_kernel(
    const float* __restrict__ px2, const float* __restrict__ py2, const int32_t* __restrict__ ranges,
    const int64_t* __restrict__ bnd, int T, int S, double* __restrict__ bp) {
  extern __shared__ unsigned char smem_raw[];
  const int n = blockIdx.x;
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  if ((long long)Un > (long long)Tn * (S - 1)) return;
  int* sp = reinterpret_cast<int*>(smem_raw);
  float* sx = reinterpret_cast<float*>(sp + T);
  float* sy = sx + (size_t)T * S;
  const size_t rbase = (size_t)n * T * S;
  for (int i = threadIdx.x; i < Tn; i += blockDim.x) sp[i] = ranges[(size_t)n * T + i];
  for (int i = threadIdx.x; i < Tn * S; i += blockDim.x) { sx[i] = px2[rbase + i]; sy[i] = py2[rbase + i]; }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int s = threadIdx.x;
  const double NI = neg_inf_d();
  double b_out = NI;
  int ts = Tn - 1;
  const int kend = (Tn - 1) + sp[Tn - 1] + S - 1;
  for (int k = kend; k >= 0; --k) {
    const bool act = (s < S) && (ts >= 0) && (ts + sp[ts] + s == k);
    const int t = ts;
    const int p = act ? sp[t] : 0;
    const int src = (act && t < Tn - 1) ? s - (sp[t + 1] - p) : s;   // slot of (t+1, u) in frame t+1
    const double rin = __shfl_sync(0xffffffffu, b_out, src >= 0 ? src : 0);
    const double uin = __shfl_down_sync(0xffffffffu, b_out, 1);
    if (act) {
      const int u = p + s;
      const bool valid = u <= Un;
      const float px = sx[t * S + s], py = sy[t * S + s];
      double right;
      if (t == Tn - 1) right = (u == Un) ? (double)py : NI;          // terminal blank
      else right = (src >= 0 && src < S) ? rin + (double)py : NI;
      const double up = (u < Un && s + 1 < S) ? uin + (double)px : NI;
      double b = logadd2_d(right, up);
      if (!valid) b = NI;
      b_out = b;
      bp[rbase + (size_t)t * S + s] = b;
      --ts;
    }
  }
}

// g_l = y'_p(t,u), g_b = empty'_p(t,u) for u = p_t + s (P:273-281 on the pruned lattice), and
// the per-(row, tile) softmax scale of the logit gradient.
__global__ void pruned_combine_kernel(const float* __restrict__ px2, const float* __restrict__ py2,
                                      const double* __restrict__ ap, const double* __restrict__ bp,
                                      const double* __restrict__ Lp, const int32_t* __restrict__ ranges,
                                      const int32_t* __restrict__ rowinfo, const float* __restrict__ mt,
                                      const float* __restrict__ lse, const int64_t* __restrict__ bnd,
                                      int N, int T, int S, int ntile, float gs, float* __restrict__ gb,
                                      float* __restrict__ gl, float* __restrict__ sc) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (long long)N * T * S) return;
  const int s = (int)(r % S);
  const long long nt = r / S;
  const int t = (int)(nt % T), n = (int)(nt / T);
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  float yb = 0.f, bb = 0.f;
  const double L2 = Lp[n] * RNNT_LOG2E;
  if (rowinfo[r] >= 0 && isfinite(L2)) {
    const int p = ranges[(size_t)n * T + t];
    const int u = p + s;
    const double a = ap[r];
    if (u < Un && s + 1 < S) yb = ex2_approx((float)(a + (double)px2[r] + bp[r + 1] - L2));
    if (t < Tn - 1) {
      const int s2 = u - ranges[(size_t)n * T + t + 1];
      if (s2 >= 0 && s2 < S) bb = ex2_approx((float)(a + (double)py2[r] + bp[r + S + (s2 - s)] - L2));
    } else if (u == Un) {
      bb = ex2_approx((float)(a + (double)py2[r] - L2));
    }
  }
  gb[r] = bb;
  gl[r] = yb;
  const float l = lse[r];
  for (int tl = 0; tl < ntile; ++tl)
    sc[r * ntile + tl] = (rowinfo[r] >= 0) ? gs * (bb + yb) * expf(mt[r * ntile + tl] - l) : 0.f;
}

// d_enc[n,t,:] = sum_s dpre[n,t,s,:];  d_dec[n,u,:] = sum_{t: p_t <= u < p_t+S} dpre[n,t,u-p_t,:]
// (frames covering u form a contiguous range since p is monotone; summed in t order).
__global__ void denc_kernel(const float* __restrict__ dpre, const int64_t* __restrict__ bnd, int N, int T,
                            int S, int J, float* __restrict__ d_enc) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)N * T * J) return;
  const int j = (int)(i % J);
  const long long nt = i / J;
  const int t = (int)(nt % T), n = (int)(nt / T);
  float acc = 0.f;
  if (t < utt_T(bnd, n))
    for (int s = 0; s < S; ++s) acc += dpre[(nt * S + s) * J + j];
  d_enc[i] = acc;
}

__global__ void ddec_kernel(const float* __restrict__ dpre, const int32_t* __restrict__ ranges,
                            const int64_t* __restrict__ bnd, int N, int T, int U, int S, int J,
                            float* __restrict__ d_dec) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)N * (U + 1) * J) return;
  const int j = (int)(i % J);
  const long long nu = i / J;
  const int u = (int)(nu % (U + 1)), n = (int)(nu / (U + 1));
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  float acc = 0.f;
  if (u <= Un && (long long)Un <= (long long)Tn * (S - 1)) {
    const int32_t* p = ranges + (size_t)n * T;
    // first t with p_t + S - 1 >= u
    int lo = 0, hi = Tn;
    while (lo < hi) { int m = (lo + hi) >> 1; if (p[m] + S - 1 >= u) hi = m; else lo = m + 1; }
    for (int t = lo; t < Tn && p[t] <= u; ++t)
      acc += dpre[(((size_t)n * T + t) * S + (u - p[t])) * J + j];
  }
  d_dec[i] = acc;
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
  long long work = d.rows() * (d.J / 8);
  RNNT_LAUNCH(KID_PRUNE, st, prune_kernel<<<(unsigned)((work + 255) / 256), 256, 0, st>>>(enc, dec, ranges, bnd, d.N, d.T, d.U, d.J,
                                                                 d.S, h));
  return cudaGetLastError();
}

size_t pruned_recursion_smem(const Dims& d) { return (size_t)d.T * 4 + (size_t)d.T * d.S * 8; }

cudaError_t pruned_loss_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, const uint16_t* W,
                               const uint16_t* b, const int64_t* sym, const int32_t* ranges,
                               const int64_t* bnd, float gs, float* loss, float* d_enc, float* d_dec,
                               float* d_w, float* d_b, int32_t* status, cudaStream_t st) {
  cudaError_t e;
  const long long R = d.rows();
  const int nt = d.ntile();
  RNNT_LAUNCH(KID_ROWINFO, st, rowinfo_kernel<<<(unsigned)((R + 255) / 256), 256, 0, st>>>(ranges, sym, bnd, d.N, d.T, d.U, d.V, d.S,
                                                               w.rowinfo));
  if ((e = joiner_fwd_launch(d, w, h, W, b, st)) != cudaSuccess) return e;
  {
    size_t sm = pruned_recursion_smem(d);
    cudaFuncSetAttribute(pruned_alpha_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(pruned_beta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    RNNT_LAUNCH(KID_PALPHA, st, pruned_alpha_kernel<<<d.N, 128, sm, st>>>(w.px2, w.py2, ranges, bnd, d.T, d.S, w.ap, w.Lp, loss, status));
    RNNT_LAUNCH(KID_PBETA, st, pruned_beta_kernel<<<d.N, 128, sm, st>>>(w.px2, w.py2, ranges, bnd, d.T, d.S, w.bp));
  }
  RNNT_LAUNCH(KID_PCOMBINE, st, pruned_combine_kernel<<<(unsigned)((R + 255) / 256), 256, 0, st>>>(
      w.px2, w.py2, w.ap, w.bp, w.Lp, ranges, w.rowinfo, w.mt, w.lse, bnd, d.N, d.T, d.S, nt, gs, w.gb,
      w.gl, w.sc));
  GradSrc g{w.Pt, w.sc, w.gb, w.gl, w.rowinfo, R, d.V, d.VP(), nt, gs};
  if (d_enc || d_dec) {
    if ((e = joiner_dh_launch(d, g, h, W, w.dpre, st)) != cudaSuccess) return e;
    if (d_enc) {
      long long n = (long long)d.N * d.T * d.J;
      RNNT_LAUNCH(KID_DENC, st, denc_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(w.dpre, bnd, d.N, d.T, d.S, d.J, d_enc));
    }
    if (d_dec) {
      long long n = (long long)d.N * d.U1() * d.J;
      RNNT_LAUNCH(KID_DDEC, st, ddec_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(w.dpre, ranges, bnd, d.N, d.T, d.U, d.S, d.J,
                                                               d_dec));
    }
  }
  {
    if ((e = joiner_dw_launch(d, g, h, w.dWp, w.dbp, w.splits, st)) != cudaSuccess) return e;
    long long M = (long long)d.V * d.J;
    RNNT_LAUNCH(KID_DW_REDUCE, st, split_reduce_kernel<<<(unsigned)((M + 255) / 256), 256, 0, st>>>(w.dWp, w.splits, M, d_w));
    RNNT_LAUNCH(KID_DB_REDUCE, st, split_reduce_kernel<<<(unsigned)((d.V + 255) / 256), 256, 0, st>>>(w.dbp, w.splits, d.V, d_b));
  }
  return cudaGetLastError();
}

}  // namespace rnnt
