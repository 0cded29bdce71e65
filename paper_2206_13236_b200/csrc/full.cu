// full.cu — SURVEY 8(f) f4: the full (unpruned) transducer loss with the non-linear joiner on the
// GPU, the comparison class of the paper's Tables 1-2, built from
// the pruned path's kernels with the band widened to every token position (S = U+1, all p_t = 0):
//   prune_kernel              h = bf16(tanh(enc[t] + dec[u])) for every (t, u)         (N,T,U+1,J)
//   rowinfo + joiner_fwd      z = W h + b, log-softmax, picks, P~ (function merging)
//   full_scatter_kernel       the joiner arcs into the simple lattice's skewed layout
//   lattice_fb + combine      alpha || beta on the (T, U+1) lattice (Eq. 3), occupancies
//   full_pack_kernel          per (V tile, row) logit-gradient scalars from the occupancies
//   joiner_dw (+ reduce)      dW, db
//   joiner_dh (generic mode)  dpre = (dz W) (1 - h^2) per row, then full_dgrad_kernel: d_enc, d_dec
// The memory is (N,T,U+1,J) for h and (N,T,U+1,V) bf16 for P~: the cost the pruned loss avoids.
#include <algorithm>

#include "common.cuh"
#include "launch.h"
#include "workspace.h"

namespace rnnt {

struct GradSrc {
  const uint16_t* Pt;
  const float4* gpk;
  const int32_t* rowinfo;
  long long R;
  int V, VP, ntile;
};
cudaError_t prune_launch(const Dims& d, const float* enc, const float* dec, const int32_t* ranges,
                         const int64_t* bnd, uint16_t* h, cudaStream_t st);
cudaError_t joiner_fwd_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, const uint16_t* W,
                              const uint16_t* b, cudaStream_t st);
cudaError_t lattice_launch(const Dims& d, const SimpleWS& w, const int64_t* bnd, float* loss, float* px_grad,
                           float* py_grad, int32_t* status, cudaStream_t st);
cudaError_t pruned_bwd_weight_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, float* d_w, float* d_b,
                                     cudaStream_t st, int mode);
cudaError_t joiner_dh_launch(const Dims& d, const GradSrc& g, const uint16_t* h, const uint16_t* W, const int* live,
                             const int* nlive, long long ntiles, float* dpre, const int* tscale, const float* gsp,
                             cudaStream_t st);
cudaError_t rowinfo_launch(const Dims& d, const PrunedWS& w, const int32_t* ranges, const int64_t* sym,
                           const int64_t* bnd, const uint16_t* b, float gs, cudaStream_t st);

// skewed arcs pxy[n][k][u] = {y(t,u), empty(t,u)} (log2e), t = k - u; the lattice conventions of
// lattice.cu: kNegBig off the lattice, y = kNegBig at u = U_n (already so in px2), and out of the
// last frame only the terminal blank
__global__ void __launch_bounds__(256) full_scatter_kernel(const float* __restrict__ px2, const float* __restrict__ py2,
                                                           const int64_t* __restrict__ bnd, int T, int U, int K, int LU,
                                                           float2* __restrict__ pxy) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  const int n = blockIdx.y;
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  const long long cells = (long long)(K + 1) * LU;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < cells; i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i / LU), u = (int)(i - (long long)k * LU);
    const int t = k - u;
    float2 v = make_float2(kNegBig, kNegBig);
    if (t >= 0 && t < Tn && u <= Un) {
      const size_t r = ((size_t)n * T + t) * (U + 1) + u;
      v.x = px2[r];
      v.y = (t == Tn - 1 && u < Un) ? kNegBig : py2[r];
    }
    pxy[(size_t)n * cells + i] = v;
  }
}

// {gs (g_b + g_l) exp(m_tile - lse), gs g_b, gs g_l, label} per (V tile, row) from the occupancies
// g_b = empty'(t,u), g_l = y'(t,u) (t-major = row order); dead rows {0, 0, 0, -1}
__global__ void full_pack_kernel(const float* __restrict__ gb, const float* __restrict__ gl,
                                 const int32_t* __restrict__ rowinfo, const float* __restrict__ mt,
                                 const float* __restrict__ lse, long long R, int ntile, float gs,
                                 float4* __restrict__ gpk) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int info = rowinfo[r];
  const float b = gb[r], y = gl[r], l = lse[r];
  for (int tl = 0; tl < ntile; ++tl) {
    float4 q = make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
    if (info >= 0) q = make_float4(gs * (b + y) * expf(mt[r * ntile + tl] - l), gs * b, gs * y, __int_as_float(info));
    gpk[(size_t)tl * R + r] = q;
  }
}

// blocks [0, N T): d_enc[n,t,:] = sum_{u <= U_n} dpre[(n,t,u),:];  blocks [N T, N T + N (U+1)):
// d_dec[n,u,:] = sum_{t < T_n} dpre[(n,t,u),:]; padded positions 0.  One thread per 4 columns.
__global__ void __launch_bounds__(128) full_dgrad_kernel(const float* __restrict__ dpre, const int64_t* __restrict__ bnd,
                                                         int N, int T, int U, int J, float* __restrict__ d_enc,
                                                         float* __restrict__ d_dec) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  const long long b = blockIdx.x;
  const long long NT = (long long)N * T;
  const int J4 = J / 4;
  if (b < NT) {
    if (!d_enc) return;
    const int n = (int)(b / T), t = (int)(b - (long long)n * T);
    const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
    for (int q = threadIdx.x; q < J4; q += blockDim.x) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t < Tn)
        for (int u = 0; u <= Un; ++u) {
          const float4 x = reinterpret_cast<const float4*>(dpre + (((size_t)n * T + t) * (U + 1) + u) * J)[q];
          a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
        }
      reinterpret_cast<float4*>(d_enc + (size_t)b * J)[q] = a;
    }
  } else {
    if (!d_dec) return;
    const long long nu = b - NT;
    const int n = (int)(nu / (U + 1)), u = (int)(nu - (long long)n * (U + 1));
    const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
    for (int q = threadIdx.x; q < J4; q += blockDim.x) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      if (u <= Un)
        for (int t = 0; t < Tn; ++t) {
          const float4 x = reinterpret_cast<const float4*>(dpre + (((size_t)n * T + t) * (U + 1) + u) * J)[q];
          a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
        }
      reinterpret_cast<float4*>(d_dec + (size_t)nu * J)[q] = a;
    }
  }
}

cudaError_t full_loss_launch(const Dims& d, void* base, const float* enc, const float* dec, const uint16_t* W,
                             const uint16_t* b, const int64_t* sym, const int64_t* bnd, float gs, float* loss,
                             float* d_enc, float* d_dec, float* d_w, float* d_b, int32_t* status, cudaStream_t st) {
  Dims df = d;
  df.S = d.U + 1;
  SimpleWS sw;
  PrunedWS pw;
  FullWS fw;
  carve_full(df, base, &sw, &pw, &fw);
  cudaError_t e;
  const long long R = df.rows();
  cudaMemsetAsync(fw.ranges0, 0, (size_t)df.N * df.T * 4, st);
  cudaMemsetAsync(sw.rS, 0, (size_t)df.N * (df.K() + 1) * df.LU() * 4, st);   // only feeds the unused G~
  if ((e = prune_launch(df, enc, dec, fw.ranges0, bnd, fw.h, st)) != cudaSuccess) return e;
  if ((e = rowinfo_launch(df, pw, fw.ranges0, sym, bnd, b, gs, st)) != cudaSuccess) return e;
  const long long ntiles = (R + 127) / 128;
  if ((e = joiner_fwd_launch(df, pw, fw.h, W, b, st)) != cudaSuccess) return e;
  {
    const long long cells = (long long)(df.K() + 1) * df.LU();
    const unsigned gx = (unsigned)std::min<long long>((cells + 255) / 256, 1024);
    RNNT_LAUNCH(KID_FULL_SCATTER, st, launch_pdl(full_scatter_kernel, dim3(gx, df.N), 256, 0, st, 
        pw.px2, pw.py2, bnd, df.T, df.U, df.K(), df.LU(), sw.pxy));
  }
  // occupancies straight into the row-ordered g_l (= y') and g_b (= empty') arrays
  if ((e = lattice_launch(df, sw, bnd, loss, pw.gl, pw.gb, status, st)) != cudaSuccess) return e;
  RNNT_LAUNCH(KID_FULL_PACK, st, launch_pdl(full_pack_kernel, (unsigned)((R + 255) / 256), 256, 0, st, 
      pw.gb, pw.gl, pw.rowinfo, pw.mt, pw.lse, R, df.ntile(), gs, pw.gpk));
  if ((e = pruned_bwd_weight_launch(df, pw, fw.h, d_w, d_b, st, 0)) != cudaSuccess) return e;
  if (d_enc || d_dec) {
    GradSrc g{pw.Pt, pw.gpk, pw.rowinfo, R, df.V, df.VP(), df.ntile()};
    if ((e = joiner_dh_launch(df, g, fw.h, W, pw.dhlive, pw.dhlive + ntiles, ntiles, fw.dpre, nullptr, nullptr, st)) != cudaSuccess)
      return e;
    RNNT_LAUNCH(KID_FULL_DGRAD, st, launch_pdl(full_dgrad_kernel, (unsigned)((long long)df.N * df.T + (long long)df.N * df.U1()), 128, 0, st, 
        fw.dpre, bnd, df.N, df.T, df.U, df.J, d_enc, d_dec));
  }
  return cudaGetLastError();
}

}  // namespace rnnt
