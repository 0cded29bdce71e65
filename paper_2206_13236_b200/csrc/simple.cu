// simple.cu — stage 1: the trivial ("simple") joiner loss, its lattice
// recursion (Eq. 3) and occupancies, and the am/lm gradients.
//
// Kernels
//   K1 rowmax_kernel         m_am(t) = max_v am[t,v], m_lm(u) = max_v lm[u,v]  (offsets)
//   K2 NormGemm (SIMT v0)    S(t,u) = sum_v e^{am-m_am} e^{lm-m_lm}; epilogue writes the
//                            skewed lattice arcs px2/py2 (base 2) and 1/S  (Eq. 5-6, Eq. 1-2)
//   K3/K4 (lattice.cu)       alpha || beta wavefronts on the skewed layout, occupancies, G~
//   K5 AmGrad/LmGrad + picks d(-L)/d am, d(-L)/d lm (chain rule through Eq. 5-6)
#include "common.cuh"
#include "gemm_simt.cuh"
#include "launch.h"
#include "workspace.h"

namespace rnnt {

// ------------------------------------------------------------------ validation
__global__ void validate_kernel(const int64_t* symbols, const int64_t* boundary, int N, int U, int V,
                                int32_t* status) {
  int n = blockIdx.x;
  int Un = utt_U(boundary, n);
  int bits = 0;
  if (threadIdx.x == 0 && (boundary[4 * n] != 0 || boundary[4 * n + 1] != 0)) bits |= kStatusBadBoundary;
  for (int u = threadIdx.x; u < Un && u < U; u += blockDim.x) {
    int64_t y = symbols[(size_t)n * U + u];
    if (y < 1 || y >= V) bits |= kStatusBadSymbol;
  }
  set_status(status, n, bits);
}

// ------------------------------------------------------------------ K1 row max
// One warp per row; padded rows get 0 (never read downstream).
__global__ void rowmax_kernel(const float* __restrict__ x, int N, int rows_per_n, int V,
                              const int64_t* __restrict__ boundary, int which /*0=am(T) 1=lm(U+1)*/,
                              float* __restrict__ m) {
  long long row = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (row >= (long long)N * rows_per_n) return;
  int n = (int)(row / rows_per_n), r = (int)(row % rows_per_n);
  int lim = which == 0 ? utt_T(boundary, n) : utt_U(boundary, n) + 1;
  if (r >= lim) {
    if (lane == 0) m[row] = 0.f;
    return;
  }
  const float* p = x + row * (long long)V;
  float mx = neg_inf_f();
  for (int v = lane; v < V; v += 32) mx = fmaxf(mx, p[v]);
  mx = warp_max(mx);
  if (lane == 0) m[row] = mx;
}

// ------------------------------------------------------------------ K2 (SIMT v0)
struct NormGemm {
  static constexpr bool kAMajorM = false, kBMajorN = false;
  const float *am, *lm, *m_am, *m_lm;
  const int64_t *sym, *bnd;
  int T, U, V, LU, K;
  float *px2, *py2, *rS;
  int32_t* status;
  __device__ bool tile_active(int n, int m0, int n0) const {
    return m0 < utt_T(bnd, n) && n0 <= utt_U(bnd, n);
  }
  __device__ void krange(int, int, int, long long& b, long long& e) const { b = 0; e = V; }
  __device__ float A(int n, int t, long long v) const {
    if (t >= utt_T(bnd, n)) return 0.f;
    size_t row = (size_t)n * T + t;
    return expf(am[row * V + v] - m_am[row]);
  }
  __device__ float B(int n, int u, long long v) const {
    if (u > utt_U(bnd, n)) return 0.f;
    size_t row = (size_t)n * (U + 1) + u;
    return expf(lm[row * V + v] - m_lm[row]);
  }
  __device__ void epi(int n, int t, int u, float S) const {
    int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
    if (t >= Tn || u > Un) return;
    size_t ra = (size_t)n * T + t, rl = (size_t)n * (U + 1) + u;
    if (!(S > 0.f)) set_status(status, n, kStatusUnderflow);
    float Lnorm = logf(S) + m_am[ra] + m_lm[rl];   // L_normalizer(t,u), Eq. 6
    const float* a = am + ra * V;
    const float* l = lm + rl * V;
    float px = kNegBig;                             // y(t,U) = -inf (sentinel, lattice.cu)
    if (u < Un) {
      long long y = sym[(size_t)n * U + u];
      y = y < 0 ? 0 : (y >= V ? V - 1 : y);      // address safety; bad symbols flagged in status
      px = (a[y] + l[y] - Lnorm) * RNNT_LOG2E_F;    // y(t,u) = L(t,u,y_{u+1})   Eq. 1 + Eq. 5
    }
    // empty(t,u) = L(t,u,0)  Eq. 2 + Eq. 5; out of the last frame only the terminal blank exists
    const float py = (t == Tn - 1 && u < Un) ? kNegBig : (a[0] + l[0] - Lnorm) * RNNT_LOG2E_F;
    size_t idx = ((size_t)n * (K + 1) + (t + u)) * LU + u;
    px2[idx] = px;
    py2[idx] = py;
    rS[idx] = 1.0f / S;
  }
};

// ------------------------------------------------------------------ K5 (SIMT v0)
// am_grad[t,v] = gs * (E_am[t,v] * sum_u G~[t,u] E_lm[u,v])   (picks subtracted after)
struct AmGradGemm {
  static constexpr bool kAMajorM = false, kBMajorN = true;
  const float *am, *lm, *m_am, *m_lm, *Gt;
  const int64_t* bnd;
  int T, U, V;
  float gs;
  float* am_grad;
  __device__ bool tile_active(int, int, int) const { return true; }
  __device__ void krange(int n, int, int, long long& b, long long& e) const { b = 0; e = utt_U(bnd, n) + 1; }
  __device__ float A(int n, int t, long long u) const {
    if (t >= utt_T(bnd, n)) return 0.f;
    return Gt[((size_t)n * T + t) * (U + 1) + u];
  }
  __device__ float B(int n, int v, long long u) const {
    if (v >= V) return 0.f;
    size_t row = (size_t)n * (U + 1) + u;
    return expf(lm[row * V + v] - m_lm[row]);
  }
  __device__ void epi(int n, int t, int v, float acc) const {
    if (t >= T || v >= V) return;
    size_t row = (size_t)n * T + t;
    float g = 0.f;
    if (t < utt_T(bnd, n)) g = gs * expf(am[row * V + v] - m_am[row]) * acc;
    am_grad[row * V + v] = g;
  }
};

struct LmGradGemm {
  static constexpr bool kAMajorM = true, kBMajorN = true;
  const float *am, *lm, *m_am, *m_lm, *Gt;
  const int64_t* bnd;
  int T, U, V;
  float gs;
  float* lm_grad;
  __device__ bool tile_active(int, int, int) const { return true; }
  __device__ void krange(int n, int, int, long long& b, long long& e) const { b = 0; e = utt_T(bnd, n); }
  __device__ float A(int n, int u, long long t) const {
    if (u > utt_U(bnd, n)) return 0.f;
    return Gt[((size_t)n * T + t) * (U + 1) + u];
  }
  __device__ float B(int n, int v, long long t) const {
    if (v >= V) return 0.f;
    size_t row = (size_t)n * T + t;
    return expf(am[row * V + v] - m_am[row]);
  }
  __device__ void epi(int n, int u, int v, float acc) const {
    if (u > U || v >= V) return;
    size_t row = (size_t)n * (U + 1) + u;
    float g = 0.f;
    if (u <= utt_U(bnd, n)) g = gs * expf(lm[row * V + v] - m_lm[row]) * acc;
    lm_grad[row * V + v] = g;
  }
};

// Label/blank picks: am_grad[t, y_{u+1}] -= gs*y'(t,u), am_grad[t,0] -= gs*sum_u empty'(t,u).
// One thread per frame, u ascending (deterministic, no atomics).
__global__ void am_picks_kernel(const float* __restrict__ px_grad, const float* __restrict__ py_grad,
                                const int64_t* __restrict__ sym, const int64_t* __restrict__ bnd,
                                int N, int T, int U, int V, float gs, float* __restrict__ am_grad) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)N * T) return;
  int n = (int)(i / T), t = (int)(i % T);
  int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  if (t >= Tn) return;
  const float* yr = px_grad + ((size_t)n * T + t) * (U + 1);
  const float* br = py_grad + ((size_t)n * T + t) * (U + 1);
  float* g = am_grad + ((size_t)n * T + t) * V;
  double sb = 0.0;
  for (int u = 0; u <= Un; ++u) sb += (double)br[u];
  g[0] = (float)((double)g[0] - (double)gs * sb);
  for (int u = 0; u < Un; ++u) {
    long long y = sym[(size_t)n * U + u];
    if (y < 1 || y >= V) continue;
    g[y] -= gs * yr[u];
  }
}

// lm_grad[u, y_{u+1}] -= gs*sum_t y'(t,u), lm_grad[u,0] -= gs*sum_t empty'(t,u).
__global__ void lm_picks_kernel(const float* __restrict__ px_grad, const float* __restrict__ py_grad,
                                const int64_t* __restrict__ sym, const int64_t* __restrict__ bnd,
                                int N, int T, int U, int V, float gs, float* __restrict__ lm_grad) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)N * (U + 1)) return;
  int n = (int)(i / (U + 1)), u = (int)(i % (U + 1));
  int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  if (u > Un) return;
  double sy = 0.0, sb = 0.0;
  for (int t = 0; t < Tn; ++t) {
    size_t o = ((size_t)n * T + t) * (U + 1) + u;
    sy += (double)px_grad[o];
    sb += (double)py_grad[o];
  }
  float* g = lm_grad + ((size_t)n * (U + 1) + u) * V;
  g[0] = (float)((double)g[0] - (double)gs * sb);
  if (u < Un) {
    long long y = sym[(size_t)n * U + u];
    if (y >= 1 && y < V) g[y] = (float)((double)g[y] - (double)gs * sy);
  }
}

// ------------------------------------------------------------------ host driver
cudaError_t skew_fill_launch(const Dims& d, const SimpleWS& w, const int64_t* bnd, cudaStream_t st);
cudaError_t lattice_launch(const Dims& d, const SimpleWS& w, const int64_t* bnd, float* loss, float* px_grad,
                           float* py_grad, int32_t* status, cudaStream_t st);

cudaError_t simple_loss_launch(const Dims& d, const SimpleWS& w, const float* am, const float* lm,
                               const int64_t* sym, const int64_t* bnd, float gs, float* loss,
                               float* px_grad, float* py_grad, float* am_grad, float* lm_grad,
                               int32_t* status, cudaStream_t st) {
  cudaError_t e;
  RNNT_LAUNCH(KID_VALIDATE, st, validate_kernel<<<d.N, 128, 0, st>>>(sym, bnd, d.N, d.U, d.V, status));
  {
    long long rows = (long long)d.N * d.T;
    RNNT_LAUNCH(KID_ROWMAX_AM, st, rowmax_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(am, d.N, d.T, d.V, bnd, 0, w.m_am));
    rows = (long long)d.N * d.U1();
    RNNT_LAUNCH(KID_ROWMAX_LM, st, rowmax_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(lm, d.N, d.U1(), d.V, bnd, 1, w.m_lm));
  }
  if ((e = skew_fill_launch(d, w, bnd, st)) != cudaSuccess) return e;
  {
    NormGemm p{am, lm, w.m_am, w.m_lm, sym, bnd, d.T, d.U, d.V, d.LU(), d.K(), w.px2, w.py2, w.rS, status};
    RNNT_LAUNCH(KID_NORM, st, e = launch_simt_gemm(p, d.T, d.U1(), d.N, st));
    if (e != cudaSuccess) return e;
  }
  if ((e = lattice_launch(d, w, bnd, loss, px_grad, py_grad, status, st)) != cudaSuccess) return e;
  if (am_grad) {
    AmGradGemm p{am, lm, w.m_am, w.m_lm, w.Gt, bnd, d.T, d.U, d.V, gs, am_grad};
    RNNT_LAUNCH(KID_AMGRAD, st, e = launch_simt_gemm(p, d.T, d.V, d.N, st));
    if (e != cudaSuccess) return e;
    long long rows = (long long)d.N * d.T;
    RNNT_LAUNCH(KID_AMPICK, st, am_picks_kernel<<<(unsigned)((rows + 127) / 128), 128, 0, st>>>(px_grad, py_grad, sym, bnd, d.N, d.T,
                                                                      d.U, d.V, gs, am_grad));
  }
  if (lm_grad) {
    LmGradGemm p{am, lm, w.m_am, w.m_lm, w.Gt, bnd, d.T, d.U, d.V, gs, lm_grad};
    RNNT_LAUNCH(KID_LMGRAD, st, e = launch_simt_gemm(p, d.U1(), d.V, d.N, st));
    if (e != cudaSuccess) return e;
    long long rows = (long long)d.N * d.U1();
    RNNT_LAUNCH(KID_LMPICK, st, lm_picks_kernel<<<(unsigned)((rows + 127) / 128), 128, 0, st>>>(px_grad, py_grad, sym, bnd, d.N, d.T,
                                                                      d.U, d.V, gs, lm_grad));
  }
  return cudaGetLastError();
}

}  // namespace rnnt
