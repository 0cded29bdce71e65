// simple.cu — stage 1: the trivial ("simple") joiner loss, its lattice
// recursion (Eq. 3) and occupancies, and the am/lm gradients.
//
// Kernels
//   K1 rowmax_kernel         m_am(t) = max_v am[t,v], m_lm(u) = max_v lm[u,v]  (offsets)
//   K2 NormGemm (SIMT v0)    S(t,u) = sum_v e^{am-m_am} e^{lm-m_lm}; epilogue writes the
//                            skewed lattice arcs px2/py2 (base 2) and 1/S  (Eq. 5-6, Eq. 1-2)
//   K3 alpha/beta            anti-diagonal wavefronts, fp64 state
//   K4 combine_kernel        y', empty', G~ = (y'+empty')/S, t-major outputs via smem transpose
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
    float px = neg_inf_f();
    if (u < Un) {
      long long y = sym[(size_t)n * U + u];
      y = y < 0 ? 0 : (y >= V ? V - 1 : y);      // address safety; bad symbols flagged in status
      px = a[y] + l[y] - Lnorm;                     // y(t,u) = L(t,u,y_{u+1})   Eq. 1 + Eq. 5
    }
    float py = a[0] + l[0] - Lnorm;                 // empty(t,u) = L(t,u,0)  Eq. 2 + Eq. 5
    size_t idx = ((size_t)n * (K + 1) + (t + u)) * LU + u;
    px2[idx] = px * RNNT_LOG2E_F;
    py2[idx] = py * RNNT_LOG2E_F;
    rS[idx] = 1.0f / S;
  }
};

// ------------------------------------------------------------------ K3 recursions
template <int R>
struct VecF {
  __device__ static void load(const float* p, float (&x)[R]) {
#pragma unroll
    for (int j = 0; j < R; ++j) x[j] = p[j];
  }
};
template <>
struct VecF<4> {
  __device__ static void load(const float* p, float (&x)[4]) {
    float4 a = *reinterpret_cast<const float4*>(p);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
  }
};
template <>
struct VecF<8> {
  __device__ static void load(const float* p, float (&x)[8]) {
    float4 a = *reinterpret_cast<const float4*>(p);
    float4 b = *reinterpret_cast<const float4*>(p + 4);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
    x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
  }
};

// alpha(t,u) = LogAdd(alpha(t-1,u)+empty(t-1,u), alpha(t,u-1)+y(t,u-1))  (Eq. 3), over
// anti-diagonals k = t+u.  Thread i owns columns u in [iR, iR+R); the only cross-thread
// dependency is the vertical arc into column iR (shfl / smem for the warp boundary).
// State carried between diagonals: h = alpha + empty (horizontal out-arc) and
// v = alpha + y (vertical out-arc) of the previous diagonal, fp64, base 2.
template <int R, int D>
__global__ void __launch_bounds__(256) lattice_alpha_kernel(
    const float* __restrict__ px2, const float* __restrict__ py2, const int64_t* __restrict__ bnd,
    int LU, int K, double* __restrict__ alpha, double* __restrict__ Ltot, float* __restrict__ loss,
    int32_t* __restrict__ status) {
  const int n = blockIdx.x;
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  const int Kn = Tn + Un;
  const size_t base = (size_t)n * (K + 1) * LU;
  const float* PX = px2 + base;
  const float* PY = py2 + base;
  double* A = alpha + base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int u0 = tid * R;
  const bool multi = blockDim.x > 32;
  const bool active = u0 < LU;
  __shared__ double sh_v[2][8];
  const double NI = neg_inf_d();

  double h[R], v[R];
#pragma unroll
  for (int j = 0; j < R; ++j) { h[j] = NI; v[j] = NI; }
  if (tid == 0) {
    A[0] = 0.0;                             // alpha(0,0) = 0
    h[0] = (double)PY[0];
    v[0] = Un > 0 ? (double)PX[0] : NI;
  }
  float bx[D][R], by[D][R];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    int k = 1 + d;
    if (active && k < Kn) { VecF<R>::load(PX + (size_t)k * LU + u0, bx[d]); VecF<R>::load(PY + (size_t)k * LU + u0, by[d]); }
  }
  if (multi) {
    if (lane == 31 && warp < 8) sh_v[0][warp] = v[R - 1];
    __syncthreads();
  }
  for (int kb = 1; kb < Kn; kb += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int k = kb + d;
      if (k < Kn) {
        double nb = __shfl_up_sync(0xffffffffu, v[R - 1], 1);
        if (lane == 0) nb = (warp == 0) ? NI : sh_v[(k - 1) & 1][warp - 1];
        double an[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int u = u0 + j, t = k - u;
          const bool valid = (t >= 0) && (t < Tn) && (u <= Un);
          const double below = (j == 0) ? nb : v[j - 1];
          const double a = logadd2_d(h[j], below);
          an[j] = valid ? a : NI;
        }
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int u = u0 + j, t = k - u;
          const bool valid = (t >= 0) && (t < Tn) && (u <= Un);
          h[j] = valid ? an[j] + (double)by[d][j] : NI;
          v[j] = (valid && u < Un) ? an[j] + (double)bx[d][j] : NI;
          if (active && valid) A[(size_t)k * LU + u] = an[j];
        }
        if (active && k + D < Kn) {
          VecF<R>::load(PX + (size_t)(k + D) * LU + u0, bx[d]);
          VecF<R>::load(PY + (size_t)(k + D) * LU + u0, by[d]);
        }
        if (multi) {
          if (lane == 31) sh_v[k & 1][warp] = v[R - 1];
          __syncthreads();
        }
      }
    }
  }
  // L_tot = alpha(T-1,U) + empty(T-1,U) = h at column U on the last diagonal.
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if (u0 + j == Un) {
      double L = h[j] * RNNT_LN2;
      Ltot[n] = L;
      loss[n] = (float)(-L);
      if (!isfinite(L)) set_status(status, n, kStatusNonFinite);
    }
  }
}

// beta(t,u) = LogAdd(beta(t+1,u)+empty(t,u), beta(t,u+1)+y(t,u)), beta(T-1,U) = empty(T-1,U):
// the backward half of the forward-backward algorithm.  Runs concurrently with alpha.
template <int R, int D>
__global__ void __launch_bounds__(256) lattice_beta_kernel(
    const float* __restrict__ px2, const float* __restrict__ py2, const int64_t* __restrict__ bnd,
    int LU, int K, double* __restrict__ beta) {
  const int n = blockIdx.x;
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  const int Kn = Tn + Un;
  const size_t base = (size_t)n * (K + 1) * LU;
  const float* PX = px2 + base;
  const float* PY = py2 + base;
  double* B = beta + base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int u0 = tid * R;
  const bool multi = blockDim.x > 32;
  const int nwarps = blockDim.x >> 5;
  const bool active = u0 < LU;
  __shared__ double sh_b[2][8];
  const double NI = neg_inf_d();

  double b[R];  // beta on diagonal k+1 (initially the virtual end node (T_n, U_n) = 0)
#pragma unroll
  for (int j = 0; j < R; ++j) b[j] = (u0 + j == Un) ? 0.0 : NI;
  float bx[D][R], by[D][R];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    int k = Kn - 1 - d;
    if (active && k >= 0) { VecF<R>::load(PX + (size_t)k * LU + u0, bx[d]); VecF<R>::load(PY + (size_t)k * LU + u0, by[d]); }
  }
  if (multi) {
    if (lane == 0) sh_b[0][warp] = b[0];
    __syncthreads();
  }
  int it = 0;
  for (int kb = Kn - 1; kb >= 0; kb -= D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int k = kb - d;
      if (k >= 0) {
        double nb = __shfl_down_sync(0xffffffffu, b[0], 1);
        if (lane == 31) nb = (warp == nwarps - 1) ? NI : sh_b[it & 1][warp + 1];
        double bn[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int u = u0 + j, t = k - u;
          const bool valid = (t >= 0) && (t < Tn) && (u <= Un);
          const double right = b[j] + (double)by[d][j];
          const double up = ((j == R - 1) ? nb : b[j + 1]) + (double)bx[d][j];
          const double r = logadd2_d(right, (u < Un) ? up : NI);
          bn[j] = valid ? r : NI;
        }
#pragma unroll
        for (int j = 0; j < R; ++j) {
          b[j] = bn[j];
          const int u = u0 + j, t = k - u;
          if (active && t >= 0 && t < Tn && u <= Un) B[(size_t)k * LU + u] = bn[j];
        }
        if (active && k - D >= 0) {
          VecF<R>::load(PX + (size_t)(k - D) * LU + u0, bx[d]);
          VecF<R>::load(PY + (size_t)(k - D) * LU + u0, by[d]);
        }
        ++it;
        if (multi) {
          if (lane == 0) sh_b[it & 1][warp] = b[0];
          __syncthreads();
        }
      }
    }
  }
}

// ------------------------------------------------------------------ K4 combine
// y'(t,u) = 2^(a + px2 + b(t,u+1) - L2), empty'(t,u) = 2^(a + py2 + b(t+1,u) - L2),
// terminal empty'(T-1,U) = 2^(a + py2 - L2).  Tile = 32 diagonals x 32 columns in skewed
// space, transposed through smem so the t-major outputs are written row-contiguously.
__global__ void __launch_bounds__(256) combine_kernel(
    const float* __restrict__ px2, const float* __restrict__ py2, const float* __restrict__ rS,
    const double* __restrict__ alpha, const double* __restrict__ beta, const double* __restrict__ Ltot,
    const int64_t* __restrict__ bnd, int T, int U, int LU, int K, float* __restrict__ px_grad,
    float* __restrict__ py_grad, float* __restrict__ Gt) {
  __shared__ float sy[32][33], sb[32][33], sg[32][33];
  const int n = blockIdx.z;
  const int k0 = blockIdx.x * 32, u0 = blockIdx.y * 32;
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t base = (size_t)n * (K + 1) * LU;
  const double L2 = Ltot[n] * RNNT_LOG2E;
  const bool finite = isfinite(L2);
  for (int kr = warp; kr < 32; kr += 8) {
    const int k = k0 + kr, u = u0 + lane, t = k - u;
    float yv = 0.f, bv = 0.f, g = 0.f;
    if (finite && t >= 0 && t < Tn && u <= Un) {
      const size_t i = base + (size_t)k * LU + u;
      const double a = alpha[i];
      if (u < Un) yv = ex2_approx((float)(a + (double)px2[i] + beta[i + LU + 1] - L2));
      if (t < Tn - 1) bv = ex2_approx((float)(a + (double)py2[i] + beta[i + LU] - L2));
      else if (u == Un) bv = ex2_approx((float)(a + (double)py2[i] - L2));
      g = (yv + bv) * rS[i];
    }
    sy[kr][lane] = yv;
    sb[kr][lane] = bv;
    sg[kr][lane] = g;
  }
  __syncthreads();
  const int t_base = k0 - u0 - 31;
  const int U1 = U + 1;
  for (int tr = warp; tr < 63; tr += 8) {
    const int t = t_base + tr, u = u0 + lane, kr = tr + lane - 31;
    if (kr >= 0 && kr < 32 && t >= 0 && t < T && u < U1) {
      const size_t o = ((size_t)n * T + t) * U1 + u;
      px_grad[o] = sy[kr][lane];
      py_grad[o] = sb[kr][lane];
      Gt[o] = sg[kr][lane];
    }
  }
}

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
static int pick_R(int LU) {
  // one warp when (U+1) <= 256, columns per lane R = next pow2 >= ceil(LU/32)
  int need = (LU + 31) / 32;
  if (need <= 1) return 1;
  if (need <= 2) return 2;
  if (need <= 4) return 4;
  return 8;
}

template <int R>
static cudaError_t launch_recursions(const Dims& d, const SimpleWS& w, const int64_t* bnd, float* loss,
                                     int32_t* status, cudaStream_t st) {
  const int LU = d.LU(), K = d.K();
  int threads = ((LU + R - 1) / R + 31) / 32 * 32;
  if (threads > 256) return cudaErrorInvalidConfiguration;
  RNNT_LAUNCH(KID_ALPHA, st, lattice_alpha_kernel<R, 4><<<d.N, threads, 0, st>>>(w.px2, w.py2, bnd, LU, K, w.alpha, w.Ltot, loss, status));
  RNNT_LAUNCH(KID_BETA, st, lattice_beta_kernel<R, 4><<<d.N, threads, 0, st>>>(w.px2, w.py2, bnd, LU, K, w.beta));
  return cudaGetLastError();
}

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
  {
    NormGemm p{am, lm, w.m_am, w.m_lm, sym, bnd, d.T, d.U, d.V, d.LU(), d.K(), w.px2, w.py2, w.rS, status};
    RNNT_LAUNCH(KID_NORM, st, e = launch_simt_gemm(p, d.T, d.U1(), d.N, st));
    if (e != cudaSuccess) return e;
  }
  {
    int R = pick_R(d.LU());
    if (R == 1) e = launch_recursions<1>(d, w, bnd, loss, status, st);
    else if (R == 2) e = launch_recursions<2>(d, w, bnd, loss, status, st);
    else if (R == 4) e = launch_recursions<4>(d, w, bnd, loss, status, st);
    else e = launch_recursions<8>(d, w, bnd, loss, status, st);
    if (e != cudaSuccess) return e;
  }
  {
    dim3 grid((d.K() + 31) / 32, (d.U1() + 31) / 32, d.N);
    RNNT_LAUNCH(KID_COMBINE, st, combine_kernel<<<grid, 256, 0, st>>>(w.px2, w.py2, w.rS, w.alpha, w.beta, w.Ltot, bnd, d.T, d.U,
                                         d.LU(), d.K(), px_grad, py_grad, w.Gt));
  }
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
