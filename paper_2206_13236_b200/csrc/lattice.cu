// lattice.cu — K3/K4: forward-backward on the simple (trivial-joiner) lattice.
//
//   alpha(t,u) = LogAdd(alpha(t-1,u) + empty(t-1,u), alpha(t,u-1) + y(t,u-1))   (Eq. 3-4)
//   beta(t,u)  = LogAdd(beta(t+1,u) + empty(t,u),   beta(t,u+1) + y(t,u))      (backward half)
//   y'(t,u) = exp(alpha + y + beta(t,u+1) - L), empty'(t,u) = exp(alpha + empty + beta(t+1,u) - L)
//                                                                              (occupancies)
// on the SKEWED (diagonal-major) layout [n][k = t+u][u] written by the normaliser epilogue, so that
// every wavefront step reads one contiguous row of arcs.  Conventions of the arc arrays (base 2):
//   pxy = {y, empty} * log2e (y = kNegBig at u = U_n; empty = kNegBig at t = T_n-1, u < U_n:
//   the only blank out of the last frame is the terminal one), kNegBig at every invalid cell.
// With these sentinels neither recursion needs a validity mask: the virtual node (T_n, U_n) on
// diagonal K_n = T_n + U_n receives alpha(T-1,U) + empty(T-1,U) = L_tot, and beta starts
// from it (beta = 0 there).
//
// Precision (D9): the state is fp32 REBASED per diagonal, alpha-hat_k = alpha_k - A_k, with
// A_k = max_u alpha_{k-2} rounded to an integer (the max of the diagonal two steps back, from one
// CREDUX.MAX per step, off the critical path), so the shifts accumulate exactly in fp32; |alpha-hat| stays within a two-step drift of 0
// where the mass is, so the fp32 rounding is ~1e-7 relative per step.  The occupancies are then
// self-normalised per anti-diagonal (every path leaves every diagonal k < K_n exactly once, so the
// outflow of a diagonal sums to 1), which removes the error common to a diagonal.
//
// Kernels
//   (the sentinels of the invalid skewed cells are written by simple_prep_kernel, simple_tc.cu)
//   lattice_fb_kernel   grid (N, 2): y = 0 alpha, y = 1 beta, concurrently.  Warp 1 streams the arc
//                       rows into a 4-stage shared-memory ring with cp.async.bulk (mbarrier
//                       complete_tx); warp 0 runs the wavefront, lane i owning columns [iR, iR+R)
//                       (one shuffle per diagonal for the arc crossing a lane boundary).
//   combine_kernel      per 32-diagonal block: outflow sums Z_k, then y', empty' / Z_k and
//                       G~ = (y' + empty') / S(t,u), transposed through smem to the t-major outputs.
#include <algorithm>

#include "common.cuh"
#include "launch.h"
#include "tc.cuh"
#include "workspace.h"

namespace rnnt {

namespace lat {
constexpr int NST = 6;   // arc-ring stages
constexpr int NX = 8;    // boundary-exchange chunk slots (>= NST + 1: no overwrite before consumption)
constexpr int MAXW = 4;  // strips (warps) per direction
// arc rows (diagonals) per staged chunk; the ring holds NST x 2 arrays x C rows x LU floats
template <int R>
constexpr int CH = R <= 2 ? 16 : (R == 4 ? 8 : 4);
struct Xchg {            // boundary values between neighbouring strips, per inbox warp
  float v[MAXW][NX][16];
  float s[MAXW][NX][16];
};
template <int R>
inline size_t smem_bytes(int W) {
  return (size_t)NST * 2 * CH<R> * 32 * R * W * sizeof(float) + sizeof(Xchg);
}
}  // namespace lat

// ------------------------------------------------------------------ wavefront
// log2(2^a + 2^b) for finite (sentinel-safe) a, b; minus the rebasing increment c.
__device__ __forceinline__ float lae2(float a, float b, float c) {
  const float m = fmaxf(a, b);
  const float e = ex2_approx(-fabsf(a - b));
  return (m - c) + lg2_approx(1.0f + e);
}

template <int R>
__device__ __forceinline__ void lds_row(const float* p, float (&x)[R]) {
  if constexpr (R % 4 == 0) {
#pragma unroll
    for (int j = 0; j < R; j += 4) {
      const float4 q = *reinterpret_cast<const float4*>(p + j);
      x[j] = q.x; x[j + 1] = q.y; x[j + 2] = q.z; x[j + 3] = q.w;
    }
  } else if constexpr (R % 2 == 0) {
#pragma unroll
    for (int j = 0; j < R; j += 2) {
      const float2 q = *reinterpret_cast<const float2*>(p + j);
      x[j] = q.x; x[j + 1] = q.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < R; ++j) x[j] = p[j];
  }
}

// R interleaved {px, py} pairs of this lane's columns
template <int R>
__device__ __forceinline__ void lds_pairs(const float* p, float (&px)[R], float (&py)[R]) {
  if constexpr (R % 2 == 0) {
#pragma unroll
    for (int j = 0; j < R; j += 2) {
      const float4 q = *reinterpret_cast<const float4*>(p + 2 * j);
      px[j] = q.x; py[j] = q.y; px[j + 1] = q.z; py[j + 1] = q.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const float2 q = *reinterpret_cast<const float2*>(p + 2 * j);
      px[j] = q.x; py[j] = q.y;
    }
  }
}

template <int R>
__device__ __forceinline__ void stg_row(float* p, const float (&x)[R]) {
  if constexpr (R % 4 == 0) {
#pragma unroll
    for (int j = 0; j < R; j += 4) *reinterpret_cast<float4*>(p + j) = make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]);
  } else if constexpr (R % 2 == 0) {
#pragma unroll
    for (int j = 0; j < R; j += 2) *reinterpret_cast<float2*>(p + j) = make_float2(x[j], x[j + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < R; ++j) p[j] = x[j];
  }
}

__device__ __forceinline__ float warp_max_uniform(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

// One direction of the wavefront for strip (warp) w of Wn active strips.
// FWD: alpha over diagonals 0 -> Kn (strips pipelined left to right); else beta over Kn -> 0
// (right to left).  Strip w lags its upstream neighbour by one chunk: the neighbour's boundary
// arc for every step of chunk c (with its fp64 shift) sits in the inbox before w starts chunk c.
// R, W and the chunk length C are compile-time so that a full chunk is straight-line code with
// immediate smem / global offsets (the per-step chain is then LogAdd + one shuffle, ~85 cycles).
template <int R, int W, bool FWD>
struct Wavefront {
  static constexpr int C = lat::CH<R>;
  static constexpr int LU = 32 * R * W;
  static constexpr size_t STAGE = (size_t)2 * C * LU;

  float a[R];
  float S = 0.f;                    // this strip's shift of the current diagonal (an integer, exact in fp32)
  float Mm2 = 0.f, Mm1 = 0.f;       // strip max of diagonals i-2, i-1 (relative to their shifts)
  float cprev = 0.f;                // rebasing increment of diagonal i-1
  int lane, w;
  bool has_in, has_out;

  // Step i of the chunk: arcs at `rx`, boundary inbox/outbox slot `xs`, outputs at `orow` (row
  // pointer of this lane's columns) and `oshift`.
  __device__ __forceinline__ void step(const float* rx, int i, const float* xv_in, const float* xs_in, float* xv_out,
                                       float* xs_out, float* orow, float* oshift) {
    float px[R], py[R];
    lds_pairs<R>(rx, px, py);
    float xin = kNegBig;
    if (has_in && lane == (FWD ? 0 : 31)) xin = *xv_in + (*xs_in - S);   // shifts are integers: exact
    // A_i = round(A_{i-2} + M_{i-2}); a strip with no live cell two diagonals back keeps A_i = A_{i-1}
    const float ci = (i >= 2 && Mm2 > -1e29f) ? rintf(Mm2 - cprev) : 0.f;
    float nw[R];
    if constexpr (FWD) {
      float h[R], v[R];
#pragma unroll
      for (int q = 0; q < R; ++q) { h[q] = a[q] + py[q]; v[q] = a[q] + px[q]; }
      if (has_out && lane == 31) { *xv_out = v[R - 1]; *xs_out = S; }
      float nb = __shfl_up_sync(0xffffffffu, v[R - 1], 1);
      if (lane == 0) nb = xin;
#pragma unroll
      for (int q = R - 1; q >= 1; --q) nw[q] = lae2(h[q], v[q - 1], ci);
      nw[0] = lae2(h[0], nb, ci);
    } else {
      if (has_out && lane == 0) { *xv_out = a[0]; *xs_out = S; }
      float nb = __shfl_down_sync(0xffffffffu, a[0], 1);
      if (lane == 31) nb = xin;
#pragma unroll
      for (int q = 0; q < R - 1; ++q) nw[q] = lae2(a[q] + py[q], a[q + 1] + px[q], ci);
      nw[R - 1] = lae2(a[R - 1] + py[R - 1], nb + px[R - 1], ci);
    }
    float mx = nw[0];
#pragma unroll
    for (int q = 0; q < R; ++q) { a[q] = nw[q]; mx = fmaxf(mx, nw[q]); }
    stg_row<R>(orow, a);
    S += ci;
    if (lane == 0) *oshift = S;
    const float Mi = warp_max_uniform(mx);
    Mm2 = Mm1;
    Mm1 = Mi;
    cprev = ci;
  }

  __device__ __forceinline__ void run(const float* ring, uint64_t* full, uint64_t* empty, uint64_t* xbar,
                                      lat::Xchg* xc, int w_, int Wn, int Kn, int Un, float* out, float* shift,
                                      double* Ltot_n, float* loss_n, int32_t* status, int n) {
    using namespace lat;
    lane = threadIdx.x & 31;
    w = w_;
    const int u0 = 32 * R * w + lane * R;
    has_in = FWD ? (w > 0) : (w < Wn - 1);
    has_out = FWD ? (w < Wn - 1) : (w > 0);
    const int inbox = w, outbox = FWD ? w + 1 : w - 1;
    const int start_u = FWD ? 0 : Un;
#pragma unroll
    for (int q = 0; q < R; ++q) a[q] = (u0 + q == start_u) ? 0.f : kNegBig;
    stg_row<R>(out + (size_t)(FWD ? 0 : Kn) * LU + u0, a);
    if (lane == 0) shift[(size_t)(FWD ? 0 : Kn) * W + w] = 0.f;

    constexpr int DR = FWD ? 1 : -1;     // output row direction
    int stage = 0, done = 0;
    uint32_t phase = 0;
    for (int c = 0; done < Kn; ++c) {
      const int rows = (Kn - done < C) ? Kn - done : C;
      tc::mbar_wait(&full[stage], phase);
      if (has_in) tc::mbar_wait(&xbar[inbox * NX + c % NX], (c / NX) & 1);
      const float* rb = ring + stage * STAGE + 2 * u0;
      const int slot = c % NX;
      const float* xvi = &xc->v[inbox][slot][0];
      const float* xsi = &xc->s[inbox][slot][0];
      float* xvo = &xc->v[outbox < 0 ? 0 : (outbox >= MAXW ? MAXW - 1 : outbox)][slot][0];
      float* xso = &xc->s[outbox < 0 ? 0 : (outbox >= MAXW ? MAXW - 1 : outbox)][slot][0];
      const int orow0 = FWD ? done + 1 : Kn - done - 1;
      float* ob = out + (size_t)orow0 * LU + u0;
      float* osb = shift + (size_t)orow0 * W + w;
      if (rows == C) {
#pragma unroll
        for (int j = 0; j < C; ++j)
          step(rb + (FWD ? j : C - 1 - j) * 2 * LU, done + j + 1, xvi + j, xsi + j, xvo + j, xso + j,
               ob + DR * j * LU, osb + DR * j * W);
      } else {
#pragma unroll 1
        for (int j = 0; j < rows; ++j)
          step(rb + (FWD ? j : rows - 1 - j) * 2 * LU, done + j + 1, xvi + j, xsi + j, xvo + j, xso + j,
               ob + DR * j * LU, osb + DR * j * W);
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&empty[stage]);
      if (has_out && lane == (FWD ? 31 : 0)) tc::mbar_arrive(&xbar[outbox * NX + slot]);
      if (++stage == NST) { stage = 0; phase ^= 1; }
      done += rows;
    }
    if constexpr (FWD) {
      // L_tot = alpha at the virtual node (T_n, U_n) = alpha(T-1,U) + empty(T-1,U)
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (u0 + q == Un) {
          const double L = ((double)a[q] + (double)S) * RNNT_LN2;
          *Ltot_n = L;
          *loss_n = (float)(-L);
          if (!isfinite(L) || L < -1e20) set_status(status, n, kStatusNonFinite);
        }
      }
    }
  }
};

// grid (N, 2): y = 0 alpha, y = 1 beta.  Warps 0..W-1: strips; warp W: bulk-copy loader.
template <int R, int W>
__global__ void __launch_bounds__(32 * (W + 1), 1) lattice_fb_kernel(
    const float2* __restrict__ pxy, const int64_t* __restrict__ bnd, int K,
    float* __restrict__ ahat, float* __restrict__ bhat, float* __restrict__ Ash, float* __restrict__ Bsh,
    double* __restrict__ Ltot, float* __restrict__ loss, int32_t* __restrict__ status) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  using namespace lat;
  constexpr int C = CH<R>, LU = 32 * R * W;
  extern __shared__ __align__(128) float ring[];
  __shared__ __align__(8) uint64_t full[NST], empty[NST], xbar[MAXW * NX];
  const int n = blockIdx.x;
  const bool fwd = blockIdx.y == 0;
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n), Kn = Tn + Un;
  const int Wn = (Un + 1 + 32 * R - 1) / (32 * R);          // strips holding a column <= U_n
  const size_t base = (size_t)n * (K + 1) * LU;
  const size_t sbase = (size_t)n * (K + 1) * W;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Xchg* xc = reinterpret_cast<Xchg*>(ring + (size_t)NST * 2 * C * LU);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], Wn); }
    for (int s = 0; s < MAXW * NX; ++s) tc::mbar_init(&xbar[s], 1);
    tc::fence_barrier_init();
  }
  __syncthreads();

  if (warp == W) {
    // ---- loader: arc rows in consumption order (alpha ascending, beta descending)
    if (lane == 0) {
      const int nch = (Kn + C - 1) / C;
      int s = 0;
      uint32_t ph = 0;
      for (int c = 0; c < nch; ++c) {
        tc::mbar_wait(&empty[s], ph ^ 1);
        int r0, r1;
        if (fwd) { r0 = c * C; r1 = min(Kn, r0 + C); }
        else { r1 = Kn - c * C; r0 = max(0, r1 - C); }
        const uint32_t bytes = (uint32_t)(r1 - r0) * LU * 8u;
        tc::mbar_arrive_expect_tx(&full[s], bytes);
        float* dx = ring + (size_t)s * 2 * C * LU;
        tc::bulk_load(dx, pxy + base + (size_t)r0 * LU, bytes, &full[s]);
        if (++s == NST) { s = 0; ph ^= 1; }
      }
    }
    return;
  }
  if (warp >= Wn) return;   // strip entirely beyond U_n: never holds a lattice cell
  if (fwd) {
    Wavefront<R, W, true> wf;
    wf.run(ring, full, empty, xbar, xc, warp, Wn, Kn, Un, ahat + base, Ash + sbase, Ltot + n, loss + n, status, n);
  } else {
    Wavefront<R, W, false> wf;
    wf.run(ring, full, empty, xbar, xc, warp, Wn, Kn, Un, bhat + base, Bsh + sbase, Ltot + n, loss + n, status, n);
  }
}

// ------------------------------------------------------------------ K4 combine
// Per block of 32 anti-diagonals (dynamic smem: the block's raw outflows Y, B and G [32][UP]):
//   phase A: raw y', empty' and (y' + empty')/S of every cell of the 32 diagonals (one pass over
//            alpha, beta, the arcs and 1/S, all skewed: every warp load is a contiguous row segment,
//            all loads of a diagonal issued before any use) and the diagonal sums Z_k (P:279-281:
//            the outflow of a diagonal sums to 1);
//   phase B: the normalised values written t-major (shared memory only): px_grad, py_grad, G~ and
//            y' as bf16 hi + lo; the cells of row t in this block are the contiguous columns u = k - t.
constexpr int kCombineZeroBlocks = 4; // zero-padding blocks per utterance (a warp per frame row)
constexpr int kCombineWindow = 512;   // staged columns per pass (3 x 32 x 512 fp32 = 192 KB)
__global__ void __launch_bounds__(256) combine_kernel(
    const float2* __restrict__ pxy, const float* __restrict__ rS,
    const float* __restrict__ ahat, const float* __restrict__ bhat, const float* __restrict__ Ash,
    const float* __restrict__ Bsh, const double* __restrict__ Ltot, const int64_t* __restrict__ bnd, int T,
    int U, int LU, int K, int W, int SW, int UP, float* __restrict__ px_grad, float* __restrict__ py_grad,
    uint16_t* __restrict__ Gt_hi, uint16_t* __restrict__ Gt_lo) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  extern __shared__ __align__(16) float cbuf[];
  const int CWs = min(UP, kCombineWindow);
  float* Ys = cbuf;                     // [32][CW]
  float* Bs = cbuf + 32 * CWs;          // [32][CW]
  float* Gs = cbuf + 64 * CWs;          // [32][CW]
  // per diagonal and strip: ob = A^w_k + B^w_{k+1} - L (blank arc, same column), ox = A^w_k +
  // B^{w+1}_{k+1} - L (label arc out of the strip's last column into the next strip)
  __shared__ float s_ob[32][lat::MAXW], s_ox[32][lat::MAXW], s_rz[32];
  const int n = blockIdx.y;
  const int k0 = blockIdx.x * 32;
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n), Kn = Tn + Un;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t base = (size_t)n * (K + 1) * LU;
  const size_t sbase = (size_t)n * (K + 1) * W;
  const double L2 = Ltot[n] * RNNT_LOG2E;
  const bool finite = isfinite(L2);
  const int U1 = U + 1;
  const int nd = (T + UP - 1 + 31) / 32;     // diagonal blocks; blocks nd.. of the row zero the padding
  if ((int)blockIdx.x >= nd) {
    // The padded cells of the t-major outputs (frames t >= T_n, columns u > U_n; everything of a non-finite
    // utterance) are exact zeros written here, a warp per frame row, so that the diagonal blocks touch only
    // lattice cells: as part of their phase B the padding was two thirds of the cell slots at c5 and made
    // the issue-bound kernel ~2x longer.
    const int Tv = finite ? Tn : 0;
    const int nz = gridDim.x - nd;
    for (int t = ((int)blockIdx.x - nd) * 8 + warp; t < T; t += 8 * nz) {
      const int c_lo = t < Tv ? Un + 1 : 0;
      const size_t o = ((size_t)n * T + t) * U1, og = ((size_t)n * T + t) * UP;
      for (int u = c_lo + lane; u < U1; u += 32) { px_grad[o + u] = 0.f; py_grad[o + u] = 0.f; }
      for (int u = c_lo + lane; u < UP; u += 32) { Gt_hi[og + u] = 0; Gt_lo[og + u] = 0; }
    }
    return;
  }
  if (!finite || k0 >= Kn) return;           // no lattice cell on these diagonals
  const int lsw = 31 - __clz(SW);
  if (threadIdx.x < 32 * lat::MAXW) {
    const int kr = threadIdx.x / lat::MAXW, w = threadIdx.x % lat::MAXW;
    const int k = k0 + kr;
    if (finite && k < Kn && w < W) {
      const double A = (double)Ash[sbase + (size_t)k * W + w];
      s_ob[kr][w] = (float)(A + (double)Bsh[sbase + (size_t)(k + 1) * W + w] - L2);
      s_ox[kr][w] = (w + 1 < W) ? (float)(A + (double)Bsh[sbase + (size_t)(k + 1) * W + w + 1] - L2) : 0.f;
    }
  }
  __syncthreads();

  // phase A: one warp per diagonal of the block; the row is read in groups of four 32-column chunks.
  // Rows wider than the staging window CW (U + 1 > CW) take two passes: the diagonal sums first, then
  // per column window the normalised values recomputed, staged and written (phase B).
  constexpr int CG = 4;
  const int CW = min(UP, kCombineWindow);
  const bool one = UP <= CW;
  auto cell = [&](int kr, int u, float a, float2 xy, float b0, float b1, float r, float& yv, float& bv, float& gv) {
    const int k = k0 + kr;
    const int ulo = max(0, k - Tn + 1), uhi = min(k, Un);
    yv = 0.f; bv = 0.f;
    if (u >= ulo && u <= uhi) {
      const int w = u >> lsw;                 // SW = 32 R is a power of two
      bv = ex2_approx(a + xy.y + b0 + s_ob[kr][w]);
      if (u < Un) yv = ex2_approx(a + xy.x + b1 + (((u & (SW - 1)) == SW - 1) ? s_ox[kr][w] : s_ob[kr][w]));
    }
    gv = (yv + bv) * r;
  };
  // values of diagonal kr for columns [u0, u0 + 32 CG) of the window starting at c0 (stage: write to smem)
  auto diag_pass = [&](int kr, int ub, int ue, int c0, bool stage) -> float {
    const int k = k0 + kr;
    const bool live = finite && k < Kn;
    const int ulo = live ? max(0, k - Tn + 1) : 1, uhi = live ? min(k, Un) : 0;
    const float* Ar = ahat + base + (size_t)k * LU;
    const float* Br = bhat + base + (size_t)(k + 1) * LU;
    const float2* XY = pxy + base + (size_t)k * LU;
    const float* Rr = rS + base + (size_t)k * LU;
    float z = 0.f;
    // only the 32-column groups holding a cell of the diagonal (about a third of the staged width at c5):
    // the staged values of every other column are never read (phase B masks by validity)
    const int ua = max(ub, ulo & ~31), uz = min(ue, uhi + 1);
    for (int u0 = ua; u0 < uz; u0 += 32 * CG) {
      float a[CG], b0[CG], b1[CG], r[CG];
      float2 xy[CG];
#pragma unroll
      for (int i = 0; i < CG; ++i) {          // every load of the group first
        const int u = u0 + 32 * i + lane;
        if (u0 + 32 * i > uhi) break;         // (warp-uniform: no cell of the diagonal in this chunk or later ones)
        const bool v = u >= ulo && u <= uhi && u < ue;
        a[i] = v ? Ar[u] : 0.f;
        xy[i] = v ? XY[u] : make_float2(0.f, 0.f);
        b0[i] = v ? Br[u] : 0.f;
        b1[i] = (v && u < Un) ? Br[u + 1] : 0.f;
        r[i] = v ? Rr[u] : 0.f;
      }
#pragma unroll
      for (int i = 0; i < CG; ++i) {
        const int u = u0 + 32 * i + lane;
        if (u >= ue || u0 + 32 * i > uhi) break;   // (staged values of chunks without a cell are never read)
        float yv = 0.f, bv = 0.f, gv = 0.f;
        if (live) cell(kr, u, a[i], xy[i], b0[i], b1[i], r[i], yv, bv, gv);
        if (stage) {
          Ys[kr * CW + (u - c0)] = yv;
          Bs[kr * CW + (u - c0)] = bv;
          Gs[kr * CW + (u - c0)] = gv;
        }
        z += yv + bv;
      }
    }
    return z;
  };
  for (int kr = warp; kr < 32; kr += 8) {
    const int k = k0 + kr;
    const bool live = finite && k < Kn;
    float z = diag_pass(kr, 0, UP, 0, one);
    z = warp_sum(z);
    if (lane == 0) s_rz[kr] = (live && z > 0.f && isfinite(z)) ? 1.0f / z : 0.f;
  }
  __syncthreads();

  for (int c0 = 0; c0 < UP; c0 += CW) {
    const int c1 = min(UP, c0 + CW);
    if (!one) {
      for (int kr = warp; kr < 32; kr += 8) diag_pass(kr, c0, c1, c0, true);
      __syncthreads();
    }
    // phase B: rows t with a cell of the window in the block: columns u = k0 + kr - t in [c0, c1)
    // (rows with a lattice cell of the window only: u = k0 + kr - t in [c0, min(c1 - 1, U_n)], t < T_n)
    const int tlo = max(0, k0 - min(c1 - 1, Un)), thi = min(Tn - 1, k0 + 31 - c0);
    for (int t = tlo + warp; t <= thi; t += 8) {
      const int kr = lane, u = k0 + kr - t;
      if (u < c0 || u >= c1 || u > Un) continue;        // (the padding is zeroed by the blocks nd..)
      const float rz = s_rz[kr];
      const float yv = Ys[kr * CW + (u - c0)] * rz, bv = Bs[kr * CW + (u - c0)] * rz;
      {
        const size_t o = ((size_t)n * T + t) * U1 + u;
        px_grad[o] = yv;
        py_grad[o] = bv;
      }
      // G~ = (y' + empty') / S for the am/lm gradient contractions: bf16 hi + lo, t-major, pitch UP
      const size_t og = ((size_t)n * T + t) * UP + u;
      const float g = Gs[kr * CW + (u - c0)] * rz;
      const __nv_bfloat16 gh = __float2bfloat16_rn(g);
      const __nv_bfloat16 gl = __float2bfloat16_rn(g - __bfloat162float(gh));
      Gt_hi[og] = *reinterpret_cast<const uint16_t*>(&gh);
      Gt_lo[og] = *reinterpret_cast<const uint16_t*>(&gl);
    }
    if (!one) __syncthreads();
  }
}

// ------------------------------------------------------------------ host
template <int R, int W>
static cudaError_t launch_fb(const Dims& d, const SimpleWS& w, const int64_t* bnd, float* loss, int32_t* status,
                             cudaStream_t st) {
  const size_t sm = lat::smem_bytes<R>(W);
  cudaFuncSetAttribute(lattice_fb_kernel<R, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  RNNT_LAUNCH(KID_ALPHA, st, launch_pdl(lattice_fb_kernel<R, W>, dim3(d.N, 2), 32 * (W + 1), sm, st, 
      w.pxy, bnd, d.K(), w.alpha, w.beta, w.Ash, w.Bsh, w.Ltot, loss, status));
  return cudaGetLastError();
}

template <int R>
static cudaError_t launch_fb_w(const Dims& d, const SimpleWS& w, const int64_t* bnd, float* loss, int32_t* status,
                               cudaStream_t st) {
  switch (d.lat_W()) {
    case 1: return launch_fb<R, 1>(d, w, bnd, loss, status, st);
    case 2: return launch_fb<R, 2>(d, w, bnd, loss, status, st);
    case 3: return launch_fb<R, 3>(d, w, bnd, loss, status, st);
    case 4: return launch_fb<R, 4>(d, w, bnd, loss, status, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t lattice_launch(const Dims& d, const SimpleWS& w, const int64_t* bnd, float* loss, float* px_grad,
                           float* py_grad, int32_t* status, cudaStream_t st) {
  cudaError_t e;
  switch (d.lat_R()) {
    case 1: e = launch_fb_w<1>(d, w, bnd, loss, status, st); break;
    case 2: e = launch_fb_w<2>(d, w, bnd, loss, status, st); break;
    case 4: e = launch_fb_w<4>(d, w, bnd, loss, status, st); break;
    case 8: e = launch_fb_w<8>(d, w, bnd, loss, status, st); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  // diagonal blocks write the lattice cells of the t-major outputs; kCombineZeroBlocks more blocks per
  // utterance their zero padding (frames t >= T_n, columns (U_n, UP) of G~ / (U_n, U] of the occupancies)
  dim3 grid((d.T + d.UP() - 1 + 31) / 32 + kCombineZeroBlocks, d.N);
  const size_t csm = (size_t)3 * 32 * std::min(d.UP(), kCombineWindow) * sizeof(float);
  cudaFuncSetAttribute(combine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
  RNNT_LAUNCH(KID_COMBINE, st, launch_pdl(combine_kernel, grid, 256, csm, st, w.pxy, w.rS, w.alpha, w.beta, w.Ash, w.Bsh,
                                                                   w.Ltot, bnd, d.T, d.U, d.LU(), d.K(), d.lat_W(),
                                                                   32 * d.lat_R(), d.UP(), px_grad, py_grad, w.Gt_hi,
                                                                   w.Gt_lo));
  return cudaGetLastError();
}

}  // namespace rnnt
