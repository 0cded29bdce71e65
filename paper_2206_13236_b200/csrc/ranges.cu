// ranges.cu — pruning bounds.
//
//   K6a raw_bounds_kernel : Eq. 8 per frame, one warp per (n,t):
//         v(p) = -y'(t,p-1) + sum_{u=p}^{p+S-1} empty'(t,u),  p = 0..max(0,U_n-S+1)
//       fp32 inputs promoted to fp64, summed u ascending then the subtraction (D5), so the
//       argmax (ties -> smallest p) is bit-exact w.r.t. the oracle on identical inputs.
//   K6b adjust_kernel     : ADJ-scan (D3) per utterance: clamp to the reachability envelope,
//       prefix max (Eq. 9), suffix max of q_t' - (t'-t)(S-1) (Eq. 10).  Integer, exact.
#include <climits>

#include "common.cuh"
#include "launch.h"
#include "workspace.h"

namespace rnnt {

__global__ void __launch_bounds__(256) raw_bounds_kernel(const float* __restrict__ px_grad,
                                                         const float* __restrict__ py_grad,
                                                         const int64_t* __restrict__ bnd, int N, int T, int U, int S,
                                                         int32_t* __restrict__ raw) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  // the warp's frame row (y' and empty', U_n + 1 values each) is staged in smem with all loads in
  // flight at once; the fp64 window sums then read smem only
  extern __shared__ float rowbuf[];   // [8 warps][2][U + 1]
  long long row = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= (long long)N * T) return;
  const int n = (int)(row / T), t = (int)(row % T);
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  if (t >= Tn) return;
  const int Umax = max(0, Un - S + 1);
  float* yb = rowbuf + (threadIdx.x / 32) * 2 * (U + 1);
  float* bb = yb + (U + 1);
  const float* yr = px_grad + row * (long long)(U + 1);
  const float* br = py_grad + row * (long long)(U + 1);
  for (int u = lane; u <= Un; u += 32) { yb[u] = yr[u]; bb[u] = br[u]; }
  __syncwarp();
  double best = -1e300;
  int bestp = 0x7fffffff;
  for (int p = lane; p <= Umax; p += 32) {
    double acc = 0.0;
    const int hi = min(p + S, Un + 1);
    for (int u = p; u < hi; ++u) acc = __dadd_rn(acc, (double)bb[u]);
    if (p > 0) acc = __dsub_rn(acc, (double)yb[p - 1]);
    if (acc > best || (acc == best && p < bestp)) { best = acc; bestp = p; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ob = __shfl_xor_sync(0xffffffffu, best, o);
    int op = __shfl_xor_sync(0xffffffffu, bestp, o);
    if (ob > best || (ob == best && op < bestp)) { best = ob; bestp = op; }
  }
  if (lane == 0) raw[row] = bestp;
}

// Inclusive max-scan over the 1024 threads of the block (reverse: over tid descending): a warp
// scan by shuffles, the 32 warp totals scanned by warp 0 through smem, then combined.
__device__ __forceinline__ int block_scan_max(int x, int* sh, bool reverse) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NEG = INT_MIN;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = reverse ? __shfl_down_sync(0xffffffffu, x, o) : __shfl_up_sync(0xffffffffu, x, o);
    if (reverse ? (lane + o < 32) : (lane >= o)) x = max(x, y);
  }
  __syncthreads();                                   // sh free (previous use complete)
  if (lane == (reverse ? 0 : 31)) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int v = sh[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = reverse ? __shfl_down_sync(0xffffffffu, v, o) : __shfl_up_sync(0xffffffffu, v, o);
      if (reverse ? (lane + o < 32) : (lane >= o)) v = max(v, y);
    }
    sh[lane] = v;                                     // inclusive over warps
  }
  __syncthreads();
  // combine with the warps before (after, reversed)
  int prev = NEG;
  if (reverse ? (warp < 31) : (warp > 0)) prev = sh[reverse ? warp + 1 : warp - 1];
  return max(x, prev);
}

// One CTA (1024 threads) per utterance; frames processed in chunks of blockDim.x with a
// carried prefix (max) / suffix (max) value.
// raw, q and ranges may alias (each frame's value is consumed before it is overwritten).
__global__ void __launch_bounds__(1024) adjust_kernel(const int32_t* raw, const int64_t* __restrict__ bnd,
                                                      int T, int S, int32_t* ranges, int32_t* q,
                                                      int32_t* __restrict__ status) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  const int n = blockIdx.x;
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  const int Umax = max(0, Un - S + 1);
  const int tid = threadIdx.x, nt = blockDim.x;
  const bool feasible = (long long)Un <= (long long)Tn * (S - 1);
  int32_t* out = ranges + (size_t)n * T;
  if (!feasible) {
    for (int t = tid; t < T; t += nt) out[t] = 0;
    if (tid == 0) set_status(status, n, kStatusInfeasible);
    return;
  }
  __shared__ int sh[1024];
  __shared__ int carry;
  int32_t* qq = q + (size_t)n * T;
  // 1+2: clamp into [l_t, h_t] and running max (Eq. 9)
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int c0 = 0; c0 < Tn; c0 += nt) {
    const int t = c0 + tid;
    int x = 0;
    if (t < Tn) {
      const long long lo = max(0LL, (long long)Umax - (long long)(Tn - 1 - t) * (S - 1));
      const long long hi = min((long long)Umax, (long long)t * (S - 1));
      long long r = raw[(size_t)n * T + t];
      r = r < lo ? lo : (r > hi ? hi : r);
      x = (int)r;
    }
    const int incl = block_scan_max(x, sh, false);
    const int c = carry;
    if (t < Tn) qq[t] = max(incl, c);
    __syncthreads();
    if (tid == nt - 1) carry = max(c, incl);
    __syncthreads();
  }
  // 3: p_t = max_{t'>=t} (q_t' - t'(S-1)) + t(S-1)   (Eq. 10)
  if (tid == 0) carry = INT_MIN;
  __syncthreads();
  const int nchunks = (Tn + nt - 1) / nt;
  for (int ci = nchunks - 1; ci >= 0; --ci) {
    const int t = ci * nt + tid;
    int g = INT_MIN;
    if (t < Tn) g = qq[t] - t * (S - 1);
    // reverse inclusive max-scan within the chunk
    const int rincl = block_scan_max(g, sh, true);
    const int c = carry;
    if (t < Tn) out[t] = max(rincl, c) + t * (S - 1);
    __syncthreads();
    if (tid == 0) carry = max(c, rincl);
    __syncthreads();
  }
  for (int t = Tn + tid; t < T; t += nt) out[t] = Umax;   // padded frames (D11)
}

cudaError_t get_ranges_launch(const Dims& d, const float* px_grad, const float* py_grad, const int64_t* bnd,
                              int32_t* ranges, int32_t* status, cudaStream_t st) {
  // raw bounds and the monotone hull q are staged in the output buffer itself (no workspace).
  long long rows = (long long)d.N * d.T;
  const size_t sm = (size_t)8 * 2 * d.U1() * sizeof(float);
  if (sm > 48 * 1024) cudaFuncSetAttribute(raw_bounds_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  RNNT_LAUNCH(KID_RAW, st, launch_pdl(raw_bounds_kernel, (unsigned)((rows + 7) / 8), 256, sm, st, px_grad, py_grad, bnd, d.N, d.T,
                                                                                         d.U, d.S, ranges));
  RNNT_LAUNCH(KID_ADJUST, st, launch_pdl(adjust_kernel, d.N, 1024, 0, st, ranges, bnd, d.T, d.S, ranges, ranges, status));
  return cudaGetLastError();
}

}  // namespace rnnt
