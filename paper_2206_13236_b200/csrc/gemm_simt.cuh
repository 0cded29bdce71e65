// gemm_simt.cuh — generic fp32 CUDA-core tile GEMM, C[m][n] = sum_k A(m,k) B(n,k),
// with operand loaders and the epilogue supplied by a problem functor.
//
// This is the v0 contraction used to bring every stage up bit-for-bit against the
// oracle; the tcgen05 kernels (gemm_tc.cuh) replace it on the hot path stage by
// stage.  64x64 tile, 256 threads, 4x4 outputs per thread, K chunk 16.
#pragma once
#include "common.cuh"

namespace rnnt {

template <class P>
__global__ void __launch_bounds__(256) simt_gemm_kernel(P p) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int z = blockIdx.z;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (!p.tile_active(z, m0, n0)) return;
  long long kbeg, kend;
  p.krange(z, m0, n0, kbeg, kend);
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (long long k0 = kbeg; k0 < kend; k0 += BK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int idx = tid + 256 * i;
      int kk, mm;
      if (P::kAMajorM) { mm = idx & 63; kk = idx >> 6; } else { kk = idx & 15; mm = idx >> 4; }
      long long k = k0 + kk;
      As[kk][mm] = (k < kend) ? p.A(z, m0 + mm, k) : 0.f;
      int nn;
      if (P::kBMajorN) { nn = idx & 63; kk = idx >> 6; } else { kk = idx & 15; nn = idx >> 4; }
      k = k0 + kk;
      Bs[kk][nn] = (k < kend) ? p.B(z, n0 + nn, k) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) p.epi(z, m0 + ty + 16 * i, n0 + tx + 16 * j, acc[i][j]);
}

template <class P>
inline cudaError_t launch_simt_gemm(const P& p, int M, int Ncols, int Z, cudaStream_t st) {
  dim3 grid((Ncols + 63) / 64, (M + 63) / 64, Z);
  if (grid.x == 0 || grid.y == 0 || grid.z == 0) return cudaSuccess;
  simt_gemm_kernel<P><<<grid, 256, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace rnnt
