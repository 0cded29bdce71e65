// exchange.cu — the data-parallel exchange step of the pruned RNN-T loss:
// the batch loss combination and the reduction of the joiner-weight gradients into one
// flat fp32 buffer  acc = [ d_w (V*J) | d_b (V) | loss sums (2) ].
//
// Accumulation targets (rnnt_exchange_mode_t in include/rnnt.h):
//   STORE     plain stores (deterministic; the caller's all_reduce, e.g. NCCL, does the rest);
//   RED       red.global.add: several shards (or ranks sharing one device buffer) add into one zeroed
//             buffer — the single-GPU form of the exchange, parity-tested on one device;
//   MULTIMEM  multimem.red.add on an NVLS multicast address: every rank's copy of the symmetric
//             buffer receives the sum over ranks inside the NVSwitch (no separate all_reduce pass).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "launch.h"

namespace rnnt {

__device__ __forceinline__ void acc_add(float* p, float v, int mode) {
  if (mode == 0) {
    *p = v;
  } else if (mode == 1) {
    asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
  } else {
    asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
  }
}

__device__ __forceinline__ void acc_add4(float4* p, float4 v, int mode) {
  if (mode == 0) {
    *p = v;
  } else if (mode == 1) {
    asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
  } else {
    asm volatile("multimem.red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
  }
}

// out[0] = simple_scale * sum_n loss_simple[n]; out[1] = pruned_scale * sum_n loss_pruned[n] over the
// utterances whose status bit0 (infeasible, D16) is clear.  One warp, fixed order: lane l sums n = l,
// l+32, ... in fp64, then a butterfly in a fixed pattern -> deterministic.
__global__ void loss_sums_kernel(const float* __restrict__ ls, const float* __restrict__ lp,
                                 const int32_t* __restrict__ status, int N, float s_scale, float p_scale,
                                 float* out, int mode) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  const int lane = threadIdx.x;
  double a = 0.0, b = 0.0;
  for (int n = lane; n < N; n += 32) {
    a += (double)ls[n];
    if (!(status && (status[n] & kStatusInfeasible))) b += (double)lp[n];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if (lane == 0) {
    acc_add(out, (float)(a * (double)s_scale), mode);
    acc_add(out + 1, (float)(b * (double)p_scale), mode);
  }
}

cudaError_t loss_sums_launch(const float* ls, const float* lp, const int32_t* status, int N, float s_scale,
                             float p_scale, float* out, int mode, cudaStream_t st) {
  RNNT_LAUNCH(KID_LOSS_SUMS, st, launch_pdl(loss_sums_kernel, 1, 32, 0, st, ls, lp, status, N, s_scale, p_scale, out, mode));
  return cudaGetLastError();
}

// Split-K reduction of the d_w / d_b partials (fixed split order) into the accumulation target.
__global__ void split_reduce_acc_kernel(const float4* __restrict__ part, int splits, long long M4,
                                        float4* out, int mode) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M4) return;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int z0 = 0; z0 < splits; z0 += 8) {
    float4 x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      x[k] = z0 + k < splits ? part[(size_t)(z0 + k) * M4 + i] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (z0 + k >= splits) break;
      acc.x += x[k].x; acc.y += x[k].y; acc.z += x[k].z; acc.w += x[k].w;
    }
  }
  acc_add4(out + i, acc, mode);
}
__global__ void split_reduce_acc1_kernel(const float* __restrict__ part, int splits, long long M, float* out,
                                         int mode) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  float acc = 0.f;
  for (int z = 0; z < splits; ++z) acc += part[(size_t)z * M + i];
  acc_add(out + i, acc, mode);
}

cudaError_t split_reduce_acc_launch(const float* part, int splits, long long M, float* out, int mode, int kid,
                                    cudaStream_t st) {
  if (M % 4 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0 && reinterpret_cast<uintptr_t>(part) % 16 == 0)
    RNNT_LAUNCH(kid, st, launch_pdl(split_reduce_acc_kernel, (unsigned)((M / 4 + 255) / 256), 256, 0, st, 
        reinterpret_cast<const float4*>(part), splits, M / 4, reinterpret_cast<float4*>(out), mode));
  else
    RNNT_LAUNCH(kid, st, launch_pdl(split_reduce_acc1_kernel, (unsigned)((M + 255) / 256), 256, 0, st, part, splits, M, out,
                                                                                                mode));
  return cudaGetLastError();
}

}  // namespace rnnt
