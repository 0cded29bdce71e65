// common.cuh — shared device helpers for the sm_100a pruned RNN-T kernels.
//
// Log-space arithmetic is kept in BASE 2 inside the recursions (x2 = x * log2(e)):
// LogAdd(x,y) = log(e^x+e^y) (Eq. 4) becomes m + log2(1 + 2^(n-m)) with
// one MUFU.EX2 and one MUFU.LG2 and no scaling multiplies.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <math.h>

#define RNNT_LOG2E 1.4426950408889634
#define RNNT_LN2 0.6931471805599453
#define RNNT_LOG2E_F 1.4426950408889634f
#define RNNT_LN2_F 0.6931471805599453f

namespace rnnt {

constexpr int kStatusInfeasible = 1;
constexpr int kStatusNonFinite = 2;
constexpr int kStatusBadSymbol = 4;
constexpr int kStatusUnderflow = 8;
constexpr int kStatusBadBoundary = 16;

// Columns per max-shift tile of the stored unnormalised joiner probabilities P~
// (D11 / DESIGN.md "K8"): P~[r,v] = bf16(exp(z[r,v] - m[r, v / kVT])).
constexpr int kVT = 128;

// "log 0" of the fp32 log-space recursions: finite, so LogAdd needs no -inf guard; any sum with it
// stays below -1e29 for 1e8 steps, and exp2 of it is exactly 0.
constexpr float kNegBig = -1.0e30f;

__device__ __forceinline__ float neg_inf_f() { return __int_as_float(0xff800000); }
__device__ __forceinline__ double neg_inf_d() { return __longlong_as_double(0xfff0000000000000ULL); }

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// tanh to ~2e-6 relative (enough that bf16 round-to-nearest of the result matches the fp64
// reference except at ~1e-3 of the rounding midpoints): odd Taylor polynomial for |x| < 1/4,
// 1 - 2 / (e^{2|x|} + 1) with MUFU ex2 / rcp above (two MUFU, no division, no cancellation
// below 0.245).
__device__ __forceinline__ float tanh_fast(float x) {
  // branch-free (no divergence within a warp): both forms are evaluated, the select picks one
  const float ax = fabsf(x);
  const float x2 = x * x;
  float p = -1382.f / 155925.f;
  p = fmaf(p, x2, 62.f / 2835.f);
  p = fmaf(p, x2, -17.f / 315.f);
  p = fmaf(p, x2, 2.f / 15.f);
  p = fmaf(p, x2, -1.f / 3.f);
  const float small = fmaf(p * x2, x, x);
  const float e = ex2_approx(ax * (2.0f * 1.4426950408889634f));
  const float big = copysignf(fmaf(-2.0f, rcp_approx(e + 1.0f), 1.0f), x);
  return ax < 0.25f ? small : big;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// LogAdd in base 2 with an fp64 state and an fp32 correction term:
//   logadd2(a,b) = max + log2(1 + 2^(min-max)),  logadd2(-inf,-inf) = -inf (D8).
// The state is fp64 so that |alpha| ~ 1e4 keeps ~1e-12 absolute precision
// (DESIGN.md "Recursion precision"); the correction is in [0,1] and fp32 suffices.
__device__ __forceinline__ double logadd2_d(double a, double b) {
  double m = fmax(a, b);
  double n = fmin(a, b);
  if (m == neg_inf_d()) return m;
  float d = (float)(n - m);
  float c = lg2_approx(1.0f + ex2_approx(d));
  return m + (double)c;
}

__device__ __forceinline__ float logadd2_f(float a, float b) {
  float m = fmaxf(a, b);
  float n = fminf(a, b);
  if (m == neg_inf_f()) return m;
  return m + lg2_approx(1.0f + ex2_approx(n - m));
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float bf16_bits_to_f(uint16_t b) {
  return __uint_as_float(((uint32_t)b) << 16);
}
__device__ __forceinline__ uint16_t f_to_bf16_bits_rn(float f) {
  __nv_bfloat16 h = __float2bfloat16_rn(f);
  return *reinterpret_cast<uint16_t*>(&h);
}

// Per-utterance lengths from boundary (N,4) {0,0,U_n,T_n}.
__device__ __forceinline__ int utt_T(const int64_t* boundary, int n) { return (int)boundary[4 * n + 3]; }
__device__ __forceinline__ int utt_U(const int64_t* boundary, int n) { return (int)boundary[4 * n + 2]; }

__device__ __forceinline__ void set_status(int32_t* status, int n, int bits) {
  if (status && bits) atomicOr(status + n, bits);
}

}  // namespace rnnt
