// Microbenchmark: per-iteration latency (cycles) of dependent chains used by the wavefronts.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float lg2(float x) { float y; asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float lae(float a, float b) { float m = fmaxf(a, b); return m + lg2(1.f + ex2(-fabsf(a - b))); }
__device__ __forceinline__ float credux(float v) { float r; asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v)); return r; }

template <int V>
__global__ void k(float* out, long long* cyc, int iters) {
  float x = threadIdx.x * 1e-3f, y = 0.5f, m1 = 0.f, m2 = 0.f;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (V == 0) { x = ex2(-fabsf(x)); }
    if (V == 1) { x = lg2(1.f + x); }
    if (V == 2) { x = lae(x, y) - 1.0f; }
    if (V == 3) { float nb = __shfl_up_sync(0xffffffffu, x, 1); x = lae(x, nb) - 1.0f; }
    if (V == 4) { float nb = __shfl_up_sync(0xffffffffu, x, 1); x = lae(x, nb) - m2; float M = credux(x); m2 = m1; m1 = M; }
    if (V == 5) { x = __shfl_up_sync(0xffffffffu, x, 1) + 1.0f; }
    if (V == 6) { float M = credux(x); x = x - M * 1e-3f; }
    if (V == 7) { out[(i & 255) * 32 + threadIdx.x] = x; x = lae(x, y) - 1.0f; }
  }
  long long t1 = clock64();
  out[threadIdx.x + 8192] = x + m1;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 8);
  const int iters = 4096;
  const char* names[] = {"ex2 chain", "lg2(1+x) chain", "lae2 chain", "lae2+shfl", "lae2+shfl+credux(delay2)", "shfl+fadd", "credux consumed", "lae2+stg"};
  for (int v = 0; v < 8; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (v) {
        case 0: k<0><<<1, 32>>>(out, cyc, iters); break;
        case 1: k<1><<<1, 32>>>(out, cyc, iters); break;
        case 2: k<2><<<1, 32>>>(out, cyc, iters); break;
        case 3: k<3><<<1, 32>>>(out, cyc, iters); break;
        case 4: k<4><<<1, 32>>>(out, cyc, iters); break;
        case 5: k<5><<<1, 32>>>(out, cyc, iters); break;
        case 6: k<6><<<1, 32>>>(out, cyc, iters); break;
        case 7: k<7><<<1, 32>>>(out, cyc, iters); break;
      }
      cudaDeviceSynchronize();
    }
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %6.1f cycles/iter\n", names[v], (double)c / iters);
  }
  return 0;
}
