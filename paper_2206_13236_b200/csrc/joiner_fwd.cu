// joiner_fwd.cu — K8: joiner output projection on the band with fused log-softmax, blank /
// label pick and the stored probabilities for function merging.
//
//   z[r,v] = sum_j h[r,j] W[v,j] + b[v]        (tcgen05.mma kind::f16, fp32 accumulation in TMEM)
//   lse[r] = log sum_v exp z[r,v]               (online over V tiles, one TMEM lane = one row)
//   py2[r] = (z[r,0] - lse) log2e, px2[r] = (z[r,y] - lse) log2e   (-inf at u = U_n)
//   P~[r,v] = bf16(exp(z[r,v] - m[r, v/128])), m = per-128-column max  (read by K10/K11)
//
// One CTA per 128-row tile of the band rows; it sweeps all of V in 256-column MMA tiles
// (N=256, K-loop over J in 64-wide TMA boxes, 4-stage mbarrier ring), double-buffered TMEM
// accumulators (2 x 256 columns) so the epilogue of tile i overlaps the MMAs of tile i+1.
// Warp 0: TMA producer.  Warp 1: TMEM allocator + single-thread MMA issuer.  Warps 2-5:
// epilogue (warp w reads TMEM lanes 32*(w%4)..+31).
#include "common.cuh"
#include "launch.h"
#include "tc.cuh"
#include "tmap.h"
#include "workspace.h"

namespace rnnt {

namespace jf {
// 128-column V tiles, double-buffered accumulators (2 x 128 TMEM columns) and a 3-stage ring
// (~97 KB smem): two CTAs per SM, so one CTA's softmax epilogue overlaps the other's MMAs.
constexpr int BM = 128, BN = 128, BK = 64, STAGES = 3;
constexpr int A_BYTES = BM * BK * 2;        // 16 KB
constexpr int B_BYTES = BN * BK * 2;        // 16 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
constexpr int THREADS = 192;
}  // namespace jf

struct JoinerFwdParams {
  const float* bias;      // (VP) fp32, padded
  const int32_t* rowinfo; // (R)
  long long R;
  int V, VP, J, nvt, nkb, ntile;
  uint16_t* Pt;           // (R, VP)
  float* mt;              // (R, ntile)
  float* lse;
  float* px2;
  float* py2;
};

__global__ void __launch_bounds__(jf::THREADS, 2)
    joiner_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         JoinerFwdParams p) {
  using namespace jf;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = tc::align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long m0 = (long long)blockIdx.x * BM;

  int act = 0;
  for (int i = threadIdx.x; i < BM; i += blockDim.x)
    if (m0 + i < p.R && p.rowinfo[m0 + i] >= 0) act = 1;
  if (!__syncthreads_or(act)) return;   // tile entirely masked / padding

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { tc::mbar_init(&tfull[s], 1); tc::mbar_init(&tempty[s], 4); }
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * BN);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = *tmem_slot;
  const int nvt = p.nvt, nkb = p.nkb;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0;
      for (int nt = 0; nt < nvt; ++nt) {
        for (int kb = 0; kb < nkb; ++kb) {
          tc::mbar_wait(&empty[stage], ph ^ 1);
          tc::mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          tc::tma_load_2d(sa, &tmA, &full[stage], kb * BK, (int)m0);
          tc::tma_load_2d(sa + A_BYTES, &tmB, &full[stage], kb * BK, nt * BN);
          if (++stage == STAGES) { stage = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16(BM, BN, false, false);
      int stage = 0;
      uint32_t ph = 0;
      for (int nt = 0; nt < nvt; ++nt) {
        const int acc = nt & 1;
        tc::mbar_wait(&tempty[acc], ((nt >> 1) & 1) ^ 1);
        tc::fence_after_sync();
        const uint32_t d = tbase + acc * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          tc::mbar_wait(&full[stage], ph);
          tc::fence_after_sync();
          const uint32_t a = tc::smem_u32(smem + stage * STAGE_BYTES), b = a + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            tc::mma_bf16(d, tc::sdesc(a + 32 * k, 16, 1024), tc::sdesc(b + 32 * k, 16, 1024), idesc,
                         (kb | k) != 0);
          tc::mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; ph ^= 1; }
        }
        tc::mma_commit(&tfull[acc]);
      }
    }
  } else {
    const int q = warp & 3;
    const long long r = m0 + 32 * q + lane;
    const int info = (r < p.R) ? p.rowinfo[r] : -1;
    const uint32_t tl = tbase + ((uint32_t)(32 * q) << 16);
    float M = neg_inf_f(), sum = 0.f, zb = neg_inf_f(), zl = neg_inf_f();
    uint16_t* prow = p.Pt + (size_t)(info >= 0 ? r : 0) * p.VP;
    for (int nt = 0; nt < nvt; ++nt) {
      const int acc = nt & 1;
      tc::mbar_wait(&tfull[acc], (nt >> 1) & 1);
      tc::fence_after_sync();
      {
        const int v0 = nt * BN;
        const uint32_t tcol = tl + acc * BN;
        float m = neg_inf_f();
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          float z[32];
          tc::tmem_ld32(tcol + 32 * c, z);
          const float4* bb = reinterpret_cast<const float4*>(p.bias + v0 + 32 * c);
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            float4 b4 = __ldg(bb + j4);
            float bj[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int j = 4 * j4 + i;
              const float zz = (v0 + 32 * c + j < p.V) ? z[j] + bj[i] : neg_inf_f();
              m = fmaxf(m, zz);
            }
          }
        }
        const float mL = m * RNNT_LOG2E_F;
        float s = 0.f;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          float z[32];
          tc::tmem_ld32(tcol + 32 * c, z);
          const int vc = v0 + 32 * c;
          const float4* bb = reinterpret_cast<const float4*>(p.bias + vc);
          uint32_t pk[16];
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            float4 b4 = __ldg(bb + j4);
            float bj[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int j = 4 * j4 + i;
              z[j] = (vc + j < p.V) ? z[j] + bj[i] : neg_inf_f();
            }
          }
          float e[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            e[j] = ex2_approx(fmaf(z[j], RNNT_LOG2E_F, -mL));
            s += e[j];
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            __nv_bfloat162 h2 = __floats2bfloat162_rn(e[2 * j], e[2 * j + 1]);
            pk[j] = *reinterpret_cast<uint32_t*>(&h2);
          }
          if (info >= 0) {
            uint4* dst = reinterpret_cast<uint4*>(prow + vc);
#pragma unroll
            for (int j = 0; j < 4; ++j) dst[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
          }
          if (vc == 0) zb = z[0];
          const int li = info - vc;
          const bool hit = (unsigned)li < 32u;
          if (__any_sync(0xffffffffu, hit)) {
            float sel = z[0];
#pragma unroll
            for (int j = 1; j < 32; ++j) sel = (li == j) ? z[j] : sel;
            if (hit) zl = sel;
          }
        }
        if (info >= 0) p.mt[(size_t)r * p.ntile + v0 / 128] = m;
        const float Mn = fmaxf(M, m);
        sum = sum * ex2_approx((M - Mn) * RNNT_LOG2E_F) + s * ex2_approx((m - Mn) * RNNT_LOG2E_F);
        M = Mn;
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
    if (r < p.R) {
      if (info >= 0) {
        const float l = M + lg2_approx(sum) * RNNT_LN2_F;
        p.lse[r] = l;
        p.py2[r] = (zb - l) * RNNT_LOG2E_F;
        p.px2[r] = info < p.V ? (zl - l) * RNNT_LOG2E_F : kNegBig;   // y(t,U) = -inf
      } else {
        p.lse[r] = 0.f;
        p.px2[r] = kNegBig;
        p.py2[r] = kNegBig;
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tbase, 2 * BN);
}

cudaError_t joiner_fwd_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, const uint16_t* W,
                              const uint16_t* b, cudaStream_t st) {
  const long long R = d.rows();
  const int VP = d.VP();
  CUtensorMap ta, tb;
  if (!make_tmap_bf16_2d(&ta, h, d.J, R, (uint64_t)d.J * 2, jf::BK, jf::BM)) return cudaErrorInvalidValue;
  if (!make_tmap_bf16_2d(&tb, W, d.J, d.V, (uint64_t)d.J * 2, jf::BK, jf::BN)) return cudaErrorInvalidValue;
  JoinerFwdParams p{w.bias, w.rowinfo, R, d.V, VP, d.J, (d.V + jf::BN - 1) / jf::BN, (d.J + jf::BK - 1) / jf::BK,
                    d.ntile(), w.Pt, w.mt, w.lse, w.px2, w.py2};
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(joiner_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, jf::SMEM_BYTES);
    attr = true;
  }
  const unsigned grid = (unsigned)((R + jf::BM - 1) / jf::BM);
  RNNT_LAUNCH(KID_JOINER_FWD, st, joiner_fwd_tc_kernel<<<grid, jf::THREADS, jf::SMEM_BYTES, st>>>(ta, tb, p));
  return cudaGetLastError();
}

}  // namespace rnnt
