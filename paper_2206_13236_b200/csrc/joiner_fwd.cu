// joiner_fwd.cu — K8: joiner output projection on the band with fused log-softmax, blank /
// label pick and the stored probabilities for function merging.
//
//   z[r,v] = sum_j h[r,j] W[v,j] + b[v]        (tcgen05.mma kind::f16, fp32 accumulation in TMEM)
//   lse[r] = log sum_v exp z[r,v]               (online over V tiles, one TMEM lane = one row)
//   py2[r] = (z[r,0] - lse) log2e, px2[r] = (z[r,y] - lse) log2e   (-inf at u = U_n)
//   P~[r,v] = bf16(exp(z[r,v] - m[r, v/128]))                             (read by K10/K11)
//   (pair kernel: m = m_ref(r) for every tile -- the max of the row's first 32 columns of V tiles 0
//    and 1 -- unless a tile holds a logit above m_ref + 60: that tile takes its exact max and raises
//    tscale; the 1-CTA kernel: m = per-128-column offset from the running max, tscale raised)
//
// Persistent CTAs (two per SM) loop over the live 128-row tiles of the band rows; each sweeps all of
// V in 128-column MMA tiles (K-loop over J in 64-wide TMA boxes, 3-stage mbarrier ring) with
// double-buffered TMEM accumulators (2 x 128 columns) so the epilogue of one tile overlaps the
// MMAs of the next.
// Warp 0: TMA producer.  Warp 1: TMEM allocator + single-thread MMA issuer.  Warps 2-5:
// epilogue (warp w reads TMEM lanes 32*(w%4)..+31).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"
#include "tc.cuh"
#include "tmap.h"
#include "workspace.h"

namespace rnnt {

namespace jf {
// One CTA per SM: a 4-stage TMA ring, four 128-column TMEM accumulators and two epilogue sets of
// four warps.  Row tiles alternate between the sets (set e owns accumulators 2e, 2e+1, double-
// buffered over its V tiles), so each set has two row tiles of MMA time for its softmax epilogue.
// P~ leaves through a per-set 32 KB staging tile by TMA (two 64-column SWIZZLE_128B boxes): full-line
// coalesced writes instead of 16-B per-row stores.
constexpr int BM = 128, BN = 128, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;        // 16 KB
constexpr int B_BYTES = BN * BK * 2;        // 16 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int STG_BYTES = BM * BN * 2;      // 32 KB bf16 P~ tile per epilogue set
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 2 * STG_BYTES + 1024 + 256;
constexpr int THREADS = 320;                // warp 0 TMA, warp 1 MMA, warps 2-5 / 6-9 epilogue sets
}  // namespace jf

// byte offset of logical 16-B chunk `c` (0..7) of 128-B row `r` in a SWIZZLE_128B atom stack
__device__ __forceinline__ uint32_t sw128f(int r, int c) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}

struct JoinerFwdParams {
  const float* bias;      // (VP) fp32, padded
  const float* bmax;      // (ntile) max of the bias over each 128-column tile
  const int32_t* rowinfo; // (R)
  const uint8_t* tlive;   // (ntiles_rows) 1 if the 128-row tile holds a live row (rowinfo_kernel)
  int* counter;           // dynamic tile scheduler (zeroed by rowinfo_kernel)
  long long R;
  int ntiles, V, VP, J, nvt, nkb, ntile;
  uint16_t* Pt;           // (R, VP)
  float* mt;              // (R, ntile)
  float* lse;
  float* px2;
  float* py2;
  int dbg;                // diagnostics (RNNT_DBG_FWD): 1 no epilogue math, 2 no MMA, 3 no TMA
  int* tscale;            // set to 1 when some row's P~ tiles do not share one offset (PrunedWS::tscale)
};

// Persistent: CTA c processes the live 128-row tiles c, c + gridDim.x, ...; the TMA ring, the
// MMA issue and the double-buffered TMEM accumulators run continuously across row tiles, so the
// softmax epilogue of one (row tile, V tile) overlaps the MMAs of the next.
__global__ void __launch_bounds__(jf::THREADS, 1)
    joiner_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ CUtensorMap tmP, JoinerFwdParams p) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  if (blockIdx.x == 0 && threadIdx.x == 0 && p.tscale) *p.tscale = 1;   // per-tile offsets (running max)
  using namespace jf;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = tc::align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + 2 * STG_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;      // [4] accumulators
  uint64_t* tempty = tfull + 4;
  uint64_t* qfull = tempty + 4;          // [4] tile queue: producer -> MMA issuer + epilogue
  uint64_t* qempty = qfull + 4;
  int* tq = reinterpret_cast<int*>(qempty + 4);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
    for (int s = 0; s < 4; ++s) { tc::mbar_init(&tfull[s], 1); tc::mbar_init(&tempty[s], 4); }
    for (int s = 0; s < 4; ++s) { tc::mbar_init(&qfull[s], 1); tc::mbar_init(&qempty[s], 9); }
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 4 * BN);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = *tmem_slot;
  const int nvt = p.nvt, nkb = p.nkb;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0, qi = 0;
      uint32_t ph = 0;
      for (;;) {
        // next live row tile from the global counter, published to the other roles
        int rt = atomicAdd(p.counter, 1);
        while (rt < p.ntiles && !p.tlive[rt]) rt = atomicAdd(p.counter, 1);
        if (rt >= p.ntiles) rt = -1;
        tc::mbar_wait(&qempty[qi & 3], ((qi >> 2) & 1) ^ 1);
        tq[qi & 3] = rt;
        tc::mbar_arrive(&qfull[qi & 3]);
        ++qi;
        if (rt < 0) break;
        const int m0 = rt * BM;
        // the h row tile comes from HBM once (then L2 for the other V tiles): prefetch its boxes
        for (int kb = 0; kb < nkb; ++kb) tc::tma_prefetch_2d(&tmA, kb * BK, m0);
        for (int nt = 0; nt < nvt; ++nt) {
          for (int kb = 0; kb < nkb; ++kb) {
            tc::mbar_wait(&empty[stage], ph ^ 1);
            uint8_t* sa = smem + stage * STAGE_BYTES;
            if (p.dbg == 3) {
              tc::mbar_arrive(&full[stage]);
            } else {
              tc::mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
              tc::tma_load_2d(sa, &tmA, &full[stage], kb * BK, m0);
              tc::tma_load_2d(sa + A_BYTES, &tmB, &full[stage], kb * BK, nt * BN);
            }
            if (++stage == STAGES) { stage = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16(BM, BN, false, false);
      int stage = 0, qi = 0, ite[2] = {0, 0};
      uint32_t ph = 0;
      for (;;) {
        tc::mbar_wait(&qfull[qi & 3], (qi >> 2) & 1);
        const int rt = tq[qi & 3];
        tc::mbar_arrive(&qempty[qi & 3]);
        const int set = qi & 1;                  // row tiles alternate between the epilogue sets
        ++qi;
        if (rt < 0) break;
        for (int nt = 0; nt < nvt; ++nt) {
          const int it = ite[set]++;
          const int acc = 2 * set + (it & 1);
          tc::mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
          tc::fence_after_sync();
          const uint32_t d = tbase + acc * BN;
          for (int kb = 0; kb < nkb; ++kb) {
            tc::mbar_wait(&full[stage], ph);
            tc::fence_after_sync();
            const uint32_t a = tc::smem_u32(smem + stage * STAGE_BYTES), b = a + A_BYTES;
            if (p.dbg != 2) {
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)
                tc::mma_bf16(d, tc::sdesc(a + 32 * k, 16, 1024), tc::sdesc(b + 32 * k, 16, 1024), idesc,
                             (kb | k) != 0);
            }
            tc::mma_commit(&empty[stage]);
            if (++stage == STAGES) { stage = 0; ph ^= 1; }
          }
          tc::mma_commit(&tfull[acc]);
        }
      }
    }
  } else {
    const int q = warp & 3;
    const int set = (warp - 2) >> 2;           // warps 2-5: set 0, warps 6-9: set 1
    const int ethr = 64 + 128 * set;           // the set's store-issuing thread
    uint8_t* stg = smem + STAGES * STAGE_BYTES + set * STG_BYTES;
    const uint32_t tl = tbase + ((uint32_t)(32 * q) << 16);
    int it = 0, qi = 0;
    for (;;) {
      tc::mbar_wait(&qfull[qi & 3], (qi >> 2) & 1);
      const int rt = tq[qi & 3];
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&qempty[qi & 3]);
      const bool mine = (qi & 1) == set;
      ++qi;
      if (rt < 0) break;
      if (!mine) continue;
      const long long r = (long long)rt * BM + 32 * q + lane;
      const int info = (r < p.R) ? p.rowinfo[r] : -1;
      float M = neg_inf_f(), sum = 0.f, zb = neg_inf_f(), zl = neg_inf_f();
      for (int nt = 0; nt < nvt; ++nt, ++it) {
        const int acc = 2 * set + (it & 1);
        const int v0 = nt * BN;
        const float zb_prev = zb, zl_prev = zl;
        tc::mbar_wait(&tfull[acc], (it >> 1) & 1);
        tc::fence_after_sync();
        const uint32_t tcol = tl + acc * BN;
        if (p.dbg == 1) {
          float z[32];
          tc::tmem_ld32(tcol, z);
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&tempty[acc]);
          if (z[0] == 12345.f) M = z[1];
          continue;
        }
        // One TMEM pass: the exp offset m of this tile is fixed from its first 32-column chunk (exact
        // max of z + b there, joined with the running max of the earlier tiles); every chunk is
        // exponentiated against it as it is read.  A chunk exceeding m by more than kRedo (could
        // overflow e^(z-m)) makes the whole warp redo the tile with a max-only first pass (rare).
        constexpr float kRedo = 60.f;
        float m = neg_inf_f(), s = 0.f;
        bool redo = false;
        if (threadIdx.x == ethr) tc::bulk_wait_read0();   // the previous tile's P~ store has left smem
        asm volatile("bar.sync %0, 128;" ::"r"(1 + set) : "memory");
        for (int attempt = 0; attempt < 2; ++attempt) {
          if (attempt == 1) {
            if (!__any_sync(0xffffffffu, redo)) break;
            // exact tile max (masked), then the exp pass again
            m = neg_inf_f();
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
              float z[32];
              tc::tmem_ld32(tcol + 32 * c, z);
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (v0 + 32 * c + j < p.V) m = fmaxf(m, z[j] + p.bias[v0 + 32 * c + j]);
            }
            s = 0.f;
            zb = zb_prev; zl = zl_prev;
          }
          float mL = m * RNNT_LOG2E_F;
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            float z[32];
            {
              uint32_t zr[32];
              tc::tmem_ld32_issue(tcol + 32 * c, zr);
              const int vc = v0 + 32 * c;
              float4 b4[8];
              const float4* bb = reinterpret_cast<const float4*>(p.bias + vc);
#pragma unroll
              for (int j4 = 0; j4 < 8; ++j4) b4[j4] = __ldg(bb + j4);     // overlapped with the TMEM load
              tc::tmem_ld32_wait(zr);
#pragma unroll
              for (int j4 = 0; j4 < 8; ++j4) {
                z[4 * j4] = __uint_as_float(zr[4 * j4]) + b4[j4].x;
                z[4 * j4 + 1] = __uint_as_float(zr[4 * j4 + 1]) + b4[j4].y;
                z[4 * j4 + 2] = __uint_as_float(zr[4 * j4 + 2]) + b4[j4].z;
                z[4 * j4 + 3] = __uint_as_float(zr[4 * j4 + 3]) + b4[j4].w;
              }
            }
            const int vc = v0 + 32 * c;
            // (columns v >= V: the padded bias is -inf there, so z = -inf and e^(z-m) = 0 with no mask)
            if (attempt == 0) {
              float cm = z[0];
#pragma unroll
              for (int j = 1; j < 32; ++j) cm = fmaxf(cm, z[j]);
              if (c == 0) {
                m = fmaxf(M, cm);
                mL = m * RNNT_LOG2E_F;
              } else if (cm - m > kRedo) {
                redo = true;
              }
              if (__any_sync(0xffffffffu, redo)) break;
            }
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float e0 = ex2_approx(fmaf(z[2 * j], RNNT_LOG2E_F, -mL));
              const float e1 = ex2_approx(fmaf(z[2 * j + 1], RNNT_LOG2E_F, -mL));
              s += e0 + e1;
              __nv_bfloat162 h2 = __floats2bfloat162_rn(e0, e1);
              pk[j] = *reinterpret_cast<uint32_t*>(&h2);
            }
            {
              // staging tile: box c/2 (64 columns), 16-B chunks (c%2)*4.. of this row, swizzled
              uint8_t* sb = stg + (c >> 1) * (STG_BYTES / 2);
              const int row = 32 * q + lane;
#pragma unroll
              for (int j = 0; j < 4; ++j)
                *reinterpret_cast<uint4*>(sb + sw128f(row, (c & 1) * 4 + j)) =
                    make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
            }
            if (vc == 0) zb = z[0];
            const int li = info - vc;
            const bool hit = (unsigned)li < 32u;
            if (__any_sync(0xffffffffu, hit)) {
              float zz[32];                 // dynamically indexed: one local-memory round trip
#pragma unroll
              for (int j = 0; j < 32; ++j) zz[j] = z[j];
              if (hit) zl = zz[li];
            }
          }
        }
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&tempty[acc]);
        tc::fence_proxy_async();                        // staging writes -> async proxy
        asm volatile("bar.sync %0, 128;" ::"r"(1 + set) : "memory");
        if (threadIdx.x == ethr && p.dbg != 4) {
          tc::tma_store_2d(&tmP, stg, v0, rt * BM);
          tc::tma_store_2d(&tmP, stg + STG_BYTES / 2, v0 + 64, rt * BM);
          tc::bulk_commit();
        }
        if (info >= 0) p.mt[(size_t)r * p.ntile + v0 / 128] = m;
        const float Mn = fmaxf(M, m);
        sum = sum * ex2_approx((M - Mn) * RNNT_LOG2E_F) + s * ex2_approx((m - Mn) * RNNT_LOG2E_F);
        M = Mn;
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
  }
  if (warp >= 2 && (threadIdx.x & 127) == 64) tc::bulk_wait0();
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tbase, 4 * BN);
}

// CTA-pair variant (cta_group::2): a cluster of two CTAs computes 256 rows (one 128-row tile per CTA)
// x 256 V columns per MMA (M = 256, N = 256).  Each CTA loads its own h rows (A) and HALF of the W rows
// (B: its 128 of the 256 V columns), so the L2 -> SM bytes per MMA flop halve against the single-CTA
// 128 x 128 tiles (the forward's bound at large V).  Row-tile pairs come from the global counter: the
// leader's producer draws the next pair with a live row and publishes it to both CTAs' tile queues
// (a 4-slot ring in shared memory, the peer's written through DSMEM).
// Each CTA holds two 256-column TMEM accumulators (double-buffered); epilogue set e of both CTAs
// takes the 128 columns 128e.. of every accumulator (V tiles 2 vp + e) and keeps its own running
// (max, sum); the two sets merge them at the end of the row tile.
namespace jf2 {
constexpr int BM = 128, BN = 128, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;        // 16 KB: this CTA's 128 h rows
constexpr int B_BYTES = BN * BK * 2;        // 16 KB: this CTA's 128 of the pair's 256 W rows
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int STG_BYTES = BM * BN * 2;      // 32 KB P~ staging per epilogue set
constexpr int MRG_OFF = STAGES * STAGE_BYTES + 2 * STG_BYTES;
constexpr int XCH_OFF = MRG_OFF + 2 * BM * 16;   // [2 sets][128 rows] first-chunk maxima (m_ref)
constexpr int BIAS_OFF = XCH_OFF + 2 * BM * 4;    // the fp32 bias (VP <= kBiasSmem): broadcast reads in the
constexpr int kBiasSmem = 4096;                   // epilogue instead of an L1-missing global load per chunk
constexpr int BAR_OFF = BIAS_OFF + kBiasSmem * 4;
constexpr int SMEM_BYTES = BAR_OFF + 256 + 1024;
constexpr int THREADS = 320;
}  // namespace jf2

// diagnostics: per (CTA, row tile < 8) timestamps {0 producer took the tile, 1 MMA vp0 start, 2 MMA vp0
// issued, 3 MMA last vp issued, 4 epilogue set 0 vp0 full, 5 set 0 vp0 done, 6 set 0 last vp full, 7 set 0
// last vp done, 8 row merged}
#ifdef RNNT_DIAGNOSTICS
__device__ unsigned long long* g_fwd_trace = nullptr;
void set_fwd_trace(void* buf) { cudaMemcpyToSymbol(g_fwd_trace, &buf, sizeof(buf)); }
#else
constexpr unsigned long long* g_fwd_trace = nullptr;   // product build: tracing compiled out
#endif
__device__ __forceinline__ void fwd_trace(int it, int k) {
  if (g_fwd_trace && it < 8) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_fwd_trace[((size_t)blockIdx.x * 8 + it) * 10 + k] = t;
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(jf2::THREADS, 1)
    joiner_fwd_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           const __grid_constant__ CUtensorMap tmP, JoinerFwdParams p) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  using namespace jf2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = tc::align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;      // [2] accumulators
  uint64_t* tempty = tfull + 2;          // [2] (leader's: 8 epilogue warps of each CTA)
  uint64_t* qfull = tempty + 2;          // [4] tile queue: leader producer -> all roles of both CTAs
  uint64_t* qempty = qfull + 4;          // [4] (leader's: 18 consumers over the pair)
  int* tq = reinterpret_cast<int*>(qempty + 4);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq + 4);
  float4* mrg = reinterpret_cast<float4*>(smem + MRG_OFF);   // [2][128] set-1 row state for the merge
  float* xch = reinterpret_cast<float*>(smem + XCH_OFF);
  float* sbias = reinterpret_cast<float*>(smem + BIAS_OFF);
  const bool bsm = p.VP <= kBiasSmem;
  if (bsm)
    for (int v = threadIdx.x; v < p.VP; v += THREADS) sbias[v] = p.bias[v];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_ctarank();
  const bool leader = rank == 0;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { tc::mbar_init(&tfull[s], 1); tc::mbar_init(&tempty[s], 16); }
    for (int s = 0; s < 4; ++s) { tc::mbar_init(&qfull[s], 1); tc::mbar_init(&qempty[s], 18); }
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmA);
    tc::tma_prefetch(&tmB);
  }
  if (warp == 1) tc::tmem_alloc2(tmem_slot, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::cluster_sync();
  tc::fence_after_sync();
  const uint32_t tbase = *tmem_slot;
  const int nvt = p.nvt, nvp = (nvt + 1) / 2, nkb = p.nkb;
  const int npairs = (p.ntiles + 1) / 2;
  auto live_pair = [&](int rp) {
    return p.tlive[2 * rp] || (2 * rp + 1 < p.ntiles && p.tlive[2 * rp + 1]);
  };
  const uint32_t qemptyL = tc::mapa(&qempty[0], 0);
  // consumers: take queue entry qi (-1 = done) and release its slot on the leader (a .cta-release remote
  // arrive, as CUTLASS's cluster-pipeline consumer release: the release.cluster form was ~10 % of the
  // kernel's stall samples at c5, its fence waiting on the warp's outstanding stores)
  auto take = [&](int qi, bool arrive) {
    tc::mbar_wait_cluster(&qfull[qi & 3], (qi >> 2) & 1);
    const int rp = *reinterpret_cast<volatile int*>(&tq[qi & 3]);
    if (arrive) tc::mbar_arrive_remote(qemptyL + (qi & 3) * 8);
    return rp;
  };

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t fullL = tc::mapa(&full[0], 0);
      const uint32_t tqP = tc::mapa(&tq[0], 1), qfullP = tc::mapa(&qfull[0], 1);
      int stage = 0;
      uint32_t ph = 0;
      // queue entry qi: the leader draws the next live row-tile pair and publishes it to both CTAs
      auto draw = [&](int qi) -> int {
        if (!leader) return take(qi, true);
        int rp = atomicAdd(p.counter, 1);
        while (rp < npairs && !live_pair(rp)) rp = atomicAdd(p.counter, 1);
        if (rp >= npairs) rp = -1;
        tc::mbar_wait_cluster(&qempty[qi & 3], ((qi >> 2) & 1) ^ 1);
        tq[qi & 3] = rp;
        tc::st_cluster_u32(tqP + (qi & 3) * 4, (uint32_t)rp);
        tc::mbar_arrive(&qfull[qi & 3]);
        tc::mbar_arrive_cluster(qfullP + (qi & 3) * 8);
        return rp;
      };
      // the next tile is drawn at the start of the current tile's last V pass and its h rows are prefetched
      // into L2 then: its first pass reads them from L2 instead of HBM (c5 trace: the first pass of a tile
      // took 6.4-7.5 us against 3.1 us for the second, every CTA fetching its h rows at the same moment)
      int rp = draw(0);
      if (rp >= 0)
        for (int kb = 0; kb < nkb; ++kb) tc::tma_prefetch_2d(&tmA, kb * BK, (2 * rp + (int)rank) * BM);
      for (int qi = 0; rp >= 0; ++qi) {
        fwd_trace(qi, 0);
        const int m0 = (2 * rp + (int)rank) * BM;
        int rpn = -1;
        for (int vp = 0; vp < nvp; ++vp) {
          if (vp == nvp - 1) {
            rpn = draw(qi + 1);
            if (rpn >= 0)
              for (int kb = 0; kb < nkb; ++kb) tc::tma_prefetch_2d(&tmA, kb * BK, (2 * rpn + (int)rank) * BM);
          }
          for (int kb = 0; kb < nkb; ++kb) {
            tc::mbar_wait(&empty[stage], ph ^ 1);
            if (leader) tc::mbar_arrive_expect_tx(&full[stage], 2 * STAGE_BYTES);
            uint8_t* sa = smem + stage * STAGE_BYTES;
            tc::tma_load_2d_2sm(sa, &tmA, fullL + stage * 8, kb * BK, m0);
            tc::tma_load_2d_2sm(sa + A_BYTES, &tmB, fullL + stage * 8, kb * BK, vp * 2 * BN + (int)rank * BN);
            if (++stage == STAGES) { stage = 0; ph ^= 1; }
          }
        }
        rp = rpn;
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = tc::idesc_bf16(2 * BM, 2 * BN, false, false);
      int stage = 0, it = 0;
      uint32_t ph = 0;
      for (int qi = 0;; ++qi) {
        if (take(qi, true) < 0) break;
        for (int vp = 0; vp < nvp; ++vp, ++it) {
          const int acc = it & 1;
          tc::mbar_wait_cluster(&tempty[acc], ((it >> 1) & 1) ^ 1);
          tc::fence_after_sync();
          if (vp == 0) fwd_trace(qi, 1);
          const uint32_t d = tbase + acc * 2 * BN;
          for (int kb = 0; kb < nkb; ++kb) {
            tc::mbar_wait_cluster(&full[stage], ph);
            tc::fence_after_sync();
            const uint32_t a = tc::smem_u32(smem + stage * STAGE_BYTES), b = a + A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              tc::mma2_bf16(d, tc::sdesc(a + 32 * k, 16, 1024), tc::sdesc(b + 32 * k, 16, 1024), idesc,
                            (kb | k) != 0);
            tc::mma2_commit(&empty[stage], 3);
            if (++stage == STAGES) { stage = 0; ph ^= 1; }
          }
          tc::mma2_commit(&tfull[acc], 3);
          fwd_trace(qi, vp == 0 ? 2 : 3);
        }
      }
    }
  } else {
    const int q = warp & 3;
    const int set = (warp - 2) >> 2;           // warps 2-5: set 0 (columns 0-127), 6-9: set 1 (128-255)
    const int ethr = 64 + 128 * set;
    uint8_t* stg = smem + STAGES * STAGE_BYTES + set * STG_BYTES;
    const uint32_t tl = tbase + ((uint32_t)(32 * q) << 16) + (uint32_t)(set * BN);
    const uint32_t temptyL = tc::mapa(&tempty[0], 0);
    int it = 0, nrt = 0;
    for (int qi = 0;; ++qi) {
      const int rp = take(qi, false);
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_remote(qemptyL + (qi & 3) * 8);
      if (rp < 0) break;
      const int rt = 2 * rp + (int)rank;
      const long long r = (long long)rt * BM + 32 * q + lane;
      const int info = (r < p.R) ? p.rowinfo[r] : -1;
      float M = neg_inf_f(), sum = 0.f, zb = neg_inf_f(), zl = neg_inf_f();
      float mref = neg_inf_f();
      for (int vp = 0; vp < nvp; ++vp, ++it) {
        const int acc = it & 1;
        const int nt = 2 * vp + set, v0 = nt * BN;
        tc::mbar_wait(&tfull[acc], (it >> 1) & 1);
        tc::fence_after_sync();
        if (threadIdx.x == 64) fwd_trace(qi, vp == 0 ? 4 : 6);
        const uint32_t tcol = tl + acc * 2 * BN;
        const bool have = nt < nvt;             // warp-uniform
        constexpr float kRedo = 60.f;
        if (vp == 0) {
          // the row's P~ offset m_ref: max of the first 32 columns of V tiles 0 (set 0) and 1 (set 1)
          float cm0 = neg_inf_f();
          if (have) {
            float z[32];
            tc::tmem_ld32(tcol, z);
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (v0 + j < p.V) cm0 = fmaxf(cm0, z[j] + (bsm ? sbias[v0 + j] : p.bias[v0 + j]));
          }
          xch[set * BM + 32 * q + lane] = cm0;
          asm volatile("bar.sync 4, 256;" ::: "memory");
          mref = fmaxf(xch[32 * q + lane], xch[BM + 32 * q + lane]);
        }
        float m = neg_inf_f(), s = 0.f;
        if (have) {
          // One TMEM pass: every tile's exp offset is the row's m_ref (one offset per row: the
          // backward's dz is then a per-row scalar times P~); a chunk above m_ref + kRedo redoes the
          // tile with its exact max and raises tscale (the backward then rescales per tile).
          const float zb_prev = zb, zl_prev = zl;
          bool redo = false;
          if (threadIdx.x == ethr) tc::bulk_wait_read0();
          asm volatile("bar.sync %0, 128;" ::"r"(1 + set) : "memory");
          for (int attempt = 0; attempt < 2; ++attempt) {
            if (attempt == 1) {
              if (!__any_sync(0xffffffffu, redo)) break;
              if (lane == 0 && p.tscale) *p.tscale = 1;
              m = neg_inf_f();
#pragma unroll 1
              for (int c = 0; c < 4; ++c) {
                float z[32];
                tc::tmem_ld32(tcol + 32 * c, z);
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (v0 + 32 * c + j < p.V) m = fmaxf(m, z[j] + p.bias[v0 + 32 * c + j]);
              }
              s = 0.f;
              zb = zb_prev; zl = zl_prev;
            }
            float mL = m * RNNT_LOG2E_F;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
              float z[32];
              {
                uint32_t zr[32];
                tc::tmem_ld32_issue(tcol + 32 * c, zr);
                const int vc = v0 + 32 * c;
                float4 b4[8];
                if (bsm) {
                  const float4* bb = reinterpret_cast<const float4*>(sbias + vc);
#pragma unroll
                  for (int j4 = 0; j4 < 8; ++j4) b4[j4] = bb[j4];
                } else {
                  const float4* bb = reinterpret_cast<const float4*>(p.bias + vc);
#pragma unroll
                  for (int j4 = 0; j4 < 8; ++j4) b4[j4] = __ldg(bb + j4);
                }
                tc::tmem_ld32_wait(zr);
#pragma unroll
                for (int j4 = 0; j4 < 8; ++j4) {
                  z[4 * j4] = __uint_as_float(zr[4 * j4]) + b4[j4].x;
                  z[4 * j4 + 1] = __uint_as_float(zr[4 * j4 + 1]) + b4[j4].y;
                  z[4 * j4 + 2] = __uint_as_float(zr[4 * j4 + 2]) + b4[j4].z;
                  z[4 * j4 + 3] = __uint_as_float(zr[4 * j4 + 3]) + b4[j4].w;
                }
              }
              const int vc = v0 + 32 * c;
              if (attempt == 0) {
                float cm = z[0];
#pragma unroll
                for (int j = 1; j < 32; ++j) cm = fmaxf(cm, z[j]);
                if (c == 0) {
                  m = mref;
                  mL = m * RNNT_LOG2E_F;
                }
                if (cm - m > kRedo) redo = true;
                if (__any_sync(0xffffffffu, redo)) break;
              }
              uint32_t pk[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const float e0 = ex2_approx(fmaf(z[2 * j], RNNT_LOG2E_F, -mL));
                const float e1 = ex2_approx(fmaf(z[2 * j + 1], RNNT_LOG2E_F, -mL));
                s += e0 + e1;
                __nv_bfloat162 h2 = __floats2bfloat162_rn(e0, e1);
                pk[j] = *reinterpret_cast<uint32_t*>(&h2);
              }
              {
                uint8_t* sb = stg + (c >> 1) * (STG_BYTES / 2);
                const int row = 32 * q + lane;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                  *reinterpret_cast<uint4*>(sb + sw128f(row, (c & 1) * 4 + j)) =
                      make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
              }
              if (vc == 0) zb = z[0];
              const int li = info - vc;
              const bool hit = (unsigned)li < 32u;
              if (__any_sync(0xffffffffu, hit)) {
                float zz[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) zz[j] = z[j];
                if (hit) zl = zz[li];
              }
            }
          }
        }
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_remote(temptyL + acc * 8);
        if (threadIdx.x == 64) fwd_trace(qi, vp == 0 ? 5 : 7);
        if (have) {
          tc::fence_proxy_async();
          asm volatile("bar.sync %0, 128;" ::"r"(1 + set) : "memory");
          if (threadIdx.x == ethr && (long long)rt * BM < p.R) {
            tc::tma_store_2d(&tmP, stg, v0, rt * BM);
            tc::tma_store_2d(&tmP, stg + STG_BYTES / 2, v0 + 64, rt * BM);
            tc::bulk_commit();
          }
          if (info >= 0) p.mt[(size_t)r * p.ntile + v0 / 128] = m;
          const float Mn = fmaxf(M, m);
          sum = sum * ex2_approx((M - Mn) * RNNT_LOG2E_F) + s * ex2_approx((m - Mn) * RNNT_LOG2E_F);
          M = Mn;
        }
      }
      // merge set 1's running state into set 0's (double-buffered by row-tile parity)
      float4* mb = mrg + (nrt & 1) * BM;
      if (set == 1) mb[32 * q + lane] = make_float4(M, sum, zb, zl);
      asm volatile("bar.sync 3, 256;" ::: "memory");
      if (set == 0 && r < p.R) {
        const float4 o = mb[32 * q + lane];
        const float Mn = fmaxf(M, o.x);
        const float tot = sum * ex2_approx((M - Mn) * RNNT_LOG2E_F) + o.y * ex2_approx((o.x - Mn) * RNNT_LOG2E_F);
        const float zlab = fmaxf(zl, o.w);   // the label's column lies in exactly one set's tiles
        if (info >= 0) {
          const float l = Mn + lg2_approx(tot) * RNNT_LN2_F;
          p.lse[r] = l;
          p.py2[r] = (zb - l) * RNNT_LOG2E_F;
          p.px2[r] = info < p.V ? (zlab - l) * RNNT_LOG2E_F : kNegBig;
        } else {
          p.lse[r] = 0.f;
          p.px2[r] = kNegBig;
          p.py2[r] = kNegBig;
        }
      }
      if (threadIdx.x == 64) fwd_trace(qi, 8);
      ++nrt;
    }
  }
  if (warp >= 2 && (threadIdx.x & 127) == 64) tc::bulk_wait0();
  tc::fence_before_sync();
  __syncthreads();
  tc::cluster_sync();
  if (warp == 1) tc::tmem_dealloc2(tbase, 512);
}

cudaError_t joiner_fwd_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, const uint16_t* W,
                              const uint16_t* b, cudaStream_t st) {
  const long long R = d.rows();
  const int VP = d.VP();
  CUtensorMap ta, tb, tp;
  if (!make_tmap_bf16_2d(&ta, h, d.J, R, (uint64_t)d.J * 2, jf::BK, jf::BM)) return cudaErrorInvalidValue;
  if (!make_tmap_bf16_2d(&tb, W, d.J, d.V, (uint64_t)d.J * 2, jf::BK, jf::BN)) return cudaErrorInvalidValue;
  if (!make_tmap_bf16_2d(&tp, w.Pt, VP, R, (uint64_t)VP * 2, 64, jf::BM)) return cudaErrorInvalidValue;
  const int ntiles = (int)((R + jf::BM - 1) / jf::BM);
  JoinerFwdParams p{w.bias, w.bmax, w.rowinfo, w.tlive, w.tcounter, R, ntiles, d.V, VP, d.J, (d.V + jf::BN - 1) / jf::BN,
                    (d.J + jf::BK - 1) / jf::BK, d.ntile(), w.Pt, w.mt, w.lse, w.px2, w.py2, 0, w.tscale};
#ifdef RNNT_DIAGNOSTICS
  if (const char* e = getenv("RNNT_DBG_FWD")) p.dbg = atoi(e);  // skips parts of the step: wrong results, timing only
#endif
  const int nsm = current_sm_count();
  static const int pair = env_int("RNNT_FWD_PAIR", 1);
  if (pair) {
    smem_optin(joiner_fwd_pair_kernel, jf2::SMEM_BYTES);
    // persistent: one CTA per SM, in pairs (at most one cluster per row-tile pair); the pair counter is
    // the row-tile counter rowinfo_kernel zeroes
    const unsigned grid = (unsigned)(2 * std::min((ntiles + 1) / 2, nsm / 2));
    RNNT_LAUNCH(KID_JOINER_FWD, st, launch_pdl(joiner_fwd_pair_kernel, grid, jf2::THREADS, jf2::SMEM_BYTES, st, ta, tb, tp, p));
    return cudaGetLastError();
  }
  smem_optin(joiner_fwd_tc_kernel, jf::SMEM_BYTES);
  const unsigned grid = (unsigned)std::min(ntiles, nsm);   // persistent: one CTA per SM
  RNNT_LAUNCH(KID_JOINER_FWD, st, launch_pdl(joiner_fwd_tc_kernel, grid, jf::THREADS, jf::SMEM_BYTES, st, ta, tb, tp, p));
  return cudaGetLastError();
}

}  // namespace rnnt
