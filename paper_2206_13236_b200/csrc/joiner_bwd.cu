// joiner_bwd.cu — K10 / K11: joiner backward on tcgen05 with the logit gradient formed inside the
// GEMM operand tiles (function merging): nothing of size (R, V) is written in the
// backward.  P~ (bf16 exp(z - m_tile), from K8) is brought into the swizzled shared-memory operand
// tile by TMA, and the producer warps turn it IN PLACE into
//     dz[r,v] = sc[r, v/128] * P~[r,v] - gs g_b[r] [v=0] - gs g_l[r] [v=y_r]      (bf16)
// (the element-wise transform preserves the SWIZZLE_128B layout: logical 16-B chunk c of tile row r
// sits at physical chunk c ^ (r % 8)), then release the stage to the MMA issuer.
//
//   K10 joiner_dh:  dh[r, j] = sum_v dz[r,v] W[v,j]     A = dz (K-major), B = W (MN-major);
//                   epilogue dpre = dh (1 - h^2)  (d tanh)
//   K11 joiner_dw:  dW[v, j] = sum_r dz[r,v] h[r,j]     A = dz^T (MN-major), B = h (MN-major);
//                   split-K over rows, fp32 partial tiles; the producers also sum db partials.
// Warps 0-3: in-place producers, then epilogue (TMEM lanes 32w..32w+31).
// Warp 4: TMEM allocator, TMA issuer (one lane) and MMA issuer (another lane).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"
#include "tc.cuh"
#include "tmap.h"
#include "workspace.h"

namespace rnnt {

struct GradSrc {
  const uint16_t* Pt;
  const float4* gpk;       // (ntile, R) {sc, gs g_b, gs g_l, label bits}, written by pruned_combine
  const int32_t* rowinfo;
  long long R;
  int V, VP, ntile;
};

// dz for the 8 logits v = vc..vc+7 of one row, from the packed bf16 P~ chunk `pv`, the row's
// scale s, the picks gbs = gs g_b (v = 0) and gls = gs g_l (v = label `info`).  Returns the bf16
// chunk and adds the bf16-rounded values (what the MMA consumes) to fsum when given.
__device__ __forceinline__ uint4 dz_chunk(uint4 pv, float s, float gbs, float gls, int info, int vc, float* fsum,
                                         bool rare = false) {
  // The blank pick is warp-uniform (vc).  The label pick: a compare and select on every element, or,
  // when `rare` (large V: a row's label falls in one of V/8 chunks, so the branch is almost never
  // taken), a per-lane branch (measured: c4 dW 2144 -> 2020 us; at V = 500 the branch costs more)
  const uint32_t w[4] = {pv.x, pv.y, pv.z, pv.w};
  const int li = info - vc;
  float g[8];
  if (rare) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      g[2 * i] = s * __uint_as_float(w[i] << 16);
      g[2 * i + 1] = s * __uint_as_float(w[i] & 0xffff0000u);
    }
    if ((unsigned)li < 8u) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (li == k) g[k] -= gls;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      g[2 * i] = s * __uint_as_float(w[i] << 16) - (li == 2 * i ? gls : 0.f);
      g[2 * i + 1] = s * __uint_as_float(w[i] & 0xffff0000u) - (li == 2 * i + 1 ? gls : 0.f);
    }
  }
  if (vc == 0) g[0] -= gbs;
  uint32_t o[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h2 = __floats2bfloat162_rn(g[2 * i], g[2 * i + 1]);
    o[i] = *reinterpret_cast<uint32_t*>(&h2);
    if (fsum) {
      fsum[2 * i] += __low2float(h2);
      fsum[2 * i + 1] += __high2float(h2);
    }
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}

// s * P~ for the 8 logits of one chunk, in packed bf16 arithmetic: s = s_hi + s_lo (two bf16), and
//   dz = bf16_rn(P~ s_hi + bf16_rn(P~ s_lo))
// (the inner product's rounding is ~2^-17 of the result, so this is within one bf16 rounding of the
// fp32 product: two HFMA2 per pair of logits, no unpacking).  The picks (-gs g_b at v = 0, -gs g_l at
// v = y) touch two logits of a row: pick_elem recomputes those in fp32 (rare, per-lane branch).
__device__ __forceinline__ uint32_t bf16x2_splat(float x) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ uint32_t bf16x2_scale(uint32_t p, uint32_t shi, uint32_t slo) {
  uint32_t lo, d;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(lo) : "r"(p), "r"(slo));
  asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(p), "r"(shi), "r"(lo));
  return d;
}
__device__ __forceinline__ uint4 dz_scale_chunk(uint4 pv, uint32_t shi, uint32_t slo) {
  return make_uint4(bf16x2_scale(pv.x, shi, slo), bf16x2_scale(pv.y, shi, slo), bf16x2_scale(pv.z, shi, slo),
                    bf16x2_scale(pv.w, shi, slo));
}
// byte offset of logical 16-B chunk `c` (0..7) of 128-B row `r` in a SWIZZLE_128B atom stack
__device__ __forceinline__ uint32_t sw128(int r, int c) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}

// ======================================================================= K10
// joiner_dh: dh = dz W over (live 128-row tile, 256-column part of J) work items, persistent, every
// role pipelined across items:
//   warp 0      lane 0: TMA producer: per 64-logit k-block the P~ tile, the W boxes and the rows' packed
//               scalars into a 4-stage ring (the item's h boxes are prefetched into L2 at its start,
//               the epilogue reads its rows of h from there)
//   warp 1      TMEM allocator (2 x 256 columns) and single-thread MMA issuer
//   warps 2..   in-place dz producers (4 or 8 warps: a thread per row or half row), release each
//               stage to the MMA
//   4 epilogue  one per TMEM lane quadrant, thread = tile row, 32-column chunks: dpre = dh (1 - h^2)
//   warps       into a swizzled 16 KB smem tile, written to the fp32 dpre (R, J) by one TMA store per
//               chunk; the accumulator of item k+1 fills while item k drains.
// The reductions d_enc[t] = sum_s dpre[(t,s)] and d_dec[u] = sum_{t: p_t <= u < p_t + S} dpre[(t, u - p_t)]
// run afterwards in band_reduce_kernel (pruned.cu): a streaming pass at HBM speed, deterministic, that
// keeps this kernel's epilogue far shorter than its mainloop.
namespace jdh {
constexpr int BM = 128, BK = 64, NSUB = 256;
constexpr int A_BYTES = BM * BK * 2;           // 16 KB, K-major (TMA box 64 v x 128 rows of P~)
constexpr int B_BYTES = NSUB * BK * 2;         // 32 KB, MN-major (4 boxes of 64 j x 64 v)
constexpr int G_BYTES = BM * 16;               // 2 KB: the rows' packed scalars for this k-block's V tile
constexpr int STAGE_BYTES = A_BYTES + B_BYTES + G_BYTES;   // 50 KB (1024-aligned)
constexpr int H_BYTES = BM * 64 * 2;           // one 64-column box of h (SWIZZLE_128B)
// Shared memory per variant.  Short V loops (4 producer warps, item = a few k-blocks): 3 stages, h by
// TMA into a 2-slot ring (3 slots with fp16 dpre rows, whose staging tiles are half the size: the
// epilogue waited on the h box loads for 15 % of its stall samples at c5), 2 dpre staging tiles (the
// epilogue is on the critical path).  Long V loops (8 producer warps): 4 stages (the per-stage chain
// load -> dz transform -> MMA is what bounds the mainloop), h read from L2 by the epilogue, 1 staging tile.
template <int NTW, bool D16> struct Cfg {
  static constexpr int STAGES = NTW == 8 ? 4 : 3;
  static constexpr int HRING = NTW == 8 ? 0 : (D16 ? 3 : 2);
  static constexpr int ORING = NTW == 8 ? 1 : 2;
  static constexpr int O_BYTES = BM * 32 * (D16 ? 2 : 4);   // one 32-column dpre chunk (128 rows)
  static constexpr int H_OFF = STAGES * STAGE_BYTES;
  static constexpr int O_OFF = H_OFF + HRING * H_BYTES;
  static constexpr int BAR_OFF = O_OFF + ORING * O_BYTES;
  static constexpr int SMEM_BYTES = BAR_OFF + 256 + 1024;
};
constexpr int kMaxHRing = 4;
// in-place dz producer warps: 4 (a thread per row) for short V loops, 8 (a thread per half row) when
// the mainloop is long
template <int NTW> struct Roles {
  static constexpr int EPI0 = 2 + NTW;          // first epilogue warp (4: quadrant = warp % 4)
  static constexpr int THREADS = (EPI0 + 4) * 32;
};
}  // namespace jdh

struct JoinerDhParams {
  GradSrc g;
  const uint16_t* h;       // (R, J) bf16 joiner input (the epilogue's 1 - h^2)
  int J, nkb, njp;
  const int* live;         // ids of the 128-row tiles with a live row (order irrelevant)
  const int* nlive;        // their count
  float* dpre;             // (R, J) fp32 out: dh (1 - h^2) of the rows of the live tiles
  int w3;                  // tmW is the 3-D (64 j, V, J/64) map: one TMA per k-block's 4 W boxes
  const int* tscale;       // PrunedWS::tscale: 0 -> plain mode (null: always rescale P~ per tile)
  const float* gsp;        // non-null: dpre is stored as fp16 dpre / *gsp (the pruned path); null: fp32
};

// diagnostics: per (CTA, item) timestamps {producer start, first MMA, last MMA commit, epilogue
// start (accumulator full), epilogue end}; 16 items per CTA
#ifdef RNNT_DIAGNOSTICS
__device__ unsigned long long* g_dh_trace = nullptr;
void set_dh_trace(void* buf) { cudaMemcpyToSymbol(g_dh_trace, &buf, sizeof(buf)); }
#else
constexpr unsigned long long* g_dh_trace = nullptr;   // product build: tracing compiled out
#endif
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void dh_trace(int it, int k) {
  if (g_dh_trace && it < 16) g_dh_trace[((size_t)blockIdx.x * 16 + it) * 5 + k] = gtimer();
}
// per (CTA, item < 3, k-block < 8): {TMA issued, stage seen loaded, transformed, MMA issued}
__device__ __forceinline__ void dh_trace_kb(int it, int kb, int k) {
  if (g_dh_trace && it < 3 && kb < 8) g_dh_trace[148 * 16 * 5 + (((size_t)blockIdx.x * 3 + it) * 8 + kb) * 4 + k] = gtimer();
}

// MC: clusters of two CTAs working on two row tiles with the same 256-column part of J in lockstep;
// each CTA TMA-loads half of every W k-block with .multicast::cluster into both CTAs' stage, so the
// L2 -> SM traffic per MMA drops from 50 to 34 KB per k-block (the contraction is L2-bandwidth bound at
// large V).  A stage is refilled once both CTAs' MMAs released it (each MMA commit arrives on both
// CTAs' empty barrier).
template <int NTW, bool MC, bool D16>
__global__ void __launch_bounds__(jdh::Roles<NTW>::THREADS, 1)
    joiner_dh_tc_kernel(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmW,
                        const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmD,
                        JoinerDhParams p) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  using namespace jdh;
  constexpr int EPI0 = Roles<NTW>::EPI0;
  using C = Cfg<NTW, D16>;
  constexpr int STAGES = C::STAGES, HRING = C::HRING, ORING = C::ORING, O_BYTES = C::O_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = tc::align1024(smem_raw);
  uint64_t* loaded = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* full = loaded + STAGES;
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;       // [2]
  uint64_t* tempty = tfull + 2;           // [2]
  uint64_t* hfull = tempty + 2;           // [HRING] (HRING > 0)
  uint64_t* hempty = hfull + kMaxHRing;   // [HRING]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hempty + kMaxHRing);
  uint8_t* hbuf = smem + C::H_OFF;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // work items: (row tile, 256-column part); with MC a cluster takes (tile pair, part) items, rank r the
  // tile 2 i + r (an odd last tile is done by both CTAs: identical values, written twice)
  const int nlive = *p.nlive;
  // plain mode (one P~ offset per row, picks folded into P~ by pruned_combine): dh = sc_r (P~' W), the
  // MMA consumes the TMA'd stage directly and the epilogue applies the row scalar; no transform warps
  const bool plain = p.tscale && *p.tscale == 0;
  // plain + two staging tiles: the idle transform warps (2..5) become a second epilogue set; set e takes
  // the 32-column chunks of parity e (both sets share each h box) and stages through tile e
  const bool dual = plain && NTW == 4 && ORING == 2;
  const int crank = MC ? (int)tc::cluster_ctarank() : 0;
  const long long cid = MC ? blockIdx.x / 2 : blockIdx.x, ncl = MC ? gridDim.x / 2 : gridDim.x;
  const long long nitems = (long long)(MC ? (nlive + 1) / 2 : nlive) * p.njp;
  auto item_tile = [&](long long idx) {
    const long long pi = idx / p.njp;
    return MC ? p.live[min(2 * pi + crank, (long long)nlive - 1)] : p.live[pi];
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&loaded[s], 1);
      tc::mbar_init(&full[s], NTW);
      tc::mbar_init(&empty[s], MC ? 2 : 1);   // MC: both CTAs' MMA commits
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&tfull[s], 1);
      tc::mbar_init(&tempty[s], dual ? 8 : 4);      // the epilogue warps
    }
    for (int s = 0; s < HRING; ++s) {
      tc::mbar_init(&hfull[s], 1);
      tc::mbar_init(&hempty[s], dual ? 8 : 4);
    }
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmP);
    tc::tma_prefetch(&tmW);
    tc::tma_prefetch(&tmH);
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * NSUB);
  tc::fence_before_sync();
  __syncthreads();
  if (MC) tc::cluster_sync();             // the peer's barriers are initialised before any multicast
  tc::fence_after_sync();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer
      int stage = 0, it = 0;
      uint32_t ph = 0;
      for (long long idx = cid; idx < nitems; idx += ncl, ++it) {
        const int tile = item_tile(idx), jp = (int)(idx % p.njp);
        dh_trace(it, 0);
        const long long m0 = (long long)tile * BM;
        const int j0 = jp * NSUB, nbox = (min(NSUB, p.J - j0) + 63) / 64;
        const int grows = (int)min((long long)BM, p.g.R - m0);
        // (3-D W box: planes past J arrive zero-filled and count in full)
        const uint32_t gbytes = plain ? 0u : (uint32_t)grows * 16u;
        const uint32_t bytes = A_BYTES + (p.w3 ? (uint32_t)B_BYTES : (uint32_t)nbox * 64 * BK * 2) + gbytes;
        constexpr int PF = 8;            // P~ boxes prefetched into L2 this many k-blocks ahead
        for (int kb = 0; kb < min(PF, p.nkb); ++kb) tc::tma_prefetch_2d(&tmP, kb * BK, (int)m0);
        // the epilogue's h boxes of this item: into L2 now, a mainloop ahead of their TMA loads
        for (int bx = 0; bx < nbox; ++bx) tc::tma_prefetch_2d(&tmH, j0 + bx * 64, (int)m0);
        for (int kb = 0; kb < p.nkb; ++kb) {
          if (kb + PF < p.nkb) tc::tma_prefetch_2d(&tmP, (kb + PF) * BK, (int)m0);
          tc::mbar_wait(&empty[stage], ph ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          dh_trace_kb(it, kb, 0);
          tc::mbar_arrive_expect_tx(&loaded[stage], bytes);
          tc::tma_load_2d(sa, &tmP, &loaded[stage], kb * BK, (int)m0);
          if (MC) {                      // this CTA's half of the W boxes, into both CTAs' stage
            if (p.w3) {
              tc::tma_load_3d_mc(sa + A_BYTES + crank * 2 * (64 * BK * 2), &tmW, &loaded[stage], 0, kb * BK,
                                 j0 / 64 + 2 * crank, 3);
            } else {
              for (int bx = crank; bx < nbox; bx += 2)
                tc::tma_load_2d_mc(sa + A_BYTES + bx * (64 * BK * 2), &tmW, &loaded[stage], j0 + bx * 64, kb * BK, 3);
            }
          } else if (p.w3) {
            tc::tma_load_3d(sa + A_BYTES, &tmW, &loaded[stage], 0, kb * BK, j0 / 64);
          } else {
            for (int bx = 0; bx < nbox; ++bx)
              tc::tma_load_2d(sa + A_BYTES + bx * (64 * BK * 2), &tmW, &loaded[stage], j0 + bx * 64, kb * BK);
          }
          if (gbytes)
            tc::bulk_load(sa + A_BYTES + B_BYTES, p.g.gpk + (size_t)((kb * BK) >> 7) * p.g.R + m0, gbytes,
                          &loaded[stage]);
          if (++stage == STAGES) { stage = 0; ph ^= 1; }
        }
      }
    } else if (lane == 1 && HRING > 0) {
      // ---- h boxes for the epilogue: box i (columns j0 + 64 i) serves chunks 2i and 2i+1
      int slot = 0;
      uint32_t ph = 0;
      for (long long idx = cid; idx < nitems; idx += ncl) {
        const int tile = item_tile(idx), jp = (int)(idx % p.njp);
        const int m0 = tile * BM, j0 = jp * NSUB;
        const int nbox = (min(NSUB, p.J - j0) + 63) / 64;
        for (int bx = 0; bx < nbox; ++bx) {
          tc::mbar_wait(&hempty[slot], ph ^ 1);
          tc::mbar_arrive_expect_tx(&hfull[slot], H_BYTES);
          tc::tma_load_2d(hbuf + slot * H_BYTES, &tmH, &hfull[slot], j0 + bx * 64, m0);
          if (++slot == HRING) { slot = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer
      constexpr uint32_t idesc = tc::idesc_bf16(BM, NSUB, false, true);
      int stage = 0, it = 0;
      uint32_t ph = 0;
      for (long long idx = cid; idx < nitems; idx += ncl, ++it) {
        const int acc = it & 1;
        tc::mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc::fence_after_sync();
        const uint32_t d = tbase + acc * NSUB;
        for (int kb = 0; kb < p.nkb; ++kb) {
          tc::mbar_wait(plain ? &loaded[stage] : &full[stage], ph);
          tc::fence_after_sync();
          if (kb == 0) dh_trace(it, 1);
          dh_trace_kb(it, kb, 3);
          const uint32_t a = tc::smem_u32(smem + stage * STAGE_BYTES), b = a + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            tc::mma_bf16(d, tc::sdesc(a + 32 * k, 16, 1024), tc::sdesc(b + 2048 * k, 64 * BK * 2, 1024), idesc,
                         (kb | k) != 0);
          if (MC) tc::mma_commit_mc(&empty[stage], 3);   // releases the stage in both CTAs
          else tc::mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; ph ^= 1; }
        }
        tc::mma_commit(&tfull[acc]);
        dh_trace(it, 2);
      }
    }
  } else if (warp < EPI0 && !dual) {
    // ---- in-place dz producers: thread = (tile row, half): transforms 4 or 8 of the 8 chunks of its row
    constexpr int CPT = 8 * 4 / NTW;                 // chunks per thread: 8 (4 warps) or 4 (8 warps)
    const int pt = threadIdx.x - 64;
    const int rl = pt & 127, c_lo = (pt >> 7) * CPT;
    int stage = 0, itx = 0;
    uint32_t ph = 0;
    for (long long idx = plain ? nitems : cid; idx < nitems; idx += ncl, ++itx) {
      const int tile = item_tile(idx);
      const long long m0 = (long long)tile * BM;
      const int grows = (int)min((long long)BM, p.g.R - m0);
      for (int kb = 0; kb < p.nkb; ++kb) {
        const int v0 = kb * BK;
        tc::mbar_wait(&loaded[stage], ph);
        if (pt == 0) dh_trace_kb(itx, kb, 1);
        uint8_t* sa = smem + stage * STAGE_BYTES;
        const float4 gq = rl < grows ? reinterpret_cast<const float4*>(sa + A_BYTES + B_BYTES)[rl]
                                     : make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
        const int info = __float_as_int(gq.w);
        const uint32_t shi = bf16x2_splat(gq.x);
        const uint32_t slo = bf16x2_splat(gq.x - __uint_as_float(shi << 16));
        // the picks (-gs g_b at v = 0, -gs g_l at v = y; labels are >= 1) touch one logit each: read
        // it before the chunk stores, recompute bf16_rn(P~ s - g) in fp32, write it back after them
        const int lv = info - (v0 + c_lo * 8);
        const bool plab = (unsigned)lv < (unsigned)(CPT * 8);
        const bool pblk = v0 == 0 && c_lo == 0 && info >= 0;
        __nv_bfloat16* lp = reinterpret_cast<__nv_bfloat16*>(sa + sw128(rl, c_lo + (plab ? lv >> 3 : 0)) + (plab ? lv & 7 : 0) * 2);
        __nv_bfloat16* bp = reinterpret_cast<__nv_bfloat16*>(sa + sw128(rl, 0));
        const float lx = plab ? __bfloat162float(*lp) * gq.x - gq.z : 0.f;
        const float bx = pblk ? __bfloat162float(*bp) * gq.x - gq.y : 0.f;
        uint4 pv[CPT];
#pragma unroll
        for (int c = 0; c < CPT; ++c) pv[c] = *reinterpret_cast<const uint4*>(sa + sw128(rl, c_lo + c));
#pragma unroll
        for (int c = 0; c < CPT; ++c)
          *reinterpret_cast<uint4*>(sa + sw128(rl, c_lo + c)) =
              info >= 0 ? dz_scale_chunk(pv[c], shi, slo) : make_uint4(0, 0, 0, 0);
        if (plab) *lp = __float2bfloat16_rn(lx);
        if (pblk) *bp = __float2bfloat16_rn(bx);
        tc::fence_proxy_async();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&full[stage]);
        if (pt == 0) dh_trace_kb(itx, kb, 2);
        if (++stage == STAGES) { stage = 0; ph ^= 1; }
      }
    }
  } else {
    // ---- epilogue: quadrant q4 = warp % 4 = TMEM lanes 32 q4 ..; thread = tile row, per 32-column chunk
    // dpre = dh (1 - h^2) -> its row of dpre (128 B per chunk).  dual: set 1 = warps 2..5, chunks of
    // odd parity, staging tile 1, named barrier 2
    const int eset = warp >= EPI0 ? 0 : 1;
    const int q4 = warp & 3;
    const int rl = 32 * q4 + lane;
    const uint32_t tl = tbase + ((uint32_t)(32 * q4) << 16);
    const bool leader = warp == (eset ? 2 : EPI0) && lane == 0;   // issues the set's TMA stores
    // fp16 rows (the pruned path): dpre / gs, so the stored range does not depend on the loss scale
    constexpr bool d16 = D16;   // (p.gsp != nullptr)
    float dsc = 1.f;
    if (d16) {
      const float gsv = *p.gsp;
      if (gsv != 0.f && isfinite(gsv)) dsc = 1.f / gsv;
    }
    int it = 0, hslot = 0;
    uint32_t hph = 0;
    long long kc = 0;                                     // chunk counter: staging tile kc % ORING
    // the row's label info and (plain) scalar of the NEXT item are loaded while this item drains: their
    // dependent global loads (live list -> rowinfo / gpk) sat on the item start otherwise
    int ninfo = -1;
    float nsc = 0.f;
    auto prefetch_row = [&](long long ix) {
      ninfo = -1;
      nsc = 0.f;
      if (ix >= nitems) return;
      const long long rr = (long long)item_tile(ix) * BM + rl;
      if (rr < p.g.R) {
        ninfo = p.g.rowinfo[rr];
        if (plain) nsc = p.g.gpk[rr].x;
      }
    };
    prefetch_row(cid);
    for (long long idx = cid; idx < nitems; idx += ncl, ++it) {
      const int tile = item_tile(idx), jp = (int)(idx % p.njp);
      const int acc = it & 1;
      const long long r = (long long)tile * BM + rl;
      const bool live = ninfo >= 0;                          // (r < R: else the prefetch left -1)
      const float sc = plain && live ? nsc : 1.f;            // plain: the row scalar (tile 0's = every tile's)
      prefetch_row(idx + ncl);
      const int j0 = jp * NSUB, nj = min(NSUB, p.J - j0);
      const int nbox = (nj + 63) / 64;
      tc::mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc::fence_after_sync();
      if (warp == EPI0 && lane == 0) dh_trace(it, 3);
      for (int ch = dual ? eset : 0; ch < 2 * nbox; ch += dual ? 2 : 1) {
        const int c0 = 32 * ch;
        const bool have = c0 < nj;
        const int nq = have ? min(4, (nj - c0) / 8) : 0;   // J % 8 == 0
        uint4 hv[4];                                       // this row's h for the chunk
        if (HRING > 0) {
          if (dual || (ch & 1) == 0) tc::mbar_wait(&hfull[hslot], hph);
          const uint8_t* hb = hbuf + hslot * H_BYTES;
#pragma unroll
          for (int qq = 0; qq < 4; ++qq)
            hv[qq] = (qq < nq && live) ? *reinterpret_cast<const uint4*>(hb + sw128(rl, 4 * (ch & 1) + qq))
                                       : make_uint4(0, 0, 0, 0);
        } else {                                           // (L2-resident: prefetched at the item's start)
#pragma unroll
          for (int qq = 0; qq < 4; ++qq)
            hv[qq] = (qq < nq && live) ? __ldg(reinterpret_cast<const uint4*>(p.h + (size_t)r * p.J + j0 + c0) + qq)
                                       : make_uint4(0, 0, 0, 0);
        }
        float accv[32];
        if (have) tc::tmem_ld32(tl + acc * NSUB + c0, accv);
        if (ch + (dual ? 2 : 1) >= 2 * nbox) {           // last TMEM read of this accumulator
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&tempty[acc]);
        }
        float out[32];
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const uint32_t hw[4] = {hv[qq].x, hv[qq].y, hv[qq].z, hv[qq].w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float ha = __uint_as_float(hw[i] << 16), hb2 = __uint_as_float(hw[i] & 0xffff0000u);
            const bool ok = qq < nq && live;
            out[8 * qq + 2 * i] = ok ? (accv[8 * qq + 2 * i] * sc) * (1.f - ha * ha) : 0.f;       // d tanh
            out[8 * qq + 2 * i + 1] = ok ? (accv[8 * qq + 2 * i + 1] * sc) * (1.f - hb2 * hb2) : 0.f;
          }
        }
        if (HRING > 0 && (dual || (ch & 1) == 1 || ch == 2 * nbox - 1)) {   // both halves of this h box are used
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&hempty[hslot]);
          if (++hslot == HRING) { hslot = 0; hph ^= 1; }
        }
        if (!have) continue;
        // staging tile kc % ORING: the TMA store issued from it ORING chunks ago has finished reading it
        uint8_t* ob = smem + C::O_OFF + (dual ? eset : (int)(kc % ORING)) * O_BYTES;
        if (leader) {
          if (ORING == 2 && !dual) tc::bulk_wait_read1();
          else tc::bulk_wait_read0();
        }
        asm volatile("bar.sync %0, 128;" ::"r"(1 + eset) : "memory");
        if (d16) {   // 128 rows x 64 B, SWIZZLE_64B: 16-B chunk qq of row rl at qq ^ ((rl >> 1) & 3)
          uint4* O = reinterpret_cast<uint4*>(ob);
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            uint32_t w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const __half2 h2 = __floats2half2_rn(out[8 * qq + 2 * i] * dsc, out[8 * qq + 2 * i + 1] * dsc);
              w[i] = *reinterpret_cast<const uint32_t*>(&h2);
            }
            O[rl * 4 + (qq ^ ((rl >> 1) & 3))] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        } else {
          float4* O4 = reinterpret_cast<float4*>(ob);
#pragma unroll
          for (int qq = 0; qq < 8; ++qq)
            O4[rl * 8 + (qq ^ (rl & 7))] = make_float4(out[4 * qq], out[4 * qq + 1], out[4 * qq + 2], out[4 * qq + 3]);
        }
        tc::fence_proxy_async();
        asm volatile("bar.sync %0, 128;" ::"r"(1 + eset) : "memory");
        if (leader) {
          tc::tma_store_3d(&tmD, ob, j0 + c0, tile * BM, 0);
          tc::bulk_commit();
        }
        ++kc;
      }
      if (warp == EPI0 && lane == 0) dh_trace(it, 4);
    }
    if (leader) tc::bulk_wait0();                         // every dpre store complete
  }
  tc::fence_before_sync();
  __syncthreads();
  if (MC) tc::cluster_sync();             // no multicast write or arrive targets an exited peer
  if (warp == 1) tc::tmem_dealloc(tbase, 2 * NSUB);
}

// ======================================================================= K11
namespace jdw {
// 2 stages (~108 KB smem, TMEM 256 columns): two CTAs per SM keep four stages in flight per SM.
// PAIR: a CTA pair (cluster of 2, cta_group::2) computes a 256 (v) x 256 (j) dW tile: each CTA holds
// its own 128 v of dz^T and HALF of the h columns (128 j), so the L2 -> SM bytes per flop of the h
// operand halve; the rank-0 CTA issues the MMAs, both CTAs transform their own dz tile.
constexpr int BM = 128, BN = 256, BK = 64;
constexpr int A_BYTES = BM * BK * 2;     // 16 KB, MN-major (2 TMA boxes of 64 v x 64 rows of P~)
constexpr int G_BYTES = BK * 16;         // 1 KB: the k-block rows' packed scalars for this V tile
// B: 4 boxes of 64 j x 64 rows of h (32 KB); a pair CTA holds 2 (16 KB), which buys a third stage
template <bool PAIR> struct Cfg {
  static constexpr int STAGES = PAIR ? 3 : 2;
  static constexpr int B_BYTES = (PAIR ? BN / 2 : BN) * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES + G_BYTES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256 + 128 * 16 * 4;
};
constexpr int THREADS = 160;
}  // namespace jdw

struct JoinerDwParams {
  GradSrc g;
  int J;
  long long kb_per_split, nkb_total;   // (unused when `live` is set: the split is derived on device)
  const int* live;   // ascending ids of the 128-row tiles with a live row, count at nlive (null: all rows)
  const int* nlive;
  const int* tscale; // PrunedWS::tscale (wide variant): 0 -> plain GEMM d_w = P~'^T Hs (null: always rescale)
  float* dWp;   // (splits, V, J)
  float* dbp;   // (splits, V)
  int pf = 6, pfmode = 1;   // wide variant: L2 prefetch distance (k-blocks); bit 0: P~ prefetched by j-tile 0 only, h by V pair 0 only; bit 1: grid x = j tile
  int h3 = 0;               // wide variant: tmH is the 3-D (64 j, rows, J/64) map (J % 64 == 0)
  int hsmem = 0;            // plain mode: Hs = bf16(sc h) formed in shared memory (else the precomputed Hs map)
  int mc = 0;               // wide variant: P~ multicast over clusters of this many J-part siblings (0/1: off)
  int pair_plain = 0;       // wide variant: the plain mode is left to joiner_dw_pair_kernel (it runs only then)
};


// The k-blocks (64 rows) of split `split`: with a live-tile list, the 2 nlive k-blocks of the live
// 128-row tiles in ascending row order, cut into gridDim.z equal ranges (dead tiles -- padded frames of
// short utterances -- are never read); else rows [kb0 BK, kb1 BK).
struct DwRange {
  long long kb0;
  int nkb;
};
__device__ __forceinline__ DwRange dw_range(const JoinerDwParams& p, int split, int splits) {
  if (p.live) {
    const long long tot = 2LL * *p.nlive, per = (tot + splits - 1) / splits;
    const long long k0 = (long long)split * per;
    return {k0, (int)max(0LL, min(tot, k0 + per) - k0)};
  }
  const long long k0 = (long long)split * p.kb_per_split;
  return {k0, (int)max(0LL, min(p.nkb_total, k0 + p.kb_per_split) - k0)};
}
__device__ __forceinline__ long long dw_row0(const JoinerDwParams& p, long long kb) {
  return p.live ? (long long)p.live[kb >> 1] * 128 + (kb & 1) * 64 : kb * 64;
}
// rows of the k-block starting at rb that exist (the last tile may end inside its first half)
__device__ __forceinline__ int dw_rows(const JoinerDwParams& p, long long rb) {
  return (int)max(0LL, min(64LL, p.g.R - rb));
}

template <bool PAIR>
__global__ void __launch_bounds__(jdw::THREADS, 2)
    joiner_dw_tc_kernel(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmH,
                        JoinerDwParams p) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  using namespace jdw;
  constexpr int STAGES = Cfg<PAIR>::STAGES, B_BYTES = Cfg<PAIR>::B_BYTES, STAGE_BYTES = Cfg<PAIR>::STAGE_BYTES;
  auto stage_of = [](int kb) { return kb % STAGES; };
  auto phase_of = [](int kb) { return (uint32_t)((kb / STAGES) & 1); };
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = tc::align1024(smem_raw);
  uint64_t* loaded = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* full = loaded + STAGES;
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  float* dbs = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256);     // [8 row groups][128 v]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool rare = p.g.V >= 6144;     // dz_chunk label pick by branch (measured: c4 -6 %, c3 (Zipf labels) +5 %)
  const uint32_t rank = PAIR ? tc::cluster_ctarank() : 0;
  const int v0 = blockIdx.x * BM, j0 = blockIdx.y * BN, split = blockIdx.z;
  const DwRange kr = dw_range(p, split, (int)gridDim.z);
  const long long kb0 = kr.kb0;
  const int nkb = kr.nkb;
  const int V = p.g.V;
  const int nj = min(BN, p.J - j0);
  // h columns this CTA loads: all nj (single CTA) or its half of the pair's 256
  const int jb = PAIR ? j0 + 128 * (int)rank : j0;
  const int nbox = PAIR ? max(0, min(2, (p.J - jb + 63) / 64)) : (nj + 63) / 64;
  const int vtile = v0 >> 7;

  if (warp == 4 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&loaded[s], 1);
      tc::mbar_init(&full[s], PAIR ? 8 : 4);     // transform warps of both CTAs (pair: arrive remotely)
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(tfull, 1);
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmP);
    tc::tma_prefetch(&tmH);
  }
  if (warp == 4) {
    if (PAIR) tc::tmem_alloc2(tmem_slot, 256);
    else tc::tmem_alloc(tmem_slot, 256);
  }
  tc::fence_before_sync();
  __syncthreads();
  if (PAIR) tc::cluster_sync();        // barrier inits visible to the peer before any remote arrive
  tc::fence_after_sync();
  const uint32_t tbase = *tmem_slot;

  if (warp < 4) {
    // ---- producers: thread handles v chunk c (8 logits) of rows g8 + 8 i of each k-block
    const int c = threadIdx.x & 15;          // 8-v chunk 0..15
    const int g8 = threadIdx.x >> 4;         // row group 0..7
    float dsum[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const bool want_db = blockIdx.y == 0;
    const uint32_t full0 = PAIR ? tc::mapa(&full[0], 0) : 0;   // the leader's full[0] (cluster address)
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      const long long rb = dw_row0(p, kb0 + kb);
      const int grows = dw_rows(p, rb);
      tc::mbar_wait(&loaded[stage], ph);
      uint8_t* sa = smem + stage * STAGE_BYTES;
      const float4* gq = reinterpret_cast<const float4*>(sa + A_BYTES + B_BYTES);
      uint4 pv[8];
      float4 sr[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {     // all shared-memory loads of the 8 rows first
        const int rl = g8 + 8 * i;
        sr[i] = rl < grows ? gq[rl] : make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
        pv[i] = *reinterpret_cast<const uint4*>(sa + (c >> 3) * (64 * BK * 2) + sw128(rl, c & 7));
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rl = g8 + 8 * i;
        const int info = __float_as_int(sr[i].w);
        *reinterpret_cast<uint4*>(sa + (c >> 3) * (64 * BK * 2) + sw128(rl, c & 7)) =
            info >= 0 ? dz_chunk(pv[i], sr[i].x, sr[i].y, sr[i].z, info, v0 + c * 8, want_db ? dsum : nullptr, rare)
                      : make_uint4(0, 0, 0, 0);
      }
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) tc::mbar_arrive_cluster(full0 + stage * 8);
        else tc::mbar_arrive(&full[stage]);
      }
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
    if (want_db) {
      // reduce the 8 row groups of each chunk deterministically through smem
#pragma unroll
      for (int j = 0; j < 8; ++j) dbs[g8 * 128 + c * 8 + j] = dsum[j];
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const int v = threadIdx.x;   // 0..127
      float s = 0.f;
#pragma unroll
      for (int gg = 0; gg < 8; ++gg) s += dbs[gg * 128 + v];
      if (v0 + v < V) p.dbp[(size_t)split * V + v0 + v] = s;
    }
    // ---- epilogue: partial dW tile -> dWp[split]
    if (nkb > 0) {
      tc::mbar_wait(tfull, 0);
      tc::fence_after_sync();
    }
    const int v = v0 + threadIdx.x;
    const uint32_t tl = tbase + ((uint32_t)(32 * warp) << 16);
    for (int c0 = 0; c0 < nj; c0 += 32) {
      float acc[32];
      if (nkb > 0) {
        tc::tmem_ld32(tl + c0, acc);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = 0.f;
      }
      if (v < V) {
        float4* o = reinterpret_cast<float4*>(p.dWp + ((size_t)split * V + v) * p.J + j0 + c0);
        const int n4 = min(8, (nj - c0) / 4);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < n4) o[q] = make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
      }
    }
  } else if (lane == 0 && nkb > 0) {
    // ---- warp 4 lane 0: TMA for A = P~[rows, v0..v0+127] (2 boxes), B = h[rows, jb..] and the scalars
    constexpr int PF = 6;                // P~ and h boxes prefetched into L2 this many k-blocks ahead
    const bool t3 = !PAIR && p.h3;       // 3-D maps: one TMA for the 2 P~ boxes, one for the 4 h boxes
    auto prefetch = [&](int kb) {
      const int rb = (int)dw_row0(p, kb0 + kb);
      if (t3) {
        tc::tma_prefetch_3d(&tmP, 0, rb, v0 / 64);
        tc::tma_prefetch_3d(&tmH, 0, rb, jb / 64);
        return;
      }
      tc::tma_prefetch_2d(&tmP, v0, rb);
      tc::tma_prefetch_2d(&tmP, v0 + 64, rb);
      for (int bx = 0; bx < nbox; ++bx) tc::tma_prefetch_2d(&tmH, jb + bx * 64, rb);
    };
    for (int kb = 0; kb < min(PF, nkb); ++kb) prefetch(kb);
    for (int kb = 0; kb < nkb; ++kb) {
      if (kb + PF < nkb) prefetch(kb + PF);
      const long long rb = dw_row0(p, kb0 + kb);
      const uint32_t gbytes = (uint32_t)dw_rows(p, rb) * 16u;
      const uint32_t bytes = A_BYTES + (t3 ? (uint32_t)B_BYTES : (uint32_t)nbox * 64 * BK * 2) + gbytes;
      tc::mbar_wait(&empty[stage_of(kb)], phase_of(kb) ^ 1);
      uint8_t* sa = smem + stage_of(kb) * STAGE_BYTES;
      uint64_t* ld = &loaded[stage_of(kb)];
      tc::mbar_arrive_expect_tx(ld, bytes);
      if (t3) {
        tc::tma_load_3d(sa, &tmP, ld, 0, (int)rb, v0 / 64);
        tc::tma_load_3d(sa + A_BYTES, &tmH, ld, 0, (int)rb, jb / 64);
      } else {
        tc::tma_load_2d(sa, &tmP, ld, v0, (int)rb);
        tc::tma_load_2d(sa + 64 * BK * 2, &tmP, ld, v0 + 64, (int)rb);
        for (int bx = 0; bx < nbox; ++bx)
          tc::tma_load_2d(sa + A_BYTES + bx * (64 * BK * 2), &tmH, ld, jb + bx * 64, (int)rb);
      }
      if (gbytes) tc::bulk_load(sa + A_BYTES + B_BYTES, p.g.gpk + (size_t)vtile * p.g.R + rb, gbytes, ld);
    }
  } else if (lane == 1 && nkb > 0 && rank == 0) {
    // ---- warp 4 lane 1 (pair: of the rank-0 CTA only): MMA issuer
    constexpr uint32_t idesc = tc::idesc_bf16(PAIR ? 2 * BM : BM, BN, true, true);
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      if (PAIR) tc::mbar_wait_cluster(&full[stage], ph);
      else tc::mbar_wait(&full[stage], ph);
      tc::fence_after_sync();
      const uint32_t a = tc::smem_u32(smem + stage * STAGE_BYTES), b = a + A_BYTES;
#pragma unroll
      for (int k = 0; k < BK / 16; ++k) {
        const uint64_t da = tc::sdesc(a + 2048 * k, 64 * BK * 2, 1024), db = tc::sdesc(b + 2048 * k, 64 * BK * 2, 1024);
        if (PAIR) tc::mma2_bf16(tbase, da, db, idesc, (kb | k) != 0);
        else tc::mma_bf16(tbase, da, db, idesc, (kb | k) != 0);
      }
      if (PAIR) tc::mma2_commit(&empty[stage], 3);
      else tc::mma_commit(&empty[stage]);
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
    if (PAIR) tc::mma2_commit(tfull, 3);
    else tc::mma_commit(tfull);
  }
  tc::fence_before_sync();
  __syncthreads();
  if (PAIR) tc::cluster_sync();        // the peer's smem / TMEM stay alive until the pair is done
  if (warp == 4) {
    if (PAIR) tc::tmem_dealloc2(tbase, 256);
    else tc::tmem_dealloc(tbase, 256);
  }
}

// K11, wide variant (large V): one CTA per SM computes a 256 (v) x 256 (j) partial dW tile as two
// 128 x 256 accumulators (TMEM columns 0..255 and 256..511) that share every h k-block, so the L2 -> SM
// bytes per MMA flop drop from 49 KB to 33 KB per 128x256x64 step (the h operand is read once per
// V-tile PAIR instead of per V tile).  Warps 0-7 transform dz (warps 0-3 tile 0, 4-7 tile 1) and run
// the epilogue; warp 8 lane 0 issues TMA, lane 1 the MMAs.
namespace jdw2 {
constexpr int BM = 128, BN = 256, BK = 64, STAGES = 3;
constexpr int A_BYTES = BM * BK * 2;                     // per V tile (2 boxes of 64 v x 64 rows)
constexpr int B_BYTES = BN * BK * 2;                     // 4 boxes of 64 j x 64 rows of h
constexpr int G_BYTES = BK * 16;
constexpr int STAGE_BYTES = 2 * A_BYTES + B_BYTES + 2 * G_BYTES;   // 66 KB
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256 + 8 * 256 * 4;
constexpr int THREADS = 288;
}  // namespace jdw2

// Plain mode (tscale == 0, one P~ offset per row, picks folded into P~ by pruned_combine, D20): dz =
// sc_r P~' with a row scalar, so d_w = P~'^T Hs with Hs = bf16(sc_r h_r) and A = P~' goes to the tensor
// cores untouched.  Hs comes either
//   precomputed (tmHs, scale_rows_kernel; large V): the MMA consumes the TMA'd stage directly and the
//     j-tile-0 CTAs' warps 0-7 read it alongside for the d_b sums (the stage is refilled once the MMAs and
//     those 8 warps are done with it), or
//   scaled in shared memory (small V, p.hsmem): warps 0-7 scale the h k-block in place (each 128-B line
//     of a box is one row) before the MMA reads it -- no Hs round trip through HBM, but 64 KB of extra smem
//     traffic per k-block, which costs more than the round trip once the mainloop is long (c3: 290 vs 238 +
//     15 us, c4: 2545 vs 1940 + 75 us; c5: 58 vs 53 + 37 us).
__global__ void __launch_bounds__(jdw2::THREADS, 1)
    joiner_dw_wide_kernel(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmH,
                          const __grid_constant__ CUtensorMap tmHs, const __grid_constant__ CUtensorMap tmP1,
                          const __grid_constant__ CUtensorMap tmO, JoinerDwParams p) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  using namespace jdw2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = tc::align1024(smem_raw);
  uint64_t* loaded = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* full = loaded + STAGES;
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  float* dbs = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256);     // [8 row groups][256 v]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool rare = p.g.V >= 6144;     // dz_chunk label pick by branch (measured: c4 -6 %, c3 (Zipf labels) +5 %)
  const bool jfirst = p.pfmode & 2;      // grid x = j tile (siblings sharing P~ adjacent)
  const int bvx = jfirst ? blockIdx.y : blockIdx.x, bjy = jfirst ? blockIdx.x : blockIdx.y;
  const int v0 = bvx * 2 * BM, j0 = bjy * BN, split = blockIdx.z;
  const DwRange kr = dw_range(p, split, (int)gridDim.z);
  const long long kb0 = kr.kb0;
  const int nkb = kr.nkb;
  const int V = p.g.V;
  const bool two = v0 + BM < V;          // the second V tile exists
  const int nj = min(BN, p.J - j0);
  const int nbox = (nj + 63) / 64;
  const int vtile = v0 >> 7;
  const bool plain = p.tscale && *p.tscale == 0;
  if (plain && p.pair_plain) return;      // the pair kernel (launched alongside) does the plain mode
  const bool hsm = plain && p.hsmem;      // Hs formed in shared memory
  const bool dbread = plain && !hsm && bjy == 0;   // precomputed Hs: the d_b readers release the stage too
  // P~ multicast (p.mc = the cluster size along x = the J parts of one (V pair, split)): each sibling
  // loads planes rank, rank + mc, .. of the 4-plane P~ k-block into every sibling's stage, so the P~
  // bytes cross L2 -> SM once per cluster instead of once per J part; a stage is refilled once every
  // sibling's MMA released it (commits multicast to all siblings' empty barriers).  With d_b readers
  // (dbread) the rank-0 CTA gates its MMA on them (full) instead of adding them to the release count.
  const int mc = p.mc > 1 ? p.mc : 0;
  const uint32_t crank = mc ? tc::cluster_ctarank() : 0u;
  const uint16_t mcmask = (uint16_t)((1u << mc) - 1u);
  const bool dbfull = dbread && mc;

  if (warp == 8 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&loaded[s], 1);
      tc::mbar_init(&full[s], 8);
      tc::mbar_init(&empty[s], mc ? mc : (dbread ? 9 : 1));
    }
    tc::mbar_init(tfull, 1);
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmP);
    tc::tma_prefetch(plain && !hsm ? &tmHs : &tmH);
  }
  if (warp == 8) tc::tmem_alloc(tmem_slot, 512);
  tc::fence_before_sync();
  __syncthreads();
  if (mc) tc::cluster_sync();             // every sibling's barriers are initialised before any multicast
  tc::fence_after_sync();
  const uint32_t tbase = *tmem_slot;

  if (warp < 8) {
    const int a = warp >> 2;                 // V tile 0 / 1 of the pair
    const int t = threadIdx.x & 127;
    const int c = t & 15;                    // 8-v chunk 0..15
    const int g8 = t >> 4;                   // row group 0..7
    const bool mine = a == 0 || two;
    float dsum[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const bool want_db = bjy == 0;
    const int va = v0 + a * BM;
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < (plain && !hsm && !want_db ? 0 : nkb); ++kb) {
      const long long rb = dw_row0(p, kb0 + kb);
      const int grows = dw_rows(p, rb);
      tc::mbar_wait(&loaded[stage], ph);
      if (plain) {
        if (want_db && mine) {   // d_b only: sum sc_r P~'[r, v] over the k-block's rows (no smem writes)
          const uint8_t* sa = smem + stage * STAGE_BYTES + a * A_BYTES;
          const float4* gq = reinterpret_cast<const float4*>(smem + stage * STAGE_BYTES + 2 * A_BYTES + B_BYTES + a * G_BYTES);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rl = g8 + 8 * i;
            const float sc = rl < grows ? gq[rl].x : 0.f;
            const uint4 pv = *reinterpret_cast<const uint4*>(sa + (c >> 3) * (64 * BK * 2) + sw128(rl, c & 7));
            const uint32_t w[4] = {pv.x, pv.y, pv.z, pv.w};
            if (sc != 0.f) {
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                dsum[2 * k] += sc * __uint_as_float(w[k] << 16);
                dsum[2 * k + 1] += sc * __uint_as_float(w[k] & 0xffff0000u);
              }
            }
          }
        }
        if (!hsm) {
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(dbfull ? &full[stage] : &empty[stage]);   // done reading the stage
          if (++stage == STAGES) { stage = 0; ph ^= 1; }
          continue;
        }
        // Hs = bf16(sc_r h_r) in place: 16-B chunk i of the B region lies in 128-B line i / 8, row (i / 8) % 64
        uint8_t* sb = smem + stage * STAGE_BYTES + 2 * A_BYTES;
        const float4* g0 = reinterpret_cast<const float4*>(smem + stage * STAGE_BYTES + 2 * A_BYTES + B_BYTES);
        constexpr int NCH = B_BYTES / 16 / 256;   // chunks per thread
        uint4 hv[NCH];
        float sc[NCH];
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
          const int ch = threadIdx.x + 256 * i;
          const int rl = (ch >> 3) & (BK - 1);
          sc[i] = rl < grows ? g0[rl].x : 0.f;
          hv[i] = *reinterpret_cast<const uint4*>(sb + ch * 16);
        }
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
          const uint32_t w[4] = {hv[i].x, hv[i].y, hv[i].z, hv[i].w};
          uint32_t q[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const __nv_bfloat162 h2 = __floats2bfloat162_rn(sc[i] * __uint_as_float(w[k] << 16),
                                                            sc[i] * __uint_as_float(w[k] & 0xffff0000u));
            q[k] = *reinterpret_cast<const uint32_t*>(&h2);
          }
          *reinterpret_cast<uint4*>(sb + (threadIdx.x + 256 * i) * 16) = make_uint4(q[0], q[1], q[2], q[3]);
        }
        tc::fence_proxy_async();
      } else if (mine) {
        uint8_t* sa = smem + stage * STAGE_BYTES + a * A_BYTES;
        const float4* gq = reinterpret_cast<const float4*>(smem + stage * STAGE_BYTES + 2 * A_BYTES + B_BYTES + a * G_BYTES);
        uint4 pv[8];
        float4 sr[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rl = g8 + 8 * i;
          sr[i] = rl < grows ? gq[rl] : make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
          pv[i] = *reinterpret_cast<const uint4*>(sa + (c >> 3) * (64 * BK * 2) + sw128(rl, c & 7));
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rl = g8 + 8 * i;
          const int info = __float_as_int(sr[i].w);
          *reinterpret_cast<uint4*>(sa + (c >> 3) * (64 * BK * 2) + sw128(rl, c & 7)) =
              info >= 0 ? dz_chunk(pv[i], sr[i].x, sr[i].y, sr[i].z, info, va + c * 8, want_db ? dsum : nullptr, rare)
                        : make_uint4(0, 0, 0, 0);
        }
        tc::fence_proxy_async();
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&full[stage]);
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
    if (want_db) {
#pragma unroll
      for (int j = 0; j < 8; ++j) dbs[g8 * 256 + a * 128 + c * 8 + j] = dsum[j];
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const int v = threadIdx.x;   // 0..255
      float s = 0.f;
#pragma unroll
      for (int gg = 0; gg < 8; ++gg) s += dbs[gg * 256 + v];
      if (v0 + v < V) p.dbp[(size_t)split * V + v0 + v] = s;
    }
    // ---- epilogue: accumulator a -> dWp[split] rows va .. va + 127: per 32-column chunk the group's 128
    // threads stage their rows in a swizzled 16 KB tile (two per group, in the now idle stage buffers) and
    // one thread TMA-stores it (rows past V / columns past J clipped by the map); the per-row float4 stores
    // this replaces were a quarter of the kernel's stall samples at c5 (32 scattered rows per instruction)
    if (nkb > 0) {
      tc::mbar_wait(tfull, 0);
      tc::fence_after_sync();
    }
    if (mine) {
      const uint32_t tl = tbase + (uint32_t)(a * 256) + ((uint32_t)(32 * (warp & 3)) << 16);
      const bool st_leader = (threadIdx.x & 127) == 0;
      int kc = 0;
      for (int c0 = 0; c0 < nj; c0 += 32, ++kc) {
        float acc[32];
        if (nkb > 0) {
          tc::tmem_ld32(tl + c0, acc);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[i] = 0.f;
        }
        uint8_t* ob = smem + (a * 2 + (kc & 1)) * (BM * 32 * 4);
        if (st_leader && kc >= 2) tc::bulk_wait_read1();   // the store issued from this tile 2 chunks ago
        asm volatile("bar.sync %0, 128;" ::"r"(2 + a) : "memory");
        float4* O4 = reinterpret_cast<float4*>(ob);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          O4[t * 8 + (q ^ (t & 7))] = make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
        tc::fence_proxy_async();
        asm volatile("bar.sync %0, 128;" ::"r"(2 + a) : "memory");
        if (st_leader) {
          tc::tma_store_3d(&tmO, ob, j0 + c0, va, split);
          tc::bulk_commit();
        }
      }
      if (st_leader) tc::bulk_wait0();
    }
  } else if (lane == 0 && nkb > 0) {
    // ---- warp 8 lane 0: TMA for both P~ tiles, the h (precomputed plain: Hs) k-block and the two tiles'
    // row scalars
    const CUtensorMap* tB = plain && !hsm ? &tmHs : &tmH;
    const bool gq_needed = !plain || hsm || bjy == 0;   // plain: the scalars scale h / feed the d_b sums
    const int PF = p.pf;
    const bool pfP = !(p.pfmode & 1) || bjy == 0, pfH = !(p.pfmode & 1) || bvx == 0;
    auto prefetch = [&](int kb) {
      const int rb = (int)dw_row0(p, kb0 + kb);
      if (pfP) tc::tma_prefetch_3d(&tmP, 0, rb, v0 / 64);
      if (pfH) {
        if (p.h3) tc::tma_prefetch_3d(tB, 0, rb, j0 / 64);
        else
          for (int bx = 0; bx < nbox; ++bx) tc::tma_prefetch_2d(tB, j0 + bx * 64, rb);
      }
    };
    for (int kb = 0; kb < min(PF, nkb); ++kb) prefetch(kb);
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      if (kb + PF < nkb) prefetch(kb + PF);
      const long long rb = dw_row0(p, kb0 + kb);
      const uint32_t gbytes = gq_needed ? (uint32_t)dw_rows(p, rb) * 16u : 0u;
      // 3-D boxes: out-of-range planes (the missing second V tile, j past J) arrive zero-filled and
      // count in full toward the transaction bytes
      const uint32_t bytes = 2 * A_BYTES + (two ? 2 : 1) * gbytes + (p.h3 ? B_BYTES : (uint32_t)nbox * 64 * BK * 2);
      tc::mbar_wait(&empty[stage], ph ^ 1);
      uint8_t* sa = smem + stage * STAGE_BYTES;
      uint64_t* ld = &loaded[stage];
      tc::mbar_arrive_expect_tx(ld, bytes);
      if (mc) {
        for (int pl = (int)crank; pl < 4; pl += mc)
          tc::tma_load_3d_mc(sa + pl * (64 * BK * 2), &tmP1, ld, 0, (int)rb, v0 / 64 + pl, mcmask);
      } else {
        tc::tma_load_3d(sa, &tmP, ld, 0, (int)rb, v0 / 64);
      }
      if (p.h3) tc::tma_load_3d(sa + 2 * A_BYTES, tB, ld, 0, (int)rb, j0 / 64);
      else
        for (int bx = 0; bx < nbox; ++bx)
          tc::tma_load_2d(sa + 2 * A_BYTES + bx * (64 * BK * 2), tB, ld, j0 + bx * 64, (int)rb);
      // (plain mode: tile 0's scalars are every tile's, and the only ones pruned_combine writes)
      const size_t gt0 = plain ? 0 : (size_t)vtile, gt1 = plain ? 0 : (size_t)(vtile + 1);
      if (gbytes) tc::bulk_load(sa + 2 * A_BYTES + B_BYTES, p.g.gpk + gt0 * p.g.R + rb, gbytes, ld);
      if (two && gbytes) tc::bulk_load(sa + 2 * A_BYTES + B_BYTES + G_BYTES, p.g.gpk + gt1 * p.g.R + rb, gbytes, ld);
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
  } else if (lane == 1 && nkb > 0) {
    // ---- warp 8 lane 1: two 128x256x16 MMAs per k-step, one per V tile, sharing the h descriptor
    constexpr uint32_t idesc = tc::idesc_bf16(BM, BN, true, true);
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      tc::mbar_wait(plain && !hsm && !dbfull ? &loaded[stage] : &full[stage], ph);
      tc::fence_after_sync();
      const uint32_t a = tc::smem_u32(smem + stage * STAGE_BYTES), b = a + 2 * A_BYTES;
#pragma unroll
      for (int k = 0; k < BK / 16; ++k) {
        const uint64_t db = tc::sdesc(b + 2048 * k, 64 * BK * 2, 1024);
        tc::mma_bf16(tbase, tc::sdesc(a + 2048 * k, 64 * BK * 2, 1024), db, idesc, (kb | k) != 0);
        if (two) tc::mma_bf16(tbase + 256, tc::sdesc(a + A_BYTES + 2048 * k, 64 * BK * 2, 1024), db, idesc, (kb | k) != 0);
      }
      if (mc) tc::mma_commit_mc(&empty[stage], mcmask);   // releases the stage in every sibling
      else tc::mma_commit(&empty[stage]);
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
    tc::mma_commit(tfull);
  }
  tc::fence_before_sync();
  __syncthreads();
  if (mc) tc::cluster_sync();             // no multicast write or arrive targets an exited sibling
  if (warp == 8) tc::tmem_dealloc(tbase, 512);
}

// K11, CTA-pair variant for the plain mode with a precomputed Hs (large V, D20): a pair (cta_group::2,
// cluster of 2) computes a 512 (v) x 256 (j) partial dW tile as two 256 x 256 accumulators, CTA r holding
// the TMEM lanes of V tiles v0 + 128 r and v0 + 256 + 128 r (512 TMEM columns: both accumulators); each
// k-block (64 rows) every CTA loads its two 128-v P~ tiles and HALF of the 256 Hs columns, so the L2 -> SM
// bytes per MMA flop drop from 64 KB to 48 KB per 2 x 128x256x64 (the wide kernel, the L2 throughput cap
// at V = 8000: 0.56 of the bf16 burst peak).  The MMA consumes the TMA'd stages directly (no producer
// transforms, so the pair needs no per-stage handshake beyond the TMA bytes landing on the leader's
// barrier).  d_b (J part 0 only): each CTA's warps sum sc_r P~'[r,v] of their tiles; there the P~ tiles are
// loaded per CTA (local barrier) and a relay thread forwards their arrival to the leader's barrier.
namespace jdwp {
constexpr int BM = 128, BNH = 128, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;                   // one V tile: 2 planes of 64 v x 64 rows
constexpr int B_BYTES = BNH * BK * 2;                  // this CTA's half of the 256 Hs columns: 2 planes
constexpr int G_BYTES = 1024;                          // the k-block's row scalars (64 x 16 B)
constexpr int STAGE_BYTES = 2 * A_BYTES + B_BYTES + G_BYTES;   // 49 KB (1024-aligned)
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256 + 8 * 256 * 4;
constexpr int THREADS = 288;
}  // namespace jdwp

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(jdwp::THREADS, 1)
    joiner_dw_pair_kernel(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmHs,
                          const __grid_constant__ CUtensorMap tmO, JoinerDwParams p) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  using namespace jdwp;
  if (*p.tscale != 0) return;             // the rescaling mode: the wide kernel (launched alongside) does it
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = tc::align1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);   // leader: MMA may start
  uint64_t* empty = full + STAGES;        // this CTA's stage may be refilled
  uint64_t* aload = empty + STAGES;       // d_b pairs: this CTA's P~ tiles + scalars landed (local)
  uint64_t* tfull = aload + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  float* dbs = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256);     // [8 row groups][256 v]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_ctarank();
  const bool leader = rank == 0;
  const int quad = blockIdx.x >> 1, bjy = blockIdx.y, split = blockIdx.z;
  const int v0 = quad * 4 * BM;
  const int va0 = v0 + (int)rank * BM, va1 = v0 + 2 * BM + (int)rank * BM;   // this CTA's two V tiles
  const int j0 = bjy * 2 * BNH, jh = j0 + (int)rank * BNH;                  // the pair's j part, this half
  const DwRange kr = dw_range(p, split, (int)gridDim.z);
  const long long kb0 = kr.kb0;
  const int nkb = kr.nkb;
  const int V = p.g.V;
  const bool two = v0 + 2 * BM < V;       // the second accumulator's tiles exist (pair-uniform)
  const int nj = min(2 * BNH, p.J - j0);
  const bool dbp = bjy == 0;              // d_b pair: local P~ loads + relay
  if (warp == 8 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], dbp ? 3 : 1);      // d_b pairs: the leader's expect-tx + both CTAs' relays
      tc::mbar_init(&empty[s], dbp ? 9 : 1);     // the leader's MMA commit (+ the 8 d_b warps)
      tc::mbar_init(&aload[s], 1);
    }
    tc::mbar_init(tfull, 1);
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmP);
    tc::tma_prefetch(&tmHs);
  }
  if (warp == 8) tc::tmem_alloc2(tmem_slot, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::cluster_sync();                     // the peer's barriers are initialised before any remote signal
  tc::fence_after_sync();
  const uint32_t tbase = *tmem_slot;
  const uint32_t fullL = tc::mapa(&full[0], 0);

  if (warp < 8) {
    const int a = warp >> 2;                 // accumulator / V tile 0 / 1 of this CTA
    const int t = threadIdx.x & 127;
    const int c = t & 15;                    // 8-v chunk 0..15
    const int g8 = t >> 4;                   // row group 0..7
    const bool mine = a == 0 || two;
    const int va = a == 0 ? va0 : va1;
    if (dbp) {
      float dsum[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      int stage = 0;
      uint32_t ph = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        const long long rb = dw_row0(p, kb0 + kb);
        const int grows = dw_rows(p, rb);
        tc::mbar_wait(&aload[stage], ph);
        if (mine) {   // d_b: sum sc_r P~'[r, v] over the k-block's rows (no smem writes)
          const uint8_t* sa = smem + stage * STAGE_BYTES + a * A_BYTES;
          const float4* gq = reinterpret_cast<const float4*>(smem + stage * STAGE_BYTES + 2 * A_BYTES + B_BYTES);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rl = g8 + 8 * i;
            const float sc = rl < grows ? gq[rl].x : 0.f;
            const uint4 pv = *reinterpret_cast<const uint4*>(sa + (c >> 3) * (64 * BK * 2) + sw128(rl, c & 7));
            const uint32_t w[4] = {pv.x, pv.y, pv.z, pv.w};
            if (sc != 0.f) {
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                dsum[2 * k] += sc * __uint_as_float(w[k] << 16);
                dsum[2 * k + 1] += sc * __uint_as_float(w[k] & 0xffff0000u);
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&empty[stage]);   // this warp is done reading the stage
        if (++stage == STAGES) { stage = 0; ph ^= 1; }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) dbs[g8 * 256 + a * 128 + c * 8 + j] = dsum[j];
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const int tv = threadIdx.x;   // 0..255: tile tv / 128, row tv % 128
      float sacc = 0.f;
#pragma unroll
      for (int gg = 0; gg < 8; ++gg) sacc += dbs[gg * 256 + tv];
      const int vv = (tv < 128 ? va0 : va1) + (tv & 127);
      if (vv < V && (tv < 128 || two)) p.dbp[(size_t)split * V + vv] = sacc;
    }
    // ---- epilogue: this CTA's accumulator lanes -> dWp[split] rows va.., one TMA store per 32 columns
    if (nkb > 0) {
      tc::mbar_wait(tfull, 0);
      tc::fence_after_sync();
    }
    if (mine) {
      const uint32_t tl = tbase + (uint32_t)(a * 256) + ((uint32_t)(32 * (warp & 3)) << 16);
      const bool st_leader = (threadIdx.x & 127) == 0;
      int kc = 0;
      for (int c0 = 0; c0 < nj; c0 += 32, ++kc) {
        float acc[32];
        if (nkb > 0) {
          tc::tmem_ld32(tl + c0, acc);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) acc[i] = 0.f;
        }
        uint8_t* ob = smem + (a * 2 + (kc & 1)) * (BM * 32 * 4);
        if (st_leader && kc >= 2) tc::bulk_wait_read1();
        asm volatile("bar.sync %0, 128;" ::"r"(2 + a) : "memory");
        float4* O4 = reinterpret_cast<float4*>(ob);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          O4[t * 8 + (q ^ (t & 7))] = make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
        tc::fence_proxy_async();
        asm volatile("bar.sync %0, 128;" ::"r"(2 + a) : "memory");
        if (st_leader) {
          tc::tma_store_3d(&tmO, ob, j0 + c0, va, split);
          tc::bulk_commit();
        }
      }
      if (st_leader) tc::bulk_wait0();
    }
  } else if (lane == 0 && nkb > 0) {
    // ---- warp 8 lane 0: TMA (P~ tiles: 2sm, or local for d_b pairs; the Hs half: 2sm; scalars: local)
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      const long long rb = dw_row0(p, kb0 + kb);
      const uint32_t gbytes = dbp ? (uint32_t)dw_rows(p, rb) * 16u : 0u;
      tc::mbar_wait(&empty[stage], ph ^ 1);
      uint8_t* sa = smem + stage * STAGE_BYTES;
      const uint32_t fb = fullL + stage * 8;
      if (dbp) {
        if (leader) tc::mbar_arrive_expect_tx(&full[stage], 2u * B_BYTES);
        tc::mbar_arrive_expect_tx(&aload[stage], (two ? 2u : 1u) * A_BYTES + gbytes);
        tc::tma_load_3d(sa, &tmP, &aload[stage], 0, (int)rb, va0 / 64);
        if (two) tc::tma_load_3d(sa + A_BYTES, &tmP, &aload[stage], 0, (int)rb, va1 / 64);
        if (gbytes) tc::bulk_load(sa + 2 * A_BYTES + B_BYTES, p.g.gpk + rb, gbytes, &aload[stage]);
      } else {
        if (leader) tc::mbar_arrive_expect_tx(&full[stage], 2u * ((two ? 2u : 1u) * A_BYTES + B_BYTES));
        tc::tma_load_3d_2sm(sa, &tmP, fb, 0, (int)rb, va0 / 64);
        if (two) tc::tma_load_3d_2sm(sa + A_BYTES, &tmP, fb, 0, (int)rb, va1 / 64);
      }
      tc::tma_load_3d_2sm(sa + 2 * A_BYTES, &tmHs, fb, 0, (int)rb, jh / 64);
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
  } else if (lane == 1 && nkb > 0 && dbp) {
    // ---- warp 8 lane 1 (d_b pairs): relay "this CTA's P~ tiles landed" to the leader's full barrier
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      tc::mbar_wait(&aload[stage], ph);
      tc::mbar_arrive_cluster(fullL + stage * 8);
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
  } else if (lane == 2 && nkb > 0 && leader) {
    // ---- warp 8 lane 2 of the leader: the pair's MMAs, two 256x256x16 per k-step sharing the Hs descriptor
    constexpr uint32_t idesc = tc::idesc_bf16(2 * BM, 2 * BNH, true, true);
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      tc::mbar_wait_cluster(&full[stage], ph);
      tc::fence_after_sync();
      const uint32_t a = tc::smem_u32(smem + stage * STAGE_BYTES), b = a + 2 * A_BYTES;
#pragma unroll
      for (int k = 0; k < BK / 16; ++k) {
        const uint64_t db = tc::sdesc(b + 2048 * k, 64 * BK * 2, 1024);
        tc::mma2_bf16(tbase, tc::sdesc(a + 2048 * k, 64 * BK * 2, 1024), db, idesc, (kb | k) != 0);
        if (two) tc::mma2_bf16(tbase + 256, tc::sdesc(a + A_BYTES + 2048 * k, 64 * BK * 2, 1024), db, idesc, (kb | k) != 0);
      }
      tc::mma2_commit(&empty[stage], 3);   // releases the stage in both CTAs
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
    tc::mma2_commit(tfull, 3);
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::cluster_sync();                     // the peer's smem / TMEM stay alive until the pair is done
  if (warp == 8) tc::tmem_dealloc2(tbase, 512);
}

// ======================================================================= host
template <int NTW, bool MC, bool D16>
static cudaError_t launch_dh_k(const JoinerDhParams& p, unsigned grid, const CUtensorMap& tp, const CUtensorMap& tw,
                               const CUtensorMap& th, const CUtensorMap& td, cudaStream_t st) {
  constexpr int SMEM = jdh::Cfg<NTW, D16>::SMEM_BYTES;
  smem_optin(joiner_dh_tc_kernel<NTW, MC, D16>, SMEM);
  if (!MC) {
    launch_pdl(joiner_dh_tc_kernel<NTW, MC, D16>, grid, jdh::Roles<NTW>::THREADS, SMEM, st, tp, tw, th, td, p);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(jdh::Roles<NTW>::THREADS);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, joiner_dh_tc_kernel<NTW, MC, D16>, tp, tw, th, td, p);
}
// 4 producer warps for short V loops, 8 for long ones; W multicast over CTA pairs (RNNT_DH_MC=0: off)
static cudaError_t launch_dh(const JoinerDhParams& p, unsigned grid, bool mc, const CUtensorMap& tp,
                             const CUtensorMap& tw, const CUtensorMap& th, const CUtensorMap& td, cudaStream_t st) {
  const bool d16 = p.gsp != nullptr, lv = p.nkb >= 32;
#define RNNT_DH(NTWV, MCV) (d16 ? launch_dh_k<NTWV, MCV, true>(p, grid, tp, tw, th, td, st) \
                                : launch_dh_k<NTWV, MCV, false>(p, grid, tp, tw, th, td, st))
  if (mc) return lv ? RNNT_DH(8, true) : RNNT_DH(4, true);
  return lv ? RNNT_DH(8, false) : RNNT_DH(4, false);
#undef RNNT_DH
}

// dpre = dh (1 - h^2) rows of the live 128-row tiles (`live`, count at `nlive`, at most ntiles) into dpre.
cudaError_t joiner_dh_launch(const Dims& d, const GradSrc& g, const uint16_t* h, const uint16_t* W, const int* live,
                             const int* nlive, long long ntiles, float* dpre, const int* tscale, const float* gsp,
                             cudaStream_t st) {
  CUtensorMap tp, tw, th;
  if (!make_tmap_bf16_2d(&tp, g.Pt, d.VP(), d.rows(), (uint64_t)d.VP() * 2, jdh::BK, jdh::BM)) return cudaErrorInvalidValue;
  static const int mc_env = env_int("RNNT_DH_MC", 1);
  const bool mc = mc_env != 0 && ntiles >= 2;
  const bool w3 = d.J % 64 == 0;
  // W as 3-D (64 j, V, J/64) boxes of 4 planes (one TMA per k-block), or 2 planes per CTA with multicast
  if (w3 ? !make_tmap_bf16_3d(&tw, W, 64, d.V, d.J / 64, (uint64_t)d.J * 2, 128, 64, 64, mc ? 2 : 4)
         : !make_tmap_bf16_2d(&tw, W, d.J, d.V, (uint64_t)d.J * 2, 64, 64))
    return cudaErrorInvalidValue;
  if (!make_tmap_bf16_2d(&th, h, d.J, d.rows(), (uint64_t)d.J * 2, 64, jdh::BM)) return cudaErrorInvalidValue;
  CUtensorMap td;   // dpre (R, J) fp32, box 32 columns x 128 rows
  if (gsp ? !make_tmap_f16_3d(&td, dpre, d.J, d.rows(), 1, (uint64_t)d.J * 2, (uint64_t)d.rows() * d.J * 2, 32, jdh::BM)
          : !make_tmap_f32_3d(&td, dpre, d.J, d.rows(), 1, (uint64_t)d.J * 4, (uint64_t)d.rows() * d.J * 4, 32, jdh::BM))
    return cudaErrorInvalidValue;
  const int njp = (d.J + jdh::NSUB - 1) / jdh::NSUB;
  JoinerDhParams p{g, h, d.J, (d.V + jdh::BK - 1) / jdh::BK, njp, live, nlive, dpre, w3 ? 1 : 0, tscale, gsp};
  const int nsm = current_sm_count();
  unsigned grid = (unsigned)std::min<long long>(ntiles * njp, nsm);
  if (mc) grid = (unsigned)std::min<long long>((ntiles + 1) / 2 * njp, nsm / 2) * 2;
  if (grid == 0) return cudaSuccess;
  RNNT_LAUNCH(KID_DH, st, launch_dh(p, grid, mc, tp, tw, th, td, st));
  return cudaGetLastError();
}

// live / nlive: the ascending live-tile list of the step (null: every row's k-block is read);
// Hs = bf16(sc_r h_r) for the rows of the live tiles (plain mode with a precomputed Hs: tscale == 0; dead
// rows 0), the B operand of the plain d_w GEMM.  Block per live tile (grid-stride), four 16-B loads in
// flight per thread.
__global__ void __launch_bounds__(256) scale_rows_kernel(const uint16_t* __restrict__ h, const float4* __restrict__ gpk,
                                                         const int* __restrict__ tscale, const int* __restrict__ live,
                                                         const int* __restrict__ nlive, long long R, int J,
                                                         uint16_t* __restrict__ Hs) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  if (*tscale != 0) return;
  const int nl = *nlive, J8 = J / 8;
  constexpr int KU = 4;
  for (int b = blockIdx.x; b < nl; b += gridDim.x) {
    const long long r0 = (long long)live[b] * 128;
    const int rows = (int)min(128LL, R - r0);
    const int tot = rows * J8;
    for (int i0 = threadIdx.x; i0 < tot; i0 += KU * blockDim.x) {
      uint4 x[KU];
      float sc[KU];
#pragma unroll
      for (int k = 0; k < KU; ++k) {
        const int i = i0 + k * blockDim.x;
        const int rl = i / J8, c = i - rl * J8;
        const long long r = r0 + rl;
        sc[k] = i < tot ? gpk[r].x : 0.f;   // tile 0's scalar (= every tile's in plain mode); dead rows 0
        x[k] = sc[k] != 0.f ? __ldg(reinterpret_cast<const uint4*>(h + r * J) + c) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int k = 0; k < KU; ++k) {
        const int i = i0 + k * blockDim.x;
        if (i >= tot) break;
        const int rl = i / J8, c = i - rl * J8;
        const uint32_t w[4] = {x[k].x, x[k].y, x[k].z, x[k].w};
        uint32_t q[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const __nv_bfloat162 h2 = __floats2bfloat162_rn(sc[k] * __uint_as_float(w[m] << 16),
                                                          sc[k] * __uint_as_float(w[m] & 0xffff0000u));
          q[m] = *reinterpret_cast<const uint32_t*>(&h2);
        }
        reinterpret_cast<uint4*>(Hs + (r0 + rl) * J)[c] = make_uint4(q[0], q[1], q[2], q[3]);
      }
    }
  }
}
cudaError_t scale_rows_launch(const Dims& d, const GradSrc& g, const uint16_t* h, const int* tscale, const int* live,
                              const int* nlive, long long ntiles, uint16_t* Hs, cudaStream_t st) {
  const unsigned grid = (unsigned)std::min<long long>(ntiles, 8LL * current_sm_count());
  if (grid == 0) return cudaSuccess;
  RNNT_LAUNCH(KID_SCALE_ROWS, st, launch_pdl(scale_rows_kernel, grid, 256, 0, st, h, g.gpk, tscale, live, nlive, g.R, d.J, Hs));
  return cudaGetLastError();
}

// tscale: the plain mode's switch (null: the rescaling path); Hs: the precomputed plain-mode B operand
// (null with tscale: formed in shared memory)
cudaError_t joiner_dw_launch(const Dims& d, const GradSrc& g, const uint16_t* h, const uint16_t* Hs, const int* tscale, const int* live, const int* nlive, float* dWp, float* dbp, int splits,
                             cudaStream_t st) {
  CUtensorMap tp, th;
  if (!make_tmap_bf16_2d(&tp, g.Pt, d.VP(), d.rows(), (uint64_t)d.VP() * 2, 64, jdw::BK)) return cudaErrorInvalidValue;
  if (!make_tmap_bf16_2d(&th, h, d.J, d.rows(), (uint64_t)d.J * 2, 64, 64)) return cudaErrorInvalidValue;
  const long long nkb = (d.rows() + jdw::BK - 1) / jdw::BK;
  const long long per = (nkb + splits - 1) / splits;
  JoinerDwParams p{g, d.J, per, nkb, live, nlive, dw_wide(d) ? tscale : nullptr, dWp, dbp};
  const int vt = (d.V + jdw::BM - 1) / jdw::BM;
  // CTA pairs (cta_group::2, V tiles rounded up to an even count) only when RNNT_DW_PAIR=1: parity-green
  // but measured slower (c2 87.6 vs 69.6 us, c4 4.42 vs 3.22 ms) -- the per-stage cross-CTA handshake
  // (remote arrive + cluster-scope acquire) costs more than the halved h traffic saves at 2-3 stages
  static const int pair = env_int("RNNT_DW_PAIR", 0) == 1;
  if (dw_wide(d)) {
    smem_optin(joiner_dw_wide_kernel, jdw2::SMEM_BYTES);
    CUtensorMap tp3, th3;
    if (!make_tmap_bf16_3d(&tp3, g.Pt, 64, d.rows(), d.VP() / 64, (uint64_t)d.VP() * 2, 128, 64, jdw2::BK, 4))
      return cudaErrorInvalidValue;
    p.h3 = d.J % 64 == 0;
    if (p.h3 && !make_tmap_bf16_3d(&th3, h, 64, d.rows(), d.J / 64, (uint64_t)d.J * 2, 128, 64, jdw2::BK, 4))
      return cudaErrorInvalidValue;
    CUtensorMap ths = p.h3 ? th3 : th;   // the precomputed plain-mode B operand Hs, same geometry as h
    if (Hs && (p.h3 ? !make_tmap_bf16_3d(&ths, Hs, 64, d.rows(), d.J / 64, (uint64_t)d.J * 2, 128, 64, jdw2::BK, 4)
                    : !make_tmap_bf16_2d(&ths, Hs, d.J, d.rows(), (uint64_t)d.J * 2, 64, 64)))
      return cudaErrorInvalidValue;
    p.hsmem = Hs ? 0 : 1;
    CUtensorMap to;   // the split partials dWp (splits, V, J) fp32, box 32 columns x 128 rows
    if (!make_tmap_f32_3d(&to, dWp, d.J, d.V, splits, (uint64_t)d.J * 4, (uint64_t)d.V * d.J * 4, 32, jdw2::BM))
      return cudaErrorInvalidValue;
    // P~ multicast over the J parts (RNNT_DW_MC=1: on): clusters of njp CTAs along grid x (j first)
    const int njp = (d.J + jdw2::BN - 1) / jdw2::BN;
    static const int mc_env = env_int("RNNT_DW_MC", 0);   // measured slower: off by default
    CUtensorMap tp1 = tp3;
    if (mc_env != 0 && njp >= 2 && njp <= 8) {
      if (!make_tmap_bf16_3d(&tp1, g.Pt, 64, d.rows(), d.VP() / 64, (uint64_t)d.VP() * 2, 128, 64, jdw2::BK, 1))
        return cudaErrorInvalidValue;
      p.mc = njp;
      p.pfmode |= 2;
    }
    static const int pf = env_int("RNNT_DW_PF", -1), pfmode = env_int("RNNT_DW_PFMODE", -1);
    if (pf >= 0) p.pf = pf;
    if (pfmode >= 0) p.pfmode = pfmode;
    if (p.mc > 1) p.pfmode |= 2;           // (clusters run along grid x: the J parts first)
    dim3 grid((unsigned)((vt + 1) / 2), (d.J + jdw2::BN - 1) / jdw2::BN, splits);
    // plain mode with a precomputed Hs: the CTA-pair kernel (RNNT_DW_PAIR2=0: off); the wide kernel then
    // only runs if the forward switched to per-tile rescaling (both decide on the device-side tscale)
    // measured: c4 (V = 8000, J = 768) 1.81 vs 1.93 ms in the step, c3 (V = 5000, J = 512) 274 vs 254 us
    // standalone, so by default only from V >= 6144 (RNNT_DW_PAIR2=1 / 0: always / never)
    static const int pair2 = env_int("RNNT_DW_PAIR2", -1);
    const bool use_pair = pair2 == 1 || (pair2 < 0 && d.V >= 6144);
    if (Hs && tscale && use_pair && p.mc <= 1 && d.J % 64 == 0) {   // (3-D Hs boxes)
      smem_optin(joiner_dw_pair_kernel, jdwp::SMEM_BYTES);
      CUtensorMap tpp, thp;
      if (!make_tmap_bf16_3d(&tpp, g.Pt, 64, d.rows(), d.VP() / 64, (uint64_t)d.VP() * 2, 128, 64, jdwp::BK, 2) ||
          !make_tmap_bf16_3d(&thp, Hs, 64, d.rows(), (d.J + 63) / 64, (uint64_t)d.J * 2, 128, 64, jdwp::BK, 2))
        return cudaErrorInvalidValue;
      p.pair_plain = 1;
      const unsigned quads = (unsigned)((vt + 3) / 4);
      dim3 pg(2 * quads, (d.J + 2 * jdwp::BNH - 1) / (2 * jdwp::BNH), splits);
      RNNT_LAUNCH(KID_DW, st, launch_pdl(joiner_dw_pair_kernel, pg, jdwp::THREADS, jdwp::SMEM_BYTES, st, tpp, thp, to, p));
    }
    if (p.pfmode & 2) std::swap(grid.x, grid.y);
    if (p.mc > 1) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = grid;
      cfg.blockDim = dim3(jdw2::THREADS);
      cfg.dynamicSmemBytes = jdw2::SMEM_BYTES;
      cfg.stream = st;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = (unsigned)p.mc;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      RNNT_LAUNCH(KID_DW, st, cudaLaunchKernelEx(&cfg, joiner_dw_wide_kernel, tp3, p.h3 ? th3 : th, ths, tp1, to, p));
    } else {
      // (with the pair kernel this launch only works in the rescaling mode: profiled under another id)
      RNNT_LAUNCH(p.pair_plain ? KID_DB : KID_DW, st,
                  launch_pdl(joiner_dw_wide_kernel, grid, jdw2::THREADS, jdw2::SMEM_BYTES, st, tp3, p.h3 ? th3 : th, ths,
                             tp1, to, p));
    }
  } else if (pair) {
    smem_optin(joiner_dw_tc_kernel<true>, jdw::Cfg<true>::SMEM_BYTES);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((vt + 1) / 2 * 2), (d.J + jdw::BN - 1) / jdw::BN, splits);
    cfg.blockDim = dim3(jdw::THREADS);
    cfg.dynamicSmemBytes = jdw::Cfg<true>::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    RNNT_LAUNCH(KID_DW, st, cudaLaunchKernelEx(&cfg, joiner_dw_tc_kernel<true>, tp, th, p));
  } else {
    smem_optin(joiner_dw_tc_kernel<false>, jdw::Cfg<false>::SMEM_BYTES);
    dim3 grid(vt, (d.J + jdw::BN - 1) / jdw::BN, splits);
    CUtensorMap tp3, th3;
    p.h3 = d.J % 64 == 0;
    if (p.h3 && (!make_tmap_bf16_3d(&tp3, g.Pt, 64, d.rows(), d.VP() / 64, (uint64_t)d.VP() * 2, 128, 64, jdw::BK, 2) ||
                 !make_tmap_bf16_3d(&th3, h, 64, d.rows(), d.J / 64, (uint64_t)d.J * 2, 128, 64, jdw::BK, 4)))
      return cudaErrorInvalidValue;
    RNNT_LAUNCH(KID_DW, st, launch_pdl(joiner_dw_tc_kernel<false>, grid, jdw::THREADS, jdw::Cfg<false>::SMEM_BYTES, st, 
                                p.h3 ? tp3 : tp, p.h3 ? th3 : th, p));
  }
  return cudaGetLastError();
}

}  // namespace rnnt
