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
__device__ __forceinline__ uint4 dz_chunk(uint4 pv, float s, float gbs, float gls, int info, int vc, float* fsum) {
  const uint32_t w[4] = {pv.x, pv.y, pv.z, pv.w};
  float g[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    g[2 * i] = s * __uint_as_float(w[i] << 16);
    g[2 * i + 1] = s * __uint_as_float(w[i] & 0xffff0000u);
  }
  if (vc == 0) g[0] -= gbs;
  const int li = info - vc;
  if ((unsigned)li < 8u) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j == li) g[j] -= gls;
  }
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

// byte offset of logical 16-B chunk `c` (0..7) of 128-B row `r` in a SWIZZLE_128B atom stack
__device__ __forceinline__ uint32_t sw128(int r, int c) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}

// ======================================================================= K10
// Frame-aligned row tiles: tile i holds the F = floor(128/S) frames [iF, iF+F) of the flattened
// (n, t) frame index, i.e. rows [iFS, iFS + FS) (the MMA computes 128 rows; the rest is ignored).
// The epilogue forms dpre = dh (1 - h^2) for a 32-column chunk in smem and reduces it there:
//   d_enc[n,t,:] = sum_s dpre[(n,t,s),:]                                      (complete in the tile)
//   d_dec[n,u,:] = sum over band rows (t, s) with p_t + s = u of dpre         (frames covering u are
//   contiguous, Eq. 9; u whose covering frames all lie in the tile are written directly, the <= S
//   u at each end of a tile's utterance segment go to a boundary-partial buffer that
//   ddec_fixup_kernel sums in tile order: deterministic, and dpre never leaves the SM).
namespace jdh {
// 256 output columns per CTA (TMEM 256 of 512 columns, ~102 KB smem): two CTAs per SM, so one
// CTA's epilogue overlaps the other's mainloop.
constexpr int BM = 128, BK = 64, NSUB = 256, MAXN = 256, STAGES = 2;
constexpr int A_BYTES = BM * BK * 2;           // 16 KB, K-major (TMA box 64 v x 128 rows of P~)
constexpr int B_BYTES = MAXN * BK * 2;         // 32 KB, MN-major (4 boxes of 64 j x 64 v)
constexpr int G_BYTES = BM * 16;               // 2 KB: the rows' packed scalars for this k-block's V tile
constexpr int STAGE_BYTES = A_BYTES + B_BYTES + G_BYTES;
constexpr int H_BYTES = BM * 64 * 2;           // 16 KB: one 64-column box of h for the epilogue
constexpr int D_OFF = 4 * H_BYTES;             // dpre staging block [128][32] fp32 after the h boxes
constexpr int MAXSEG = 128;
constexpr int TAB_BYTES = 4 * 128 + MAXSEG * 8 * 4 + 4 * 128 + 16 + 128 * 16 + 3 * 4 * 128;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256 + TAB_BYTES;
constexpr int THREADS = 160;
}  // namespace jdh

struct JoinerDhParams {
  GradSrc g;
  int J, nkb;
  int N, T, U, S, F;
  const int32_t* ranges;   // (N,T) p_t
  const int2* urange;      // (N,U+1) frames [lo, hi) covering u
  const int64_t* bnd;
  float* d_enc;            // (N,T,J) nullable
  float* d_dec;            // (N,U+1,J) nullable
  float* part;             // (ntiles, 2, S, J) boundary partials of d_dec
};

// per-tile utterance segment: live frames f in [fb, fe) of utterance n, token positions [ub, ue],
// its entries e in [off, off + ue - ub + 1); pnext = p at the frame after the segment (if covered)
struct Seg {
  int n, fb, fe, ub, ue, off, pnext, ta;
};

__global__ void __launch_bounds__(jdh::THREADS, 2)
    joiner_dh_tc_kernel(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmW,
                        const __grid_constant__ CUtensorMap tmH, JoinerDhParams p) {
  using namespace jdh;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = tc::align1024(smem_raw);
  uint64_t* loaded = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* full = loaded + STAGES;
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* hfull = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hfull + 1);
  int* sp = reinterpret_cast<int*>(smem + STAGES * STAGE_BYTES + 256);   // [128] p of tile frames (-1 dead)
  Seg* seg = reinterpret_cast<Seg*>(sp + 128);                          // [MAXSEG]
  uint8_t* eseg = reinterpret_cast<uint8_t*>(seg + MAXSEG);             // [128] segment of entry e
  int* nseg_ent = reinterpret_cast<int*>(eseg + 128);                   // {#segments, #entries}
  int4* ent = reinterpret_cast<int4*>(nseg_ent + 4);                   // [128] {fl, fh, u, dst row}
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.S, F = p.F, RT = F * S;
  const long long g0 = (long long)blockIdx.x * F;                      // first flattened frame
  const long long m0 = g0 * S;                                          // first row
  const long long NT = (long long)p.N * p.T;
  const int j0 = blockIdx.y * MAXN;
  const int nj = min(MAXN, p.J - j0);               // columns of this CTA
  const int nsub = (nj + NSUB - 1) / NSUB;
  const int nbox = (nj + 63) / 64;

  // ---- per-frame tables of the tile (parallel global loads): p_t (dead = -1), p_{t+1}, n, t
  int* spn = reinterpret_cast<int*>(ent + 128);                          // [128] p_{t+1}
  int* sfn = spn + 128;                                                  // [128] utterance n
  int* sft = sfn + 128;                                                  // [128] frame t
  if (threadIdx.x < F) {
    const long long g = g0 + threadIdx.x;
    int pv = -1, pn = 0, n = -1, t = 0;
    if (g < NT) {
      n = (int)(g / p.T);
      t = (int)(g - (long long)n * p.T);
      const int Tn = utt_T(p.bnd, n), Un = utt_U(p.bnd, n);
      if (t < Tn && (long long)Un <= (long long)Tn * (S - 1)) {
        pv = p.ranges[(size_t)n * p.T + t];
        if (t + 1 < Tn) pn = p.ranges[(size_t)n * p.T + t + 1];
      }
    }
    sp[threadIdx.x] = pv;
    spn[threadIdx.x] = pn;
    sfn[threadIdx.x] = n;
    sft[threadIdx.x] = t;
  }
  int act = 0;
  for (int i = threadIdx.x; i < RT; i += blockDim.x)
    if (m0 + i < p.g.R && p.g.rowinfo[m0 + i] >= 0) act = 1;
  const bool any = __syncthreads_or(act);

  if (!any) {
    // no live row: d_enc of the tile's frames is zero (d_dec gets nothing from this tile)
    if (p.d_enc)
      for (int idx = threadIdx.x; idx < F * (nj / 4); idx += blockDim.x) {
        const int f = idx / (nj / 4), jq = idx - f * (nj / 4);
        if (g0 + f < NT)
          reinterpret_cast<float4*>(p.d_enc + (size_t)(g0 + f) * p.J + j0)[jq] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    return;
  }
  if (warp == 4 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&loaded[s], 1);
      tc::mbar_init(&full[s], 4);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(tfull, 1);
    tc::mbar_init(hfull, 1);
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmP);
    tc::tma_prefetch(&tmW);
    tc::tma_prefetch(&tmH);
  }
  if (warp == 4) tc::tmem_alloc(tmem_slot, MAXN);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = *tmem_slot;
  const int grows = (int)min((long long)BM, p.g.R - m0);   // rows of the packed-scalar copy

  if (warp < 4) {
    // ---- producers: thread = tile row; transform the 8 chunks of its row in place
    const int rl = threadIdx.x;
    const long long r = m0 + rl;
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < p.nkb; ++kb) {
      const int v0 = kb * BK;
      tc::mbar_wait(&loaded[stage], ph);
      uint8_t* sa = smem + stage * STAGE_BYTES;
      const float4 gq = (rl < grows && rl < RT) ? reinterpret_cast<const float4*>(sa + A_BYTES + B_BYTES)[rl]
                                                : make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
      const int info = __float_as_int(gq.w);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint4* q = reinterpret_cast<uint4*>(sa + sw128(rl, c));
        const uint4 pv = *q;
        *q = info >= 0 ? dz_chunk(pv, gq.x, gq.y, gq.z, info, v0 + c * 8, nullptr) : make_uint4(0, 0, 0, 0);
      }
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&full[stage]);
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
    // ---- tile tables (while the last MMAs drain): utterance segments from the per-frame smem
    // tables, then one entry per token position of a segment: covering frames and destination
    if (threadIdx.x == 0) {
      int ns = 0, ne = 0;
      for (int f = 0; f < F;) {
        if (sp[f] < 0) { ++f; continue; }
        const int n = sfn[f];
        int fe = f + 1;
        while (fe < F && sp[fe] >= 0 && sfn[fe] == n) ++fe;
        Seg q;
        q.n = n; q.fb = f; q.fe = fe; q.ta = sft[f];
        q.ub = sp[f];
        q.ue = min(utt_U(p.bnd, n), sp[fe - 1] + S - 1);
        q.off = ne;
        q.pnext = spn[fe - 1];
        if (ns < MAXSEG) {
          seg[ns] = q;
          for (int e = 0; e <= q.ue - q.ub && ne + e < 128; ++e) eseg[ne + e] = (uint8_t)ns;
          ++ns;
          ne += q.ue - q.ub + 1;
        }
        f = fe;
      }
      nseg_ent[0] = ns;
      nseg_ent[1] = min(ne, 128);
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    //   dst >= 0: row n(U+1)+u of d_dec (complete here); dst < 0: row -(1+dst) of the partial buffer
    if (threadIdx.x < nseg_ent[1]) {
      const int e = threadIdx.x;
      const Seg q = seg[eseg[e]];
      const int u = q.ub + (e - q.off);
      const int2 cov = p.urange[(size_t)q.n * (p.U + 1) + u];           // frames [lo, hi) covering u
      const int fl = max(q.fb, cov.x - q.ta + q.fb), fh = min(q.fe, cov.y - q.ta + q.fb);
      const int tb = q.ta + (q.fe - q.fb);
      int dst;
      if (cov.x >= q.ta && cov.y <= tb) dst = q.n * (p.U + 1) + u;                               // complete here
      else if (cov.x < q.ta) dst = -1 - (int)((blockIdx.x * 2 + 0) * S + (u - q.ub));          // left boundary
      else dst = -1 - (int)((blockIdx.x * 2 + 1) * S + (u - q.pnext));                          // right boundary
      ent[e] = make_int4(fl, fh, u, dst);
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    // ---- epilogue
    tc::mbar_wait(tfull, 0);
    tc::fence_after_sync();
    tc::mbar_wait(hfull, 0);
    const bool live = rl < RT && r < p.g.R && p.g.rowinfo[r] >= 0;
    const uint32_t tl = tbase + ((uint32_t)(32 * warp) << 16);
    // dpre chunk staging: row r, float4 group q (columns 4q..4q+3) at D4[r * 8 + (q ^ (r & 7))]
    float4* D4 = reinterpret_cast<float4*>(smem + D_OFF);
    const int nseg = nseg_ent[0], nent = nseg_ent[1];
    for (int c0 = 0; c0 < nj; c0 += 32) {
      float acc[32];
      tc::tmem_ld32(tl + c0, acc);
      const uint8_t* hb = smem + (c0 >> 6) * H_BYTES;         // 64-column box of h
      const int qh = ((c0 >> 5) & 1) * 4;                     // 16-B chunk of the 32-column half
      const int nq = min(4, (nj - c0) / 8);                   // J % 8 == 0
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float out[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (q < nq && live) {
          const uint4 hv = *reinterpret_cast<const uint4*>(hb + sw128(rl, qh + q));
          const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float ha = __uint_as_float(hw[i] << 16), hb2 = __uint_as_float(hw[i] & 0xffff0000u);
            out[2 * i] = acc[8 * q + 2 * i] * (1.f - ha * ha);            // d tanh
            out[2 * i + 1] = acc[8 * q + 2 * i + 1] * (1.f - hb2 * hb2);
          }
        }
        D4[rl * 8 + ((2 * q) ^ (rl & 7))] = make_float4(out[0], out[1], out[2], out[3]);
        D4[rl * 8 + ((2 * q + 1) ^ (rl & 7))] = make_float4(out[4], out[5], out[6], out[7]);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const int ncol4 = min(32, nj - c0) / 4;
      // d_enc: one float4 output per (frame, 4-column group)
      if (p.d_enc)
        for (int idx = threadIdx.x; idx < F * 8; idx += 128) {
          const int f = idx >> 3, q = idx & 7;
          if (q < ncol4 && g0 + f < NT) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int s = 0; s < S; ++s) {
              const int rr = f * S + s;
              const float4 x = D4[rr * 8 + (q ^ (rr & 7))];
              v.x += x.x; v.y += x.y; v.z += x.z; v.w += x.w;
            }
            reinterpret_cast<float4*>(p.d_enc + (size_t)(g0 + f) * p.J + j0 + c0)[q] = v;
          }
        }
      // d_dec: one float4 output per (token position of a segment, 4-column group)
      if (p.d_dec)
        for (int idx = threadIdx.x; idx < nent * 8; idx += 128) {
          const int e = idx >> 3, q = idx & 7;
          if (q >= ncol4) continue;
          const int4 en = ent[e];
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int f = en.x; f < en.y; ++f) {
            const int rr = f * S + (en.z - sp[f]);
            const float4 x = D4[rr * 8 + (q ^ (rr & 7))];
            v.x += x.x; v.y += x.y; v.z += x.z; v.w += x.w;
          }
          float* dst = en.w >= 0 ? p.d_dec + (size_t)en.w * p.J : p.part + (size_t)(-1 - en.w) * p.J;
          reinterpret_cast<float4*>(dst + j0 + c0)[q] = v;
        }
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    (void)nseg;
  } else if (lane == 0) {
    // ---- warp 4 lane 0: TMA for A = P~[m0.., kb*64..], B = W[kb*64.., j0..] and the rows' scalars
    const uint32_t gbytes = (uint32_t)grows * 16u;
    const uint32_t bytes = A_BYTES + (uint32_t)nbox * 64 * BK * 2 + gbytes;
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < p.nkb; ++kb) {
      tc::mbar_wait(&empty[stage], ph ^ 1);
      uint8_t* sa = smem + stage * STAGE_BYTES;
      tc::mbar_arrive_expect_tx(&loaded[stage], bytes);
      tc::tma_load_2d(sa, &tmP, &loaded[stage], kb * BK, (int)m0);
      for (int bx = 0; bx < nbox; ++bx)
        tc::tma_load_2d(sa + A_BYTES + bx * (64 * BK * 2), &tmW, &loaded[stage], j0 + bx * 64, kb * BK);
      tc::bulk_load(sa + A_BYTES + B_BYTES, p.g.gpk + (size_t)((kb * BK) >> 7) * p.g.R + m0, gbytes, &loaded[stage]);
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
    // h tiles for the epilogue, into the idle stage buffers once the MMAs are done
    tc::mbar_wait(tfull, 0);
    tc::mbar_arrive_expect_tx(hfull, (uint32_t)nbox * H_BYTES);
    for (int bx = 0; bx < nbox; ++bx) tc::tma_load_2d(smem + bx * H_BYTES, &tmH, hfull, j0 + bx * 64, (int)m0);
  } else if (lane == 1) {
    // ---- warp 4 lane 1: MMA issuer
    constexpr uint32_t idesc = tc::idesc_bf16(BM, NSUB, false, true);
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < p.nkb; ++kb) {
      tc::mbar_wait(&full[stage], ph);
      tc::fence_after_sync();
      const uint32_t a = tc::smem_u32(smem + stage * STAGE_BYTES), b = a + A_BYTES;
      for (int ns = 0; ns < nsub; ++ns) {
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)
          tc::mma_bf16(tbase + ns * NSUB, tc::sdesc(a + 32 * k, 16, 1024),
                       tc::sdesc(b + ns * 4 * (64 * BK * 2) + 2048 * k, 64 * BK * 2, 1024), idesc, (kb | k) != 0);
      }
      tc::mma_commit(&empty[stage]);
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
    tc::mma_commit(tfull);
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 4) tc::tmem_dealloc(tbase, MAXN);
}

// d_dec for the token positions whose covering frames span several tiles (sum of the boundary
// partials in tile order), and zeros for u > U_n / infeasible utterances.  Positions complete in
// one tile were written by joiner_dh_tc_kernel and are left untouched.  One warp per (n, u).
__global__ void __launch_bounds__(256) ddec_fixup_kernel(const int32_t* __restrict__ ranges,
                                                         const int2* __restrict__ urange,
                                                         const int64_t* __restrict__ bnd, int N, int T, int U, int S,
                                                         int F, int J, const float* __restrict__ part,
                                                         float* __restrict__ d_dec) {
  const long long nu = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (nu >= (long long)N * (U + 1)) return;
  const int n = (int)(nu / (U + 1)), u = (int)(nu - (long long)n * (U + 1));
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  const int J4 = J / 4;
  float4* dst = reinterpret_cast<float4*>(d_dec + (size_t)nu * J);
  if (u > Un || (long long)Un > (long long)Tn * (S - 1)) {
    for (int j = lane; j < J4; j += 32) dst[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const int2 cov = urange[nu];
  const long long gbase = (long long)n * T;
  const long long k0 = (gbase + cov.x) / F, k1 = (gbase + cov.y - 1) / F;
  if (k0 == k1) return;
  const int32_t* pr = ranges + (size_t)n * T;
  const int tb0 = (int)((k0 + 1) * F - gbase);                     // first frame of tile k0 + 1
  const float4* first = reinterpret_cast<const float4*>(part + (((size_t)k0 * 2 + 1) * S + (u - pr[tb0])) * J);
  float4 acc[4];
  for (int q = 0; q < 4; ++q) {
    const int j = lane + 32 * q;
    acc[q] = j < J4 ? first[j] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (long long k = k0 + 1; k <= k1; ++k) {
    const int ta = (int)(k * F - gbase);
    const float4* src = reinterpret_cast<const float4*>(part + (((size_t)k * 2 + 0) * S + (u - pr[ta])) * J);
    for (int q = 0; q < 4; ++q) {
      const int j = lane + 32 * q;
      if (j < J4) {
        const float4 x = src[j];
        acc[q].x += x.x; acc[q].y += x.y; acc[q].z += x.z; acc[q].w += x.w;
      }
    }
  }
  for (int q = 0; q < 4; ++q) {
    const int j = lane + 32 * q;
    if (j < J4) dst[j] = acc[q];
  }
  for (int j = lane + 128; j < J4; j += 32) {   // J > 512: remaining columns
    float4 v = first[j];
    for (long long k = k0 + 1; k <= k1; ++k) {
      const int ta = (int)(k * F - gbase);
      const float4 x = reinterpret_cast<const float4*>(part + (((size_t)k * 2 + 0) * S + (u - pr[ta])) * J)[j];
      v.x += x.x; v.y += x.y; v.z += x.z; v.w += x.w;
    }
    dst[j] = v;
  }
}

// ======================================================================= K11
namespace jdw {
// 2 stages (~108 KB smem, TMEM 256 columns): two CTAs per SM keep four stages in flight per SM.
constexpr int BM = 128, BN = 256, BK = 64, STAGES = 2;
constexpr int A_BYTES = BM * BK * 2;     // 16 KB, MN-major (2 TMA boxes of 64 v x 64 rows of P~)
constexpr int B_BYTES = BN * BK * 2;     // 32 KB, MN-major (4 boxes of 64 j x 64 rows of h)
constexpr int G_BYTES = BK * 16;         // 1 KB: the k-block rows' packed scalars for this V tile
constexpr int STAGE_BYTES = A_BYTES + B_BYTES + G_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256 + 128 * 16 * 4;
constexpr int THREADS = 160;
}  // namespace jdw

struct JoinerDwParams {
  GradSrc g;
  int J;
  long long kb_per_split, nkb_total;
  float* dWp;   // (splits, V, J)
  float* dbp;   // (splits, V)
};

__global__ void __launch_bounds__(jdw::THREADS, 2)
    joiner_dw_tc_kernel(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmH,
                        JoinerDwParams p) {
  using namespace jdw;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = tc::align1024(smem_raw);
  uint64_t* loaded = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* full = loaded + STAGES;
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  float* dbs = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256);     // [8 row groups][128 v]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int v0 = blockIdx.x * BM, j0 = blockIdx.y * BN, split = blockIdx.z;
  const long long kb0 = (long long)split * p.kb_per_split;
  const long long kb1 = min(p.nkb_total, kb0 + p.kb_per_split);
  const int nkb = (int)max(0LL, kb1 - kb0);
  const int V = p.g.V;
  const int nj = min(BN, p.J - j0);
  const int nbox = (nj + 63) / 64;
  const int vtile = v0 >> 7;

  if (warp == 4 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&loaded[s], 1);
      tc::mbar_init(&full[s], 4);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(tfull, 1);
    tc::fence_barrier_init();
    tc::tma_prefetch(&tmP);
    tc::tma_prefetch(&tmH);
  }
  if (warp == 4) tc::tmem_alloc(tmem_slot, 256);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = *tmem_slot;

  if (warp < 4) {
    // ---- producers: thread handles v chunk c (8 logits) of rows g8 + 8 i of each k-block
    const int c = threadIdx.x & 15;          // 8-v chunk 0..15
    const int g8 = threadIdx.x >> 4;         // row group 0..7
    float dsum[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const bool want_db = blockIdx.y == 0;
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      const long long rb = (kb0 + kb) * BK;
      const int grows = (int)min((long long)BK, p.g.R - rb);
      tc::mbar_wait(&loaded[stage], ph);
      uint8_t* sa = smem + stage * STAGE_BYTES;
      const float4* gq = reinterpret_cast<const float4*>(sa + A_BYTES + B_BYTES);
#pragma unroll 4
      for (int i = 0; i < 8; ++i) {
        const int rl = g8 + 8 * i;
        const float4 sr = rl < grows ? gq[rl] : make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
        const int info = __float_as_int(sr.w);
        uint4* q = reinterpret_cast<uint4*>(sa + (c >> 3) * (64 * BK * 2) + sw128(rl, c & 7));
        const uint4 pv = *q;
        *q = info >= 0 ? dz_chunk(pv, sr.x, sr.y, sr.z, info, v0 + c * 8, want_db ? dsum : nullptr)
                       : make_uint4(0, 0, 0, 0);
      }
      tc::fence_proxy_async();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&full[stage]);
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
    // ---- warp 4 lane 0: TMA for A = P~[rows, v0..v0+127] (2 boxes), B = h[rows, j0..] and the scalars
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      const long long rb = (kb0 + kb) * BK;
      const uint32_t gbytes = (uint32_t)min((long long)BK, p.g.R - rb) * 16u;
      const uint32_t bytes = A_BYTES + (uint32_t)nbox * 64 * BK * 2 + gbytes;
      tc::mbar_wait(&empty[stage], ph ^ 1);
      uint8_t* sa = smem + stage * STAGE_BYTES;
      tc::mbar_arrive_expect_tx(&loaded[stage], bytes);
      tc::tma_load_2d(sa, &tmP, &loaded[stage], v0, (int)rb);
      tc::tma_load_2d(sa + 64 * BK * 2, &tmP, &loaded[stage], v0 + 64, (int)rb);
      for (int bx = 0; bx < nbox; ++bx)
        tc::tma_load_2d(sa + A_BYTES + bx * (64 * BK * 2), &tmH, &loaded[stage], j0 + bx * 64, (int)rb);
      tc::bulk_load(sa + A_BYTES + B_BYTES, p.g.gpk + (size_t)vtile * p.g.R + rb, gbytes, &loaded[stage]);
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
  } else if (lane == 1 && nkb > 0) {
    // ---- warp 4 lane 1: MMA issuer
    constexpr uint32_t idesc = tc::idesc_bf16(BM, BN, true, true);
    int stage = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      tc::mbar_wait(&full[stage], ph);
      tc::fence_after_sync();
      const uint32_t a = tc::smem_u32(smem + stage * STAGE_BYTES), b = a + A_BYTES;
#pragma unroll
      for (int k = 0; k < BK / 16; ++k)
        tc::mma_bf16(tbase, tc::sdesc(a + 2048 * k, 64 * BK * 2, 1024), tc::sdesc(b + 2048 * k, 64 * BK * 2, 1024),
                     idesc, (kb | k) != 0);
      tc::mma_commit(&empty[stage]);
      if (++stage == STAGES) { stage = 0; ph ^= 1; }
    }
    tc::mma_commit(tfull);
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 4) tc::tmem_dealloc(tbase, 256);
}

// ======================================================================= host
cudaError_t joiner_dh_launch(const Dims& d, const GradSrc& g, const uint16_t* h, const uint16_t* W,
                             const int32_t* ranges, const int2* urange, const int64_t* bnd, float* d_enc,
                             float* d_dec, float* part, cudaStream_t st) {
  CUtensorMap tp, tw, th;
  if (!make_tmap_bf16_2d(&tp, g.Pt, d.VP(), d.rows(), (uint64_t)d.VP() * 2, jdh::BK, jdh::BM)) return cudaErrorInvalidValue;
  if (!make_tmap_bf16_2d(&tw, W, d.J, d.V, (uint64_t)d.J * 2, 64, 64)) return cudaErrorInvalidValue;
  if (!make_tmap_bf16_2d(&th, h, d.J, d.rows(), (uint64_t)d.J * 2, 64, jdh::BM)) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(joiner_dh_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, jdh::SMEM_BYTES);
    attr = true;
  }
  const int F = d.dh_frames();
  JoinerDhParams p{g, d.J, (d.V + jdh::BK - 1) / jdh::BK, d.N, d.T, d.U, d.S, F, ranges, urange, bnd, d_enc, d_dec,
                   part};
  dim3 grid((unsigned)d.dh_tiles(), (d.J + jdh::MAXN - 1) / jdh::MAXN);
  RNNT_LAUNCH(KID_DH, st, joiner_dh_tc_kernel<<<grid, jdh::THREADS, jdh::SMEM_BYTES, st>>>(tp, tw, th, p));
  if (d_dec)
    RNNT_LAUNCH(KID_DDEC, st, ddec_fixup_kernel<<<(unsigned)(((long long)d.N * d.U1() + 7) / 8), 256, 0, st>>>(
        ranges, urange, bnd, d.N, d.T, d.U, d.S, F, d.J, part, d_dec));
  return cudaGetLastError();
}

cudaError_t joiner_dw_launch(const Dims& d, const GradSrc& g, const uint16_t* h, float* dWp, float* dbp,
                             int splits, cudaStream_t st) {
  CUtensorMap tp, th;
  if (!make_tmap_bf16_2d(&tp, g.Pt, d.VP(), d.rows(), (uint64_t)d.VP() * 2, 64, jdw::BK)) return cudaErrorInvalidValue;
  if (!make_tmap_bf16_2d(&th, h, d.J, d.rows(), (uint64_t)d.J * 2, 64, 64)) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(joiner_dw_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, jdw::SMEM_BYTES);
    attr = true;
  }
  const long long nkb = (d.rows() + jdw::BK - 1) / jdw::BK;
  const long long per = (nkb + splits - 1) / splits;
  JoinerDwParams p{g, d.J, per, nkb, dWp, dbp};
  dim3 grid((d.V + jdw::BM - 1) / jdw::BM, (d.J + jdw::BN - 1) / jdw::BN, splits);
  RNNT_LAUNCH(KID_DW, st, joiner_dw_tc_kernel<<<grid, jdw::THREADS, jdw::SMEM_BYTES, st>>>(tp, th, p));
  return cudaGetLastError();
}

}  // namespace rnnt
