// pruned.cu — stages 3-4: gather on the band, full joiner with fused
// log-softmax / pick / logit gradient (function merging), pruned recursion
// (P:253-256), joiner gradients.
//
// Kernels
//   K7  prune_kernel          h = bf16(tanh(enc[t] + dec[p_t+s])), masked rows 0
//   K7b rowinfo_kernel        per band row: label y_{u+1} (V at u=U_n), -1 if masked/padded
//   K8  ZGemm + softmax_rows  z = W h + b; lse, picks, P~ = bf16(exp(z - m_tile)), m_tile
//   K9  pruned_alpha/beta     banded wavefront, one lane per slot s, frames advance per lane
//   K9c pruned_combine        g_b = empty'_p, g_l = y'_p per row; sc = gs (g_b+g_l) e^{m_tile-lse}
//   K10 DhGemm + reduce       dpre = (W^T dz) (1-h^2); d_enc = sum_s dpre; d_dec gather-reduce
//   K11 DwGemm (split-K)      d_w = sum dz h^T, d_b = sum dz, deterministic split reduction
#include <algorithm>

#include "common.cuh"
#include "launch.h"
#include "tc.cuh"
#include "workspace.h"

namespace rnnt {

__device__ __forceinline__ float warp_max_uniform_p(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

cudaError_t joiner_fwd_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, const uint16_t* W,
                              const uint16_t* b, cudaStream_t st);
struct GradSrc {
  const uint16_t* Pt;
  const float4* gpk;
  const int32_t* rowinfo;
  long long R;
  int V, VP, ntile;
};
cudaError_t joiner_dh_launch(const Dims& d, const GradSrc& g, const uint16_t* h, const uint16_t* W, const int* live,
                             const int* nlive, long long ntiles, float* dpre, const int* tscale, const float* gsp,
                             cudaStream_t st);
cudaError_t scale_rows_launch(const Dims& d, const GradSrc& g, const uint16_t* h, const int* tscale, const int* live,
                              const int* nlive, long long ntiles, uint16_t* Hs, cudaStream_t st);
cudaError_t joiner_dw_launch(const Dims& d, const GradSrc& g, const uint16_t* h, const uint16_t* Hs, const int* tscale, const int* live, const int* nlive, float* dWp, float* dbp, int splits,
                             cudaStream_t st);

// ------------------------------------------------------------------ K7 prune
// Block (J/8, FPB): thread (x, y) owns the 8 columns 8x of frame blockIdx.x * FPB + y and walks its
// S band rows, so enc[t] is loaded once per thread and the per-frame index work (ranges, lengths,
// row addresses) is paid once per S rows instead of per 16-B output (the kernel is issue-bound on
// the accurate tanh; the division-based (slot, column) split cost a third of its instructions).
// Rows of padded frames and masked slots are written as zeros (the joiner GEMMs read whole
// 128-row tiles).
__global__ void __launch_bounds__(1024) prune_kernel(const float* __restrict__ enc, const float* __restrict__ dec,
                                                     const int32_t* __restrict__ ranges, const int64_t* __restrict__ bnd,
                                                     int N, int T, int U, int J, int S, uint16_t* __restrict__ h) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  const unsigned nt = blockIdx.x * blockDim.y + threadIdx.y;   // N T < 2^31 (checked by the launcher)
  if (nt >= (unsigned)N * (unsigned)T) return;
  const int n = (int)(nt / (unsigned)T), t = (int)(nt - (unsigned)n * (unsigned)T);
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  const int j0 = threadIdx.x * 8;
  const bool live = t < Tn;
  const int p = live ? ranges[nt] : 0;
  float4 e0 = make_float4(0.f, 0.f, 0.f, 0.f), e1 = e0;
  if (live) {
    const float* e = enc + (size_t)nt * J + j0;
    e0 = __ldg(reinterpret_cast<const float4*>(e));
    e1 = __ldg(reinterpret_cast<const float4*>(e + 4));
  }
  const float* dbase = dec + ((size_t)n * (U + 1) + p) * J + j0;
  uint4* out = reinterpret_cast<uint4*>(h + (size_t)nt * S * J + j0);
  const int J8 = J / 8;
  for (int s = 0; s < S; ++s) {
    uint4 o = make_uint4(0, 0, 0, 0);
    if (live && p + s <= Un) {
      const float* d = dbase + (size_t)s * J;
      const float4 d0 = __ldg(reinterpret_cast<const float4*>(d)), d1 = __ldg(reinterpret_cast<const float4*>(d + 4));
      const float x[8] = {e0.x + d0.x, e0.y + d0.y, e0.z + d0.z, e0.w + d0.w,
                          e1.x + d1.x, e1.y + d1.y, e1.z + d1.z, e1.w + d1.w};
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const __nv_bfloat162 h2 = __floats2bfloat162_rn(tanh_fast(x[2 * q]), tanh_fast(x[2 * q + 1]));
        w[q] = *reinterpret_cast<const uint32_t*>(&h2);
      }
      o = make_uint4(w[0], w[1], w[2], w[3]);
    }
    out[(size_t)s * J8] = o;
  }
}

// Does 128-row tile i of the band rows hold a live row?  Row (n, t, s) is live iff t < T_n, the utterance
// is feasible and p_t + s <= U_n; the s = 0 row of a live frame always is (p_t <= max(0, U_n - S + 1)).  So
// the tile is live iff its first frame's first row in the tile is, or a later frame of the tile is a live
// frame -- O(utterances spanned) per tile instead of a pass over its 128 rows.
__device__ __forceinline__ bool band_tile_live(long long i, const int32_t* __restrict__ ranges,
                                               const int64_t* __restrict__ bnd, int T, int S, long long R) {
  const long long r0 = i * 128, r1 = min(R, r0 + 128) - 1;
  const long long f0 = r0 / S, f1 = r1 / S;
  const int s0 = (int)(r0 - f0 * S);
  {
    const int n = (int)(f0 / T), t = (int)(f0 - (long long)n * T);
    const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
    if (t < Tn && (long long)Un <= (long long)Tn * (S - 1) && ranges[f0] + s0 <= Un) return true;
  }
  for (long long f = f0 + 1; f <= f1;) {
    const int n = (int)(f / T), t = (int)(f - (long long)n * T);
    const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
    if (t < Tn && (long long)Un <= (long long)Tn * (S - 1)) return true;
    f = (long long)(n + 1) * T;   // the utterance's later frames are padded as well
  }
  return false;
}

// blocks [0, nb_rows): per band row label info (and the frames covering each u); the last block pads the
// bias to fp32 (VP columns, zero beyond V) for the joiner epilogue and writes the 128-row tile liveness
// and the ascending list of live tiles (count at live[ntiles]) that the joiner kernels work through.
__global__ void rowinfo_kernel(const int32_t* __restrict__ ranges, const int64_t* __restrict__ sym,
                               const int64_t* __restrict__ bnd, int N, int T, int U, int V, int S,
                               int32_t* __restrict__ rowinfo, int2* __restrict__ urange,
                               const uint16_t* __restrict__ bias_bf16, int VP, float* __restrict__ bias,
                               float* __restrict__ bmax, uint8_t* __restrict__ tlive, int* __restrict__ tcounter,
                               int tscale0, float gs, int* __restrict__ live) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  if (blockIdx.x == gridDim.x - 1) {
    if (threadIdx.x == 0) {
      tcounter[0] = 0;
      tcounter[1] = tscale0;   // PrunedWS::tscale (the joiner forward raises it on a per-tile offset)
      tcounter[2] = __float_as_int(gs);   // PrunedWS::gsp (the joiner backward's fp16 dpre scale)
    }
    // padded columns v >= V get -inf: the joiner epilogue's z = acc + b is then -inf there (W rows past
    // V are zero-filled by TMA) and e^(z - m) = 0 without a per-element mask.  The row blocks convert one
    // 256-column slice each (below); this block only the columns past their reach, and it takes the tile
    // maxima from the bf16 input directly (as one block's serial loops the conversion and the maxima were
    // ~20 us of this kernel at V = 5000-8000, on the step's critical path)
    for (int v = (int)(gridDim.x - 1) * (int)blockDim.x + threadIdx.x; v < VP; v += blockDim.x)
      bias[v] = v < V ? bf16_bits_to_f(bias_bf16[v]) : neg_inf_f();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int tl = warp; tl < VP / 128; tl += blockDim.x / 32) {   // bias max per 128-column tile
      float m = neg_inf_f();
#pragma unroll
      for (int j = lane; j < 128; j += 32)
        if (tl * 128 + j < V) m = fmaxf(m, bf16_bits_to_f(bias_bf16[tl * 128 + j]));
      m = warp_max(m);
      if (lane == 0) bmax[tl] = m;
    }
    // tile liveness and the ascending live-tile list: thread k takes a contiguous range of tiles and
    // writes its live ones at its exclusive-scan offset (deterministic order: the d_w split-K partials
    // follow it)
    __shared__ int wsum[32];
    const long long R = (long long)N * T * S, ntiles = (R + 127) / 128;
    const long long per = (ntiles + blockDim.x - 1) / blockDim.x;
    const long long i0 = min(ntiles, (long long)threadIdx.x * per), i1 = min(ntiles, i0 + per);
    int c = 0;
    for (long long i = i0; i < i1; ++i) {
      const bool lv = band_tile_live(i, ranges, bnd, T, S, R);
      tlive[i] = lv ? 1 : 0;
      c += lv;
    }
    int x = c;   // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int sw = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, sw, o);
        if (lane >= o) sw += y;
      }
      wsum[lane] = sw;   // inclusive over warps
    }
    __syncthreads();
    int off = x - c + (warp > 0 ? wsum[warp - 1] : 0);
    for (long long i = i0; i < i1; ++i)
      if (tlive[i]) live[off++] = (int)i;
    if (threadIdx.x == blockDim.x - 1) live[ntiles] = off;
    return;
  }
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long R = (long long)N * T * S;
  if (r < VP) bias[r] = r < V ? bf16_bits_to_f(bias_bf16[r]) : neg_inf_f();   // this block's slice of the fp32 bias
  int info = -1;
  if (r < R) {
    const int s = (int)(r % S);
    const long long nt = r / S;
    const int t = (int)(nt % T), n = (int)(nt / T);
    const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
    const bool feasible = (long long)Un <= (long long)Tn * (S - 1);
    if (t < Tn && feasible) {
      const int32_t* p = ranges + (size_t)n * T;
      const int u = p[t] + s;
      if (u < Un) {
        long long y = sym[(size_t)n * U + u];
        info = (y >= 1 && y < V) ? (int)y : V;
      } else if (u == Un) {
        info = V;  // no label arc at u = U_n (y(t,U) = -inf)
      }
      if (s == 0) {
        // Frames covering token position u form the contiguous range [lo(u), hi(u)) (p monotone,
        // Eq. 9).  Frame t is the first cover of u in (p_{t-1}+S-1, p_t+S-1] and the last cover of
        // u in [p_t, p_{t+1}-1]; over t these intervals partition [0, U_n], so each entry is
        // written once.
        int2* ur = urange + (size_t)n * (U + 1);
        const int a0 = (t == 0) ? 0 : p[t - 1] + S;
        const int a1 = min(p[t] + S - 1, Un);
        for (int uu = a0; uu <= a1; ++uu) ur[uu].x = t;
        const int b1 = (t == Tn - 1) ? Un : p[t + 1] - 1;
        for (int uu = p[t]; uu <= b1; ++uu) ur[uu].y = t + 1;
      }
    }
    rowinfo[r] = info;
  }
}

// ------------------------------------------------------------------ K9 pruned recursion
// Eq. 3 on the band (Fig. 1b lattice) as a chunked scan over frames in the
// (log-add, +) semiring.  Slot s of frame t is node (t, p_t + s).  Forward, frame t >= 1:
//   h[s] = alpha(t-1, s + d_t) + empty(t-1, s + d_t)        (d_t = p_t - p_{t-1}; -inf if s+d_t >= S)
//   alpha(t, s) = LogAdd(h[s], alpha(t, s-1) + y(t, s-1))    (the vertical chain inside the frame)
// i.e. alpha_t = alpha_{t-1} (x) M_t with an S x S transfer matrix M_t.  Backward mirrors it:
//   g[s] = beta(t+1, s - d_{t+1}) + empty(t, s),  beta(t, s) = LogAdd(g[s], beta(t, s+1) + y(t, s)),
// with beta(T-1, U - p_{T-1}) = empty(T-1, U) (the terminal blank).
// Instead of T_n + U_n dependent anti-diagonal steps the kernel does three short phases:
//   A  (parallel over chunks of C frames) the chunk transfer matrix P_c = M_{t0} (x) ... (x) M_{t1-1},
//      lane s of an S-lane segment holding column s (forward) / row s (backward) in registers;
//   B  (one segment) the boundary vectors alpha_{end of chunk c} = alpha_{start} (x) P_c, sequentially;
//   C  (parallel over chunks) every frame of the chunk from its boundary vector; writes alpha-hat.
// The frame step is one shuffle (the band shift d_t) plus S-1 shuffle + LogAdd steps (the chain).
// Precision: every vector / matrix is rebased before each frame by an integer (exact in fp32)
// taken from slot 0 -- node (t, p_t) is reachable from (0,0) and reaches (T-1, U_n) on every
// consistent band (Eq. 9-10), so its value is finite -- and the shifts are summed in fp64 per frame:
//   alpha(t,s) log2e = ap[r] + Af[n,t],  beta(t,s) log2e = bp[r] + Bf[n,t].
// Arcs are base 2 (px2 = y log2e, py2 = empty log2e, kNegBig off the lattice / at masked slots).
__device__ __forceinline__ float lae2(float a, float b) {
  const float m = fmaxf(a, b);
  return m + lg2_approx(1.0f + ex2_approx(-fabsf(a - b)));
}
__device__ __forceinline__ float rebase_of(float v) { return v > -1e29f ? rintf(v) : 0.f; }

__device__ __forceinline__ uint32_t cluster_dim_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctaid.x;" : "=r"(r));
  return r;
}
// diagnostics: per (utterance, direction) CTA timestamps {start, staged, phase A, phase B, phase C}
#ifdef RNNT_DIAGNOSTICS
__device__ unsigned long long* g_scan_trace = nullptr;
void set_scan_trace(void* buf) { cudaMemcpyToSymbol(g_scan_trace, &buf, sizeof(buf)); }
#else
constexpr unsigned long long* g_scan_trace = nullptr;   // product build: tracing compiled out
#endif
__device__ __forceinline__ void scan_trace(int k) {
  if (g_scan_trace && threadIdx.x == 0 && blockIdx.x % max(1u, (unsigned)cluster_dim_x()) == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_scan_trace[((size_t)(blockIdx.x / cluster_dim_x()) * 2 + blockIdx.y) * 8 + k] = t;
  }
}

struct StepIn {
  int t, d;
  bool act;
  float py, px;
};

struct ScanParams {
  const float *px2, *py2;
  const int32_t* ranges;
  const int64_t* bnd;
  int T, S, C, ncmax;
  float *ap, *bp;
  double *Af, *Bf;   // (N, T) per-frame shifts (log2 units)
  double* Lp;
  float* loss;
  int32_t* status;
  int G;             // CTAs per (utterance, direction): a thread-block cluster sharing the chunk work
  int staged;        // 1: the utterance's arcs and bounds are staged in shared memory (T S 8 + T 4 bytes
                     // fit); 0 (long utterances): every phase reads them from global memory (L2)
  int prefix;        // 1: phase B as a parallel (Hillis-Steele) prefix of the chunk matrices over the whole
                     // rank-0 CTA instead of a chain of nc vector-matrix steps (small S)
};

// SMAX: register rows per lane; SC: the band width S as a compile-time constant (0: runtime S <= SMAX),
// so that the per-row loops unroll without branches and the rows' shuffles and LogAdds interleave.
template <int SMAX, int SC>
__global__ void __launch_bounds__(256) pruned_scan_kernel(ScanParams q) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // a cluster of G CTAs per (utterance, direction): phases A and C are spread over its CTAs (chunk
  // c goes to rank c % G), the chunk matrices land in the rank-0 CTA's shared memory (DSMEM
  // stores), rank 0 runs the boundary chain (B), the others read the boundary vectors back
  const int G = q.G;
  const int rank = G > 1 ? (int)tc::cluster_ctarank() : 0;
  const int n = blockIdx.x / G;
  const bool fwd = blockIdx.y == 0;
  const int S = SC > 0 ? SC : q.S, C = q.C;
  constexpr int KR = SC > 0 ? SC : SMAX;     // rows actually carried
  const int Tn = utt_T(q.bnd, n), Un = utt_U(q.bnd, n);
  const bool feasible = (long long)Un <= (long long)Tn * (S - 1);
  if (!feasible) {                 // (every CTA of the cluster returns here: same utterance)
    if (fwd && threadIdx.x == 0 && rank == 0) {
      q.Lp[n] = neg_inf_d();
      q.loss[n] = __int_as_float(0x7f800000);  // +inf: no band-respecting path (kept visible, D16)
      set_status(q.status, n, kStatusInfeasible);
    }
    return;
  }
  scan_trace(0);
  // smem: chunk matrices Pm[c][lane s][i], their shifts, boundary vectors and their shifts, then
  // the utterance's band arcs and bounds (staged once, coalesced: every phase reads them from smem)
  float* Pm = reinterpret_cast<float*>(smem_raw);
  float* psh = Pm + (size_t)q.ncmax * S * S;
  float* bv = psh + q.ncmax;
  const size_t mat_bytes = ((((size_t)q.ncmax * S * S + q.ncmax + (size_t)(q.ncmax + 1) * S) * 4 + 15) / 16) * 16;
  double* bsh = reinterpret_cast<double*>(smem_raw + mat_bytes);
  float* PXs = reinterpret_cast<float*>(smem_raw + mat_bytes + (size_t)(q.ncmax + 1) * 8);
  float* PYs = PXs + (size_t)q.T * S;
  int* prs = reinterpret_cast<int*>(PYs + (size_t)q.T * S);
  // phase B prefix buffers (q.prefix): a second set of nc S x S matrices and two fp64 shift arrays, after the
  // staged arcs and bounds (or straight after the chunk data when nothing is staged)
  unsigned char* pfx_base = q.staged ? reinterpret_cast<unsigned char*>(prs + q.T)
                                     : reinterpret_cast<unsigned char*>(PXs);
  pfx_base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(pfx_base) + 15) & ~uintptr_t(15));
  const size_t rb = (size_t)n * q.T * S;
  if (q.staged) {
    const int m = Tn * S;
    const float* gx = q.px2 + rb;
    const float* gy = q.py2 + rb;
    // 8 independent loads per array in flight per thread (one load per iteration left the staging
    // latency-bound: 19 us at c4)
    constexpr int U8 = 8;
    for (int i0 = threadIdx.x; i0 < m; i0 += U8 * blockDim.x) {
      float x[U8], y[U8];
#pragma unroll
      for (int k = 0; k < U8; ++k) {
        const int i = i0 + k * blockDim.x;
        x[k] = i < m ? gx[i] : 0.f;
        y[k] = i < m ? gy[i] : 0.f;
      }
#pragma unroll
      for (int k = 0; k < U8; ++k) {
        const int i = i0 + k * blockDim.x;
        if (i < m) { PXs[i] = x[k]; PYs[i] = y[k]; }
      }
    }
    const int32_t* gp = q.ranges + (size_t)n * q.T;
    for (int i = threadIdx.x; i < Tn; i += blockDim.x) prs[i] = gp[i];
  }
  __syncthreads();
  scan_trace(1);
  const int* pr = q.staged ? prs : q.ranges + (size_t)n * q.T;
  const float* PX = q.staged ? PXs : q.px2 + rb;
  const float* PY = q.staged ? PYs : q.py2 + rb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int spw = 32 / S;                       // segments per warp
  const int seg = warp * spw + lane / S, s = lane % S;
  const bool on = lane < spw * S;
  const int base = lane - s;
  const int nseg = 8 * spw;
  const int nc = (Tn - 1 + C - 1) / C;          // chunks over frames 1..Tn-1 (fwd) / Tn-2..0 (bwd)
  const float NB = kNegBig;
  const int sU = Un - pr[Tn - 1];               // slot of (T-1, U)

  // step i of chunk c: its frame (processing order), band shift and this lane's two arcs
  //   fwd: d = p_t - p_{t-1}, py = empty(t-1, s) (sent along the shift), px = y(t, s) (sent up the chain)
  //   bwd: d = p_{t+1} - p_t, py = empty(t, s), px = y(t, s) (both added on arrival)
  // (neutral values on inactive lanes keep every shuffle warp-uniform)
  auto load_step = [&](int c, int i, bool cact) {
    StepIn r;
    r.t = fwd ? 1 + c * C + i : Tn - 2 - c * C - i;
    r.act = cact && (fwd ? r.t < Tn : r.t >= 0);
    r.d = 0; r.py = NB; r.px = NB;
    if (r.act) {
      const int t = r.t;
      r.d = fwd ? pr[t] - pr[t - 1] : pr[t + 1] - pr[t];
      r.py = PY[(size_t)(fwd ? t - 1 : t) * S + s];
      r.px = PX[(size_t)t * S + s];
    }
    return r;
  };

  // ---------------- phase A: chunk transfer matrices
  const int rounds = (nc + nseg * G - 1) / (nseg * G);
  for (int rd = 0; rd < rounds; ++rd) {
    const int c = rank + G * (seg + rd * nseg);
    const bool cact = on && c < nc;
    float P[KR];
#pragma unroll
    for (int i = 0; i < KR; ++i) P[i] = (i == s) ? 0.f : NB;   // identity
    float shacc = 0.f;
    StepIn nx = load_step(c, 0, cact);
    for (int i = 0; i < C; ++i) {
      const StepIn in = nx;
      if (i + 1 < C) nx = load_step(c, i + 1, cact);   // next frame's arcs in flight during this step
      __syncwarp();        // reconverge after the lane-dependent loads: the shuffles below stay on the fast path
      const bool act = in.act;
      const int d = in.d;
      const float own_py = in.py, own_px = in.px;
      const float m = rebase_of(__shfl_sync(0xffffffffu, P[0], base));   // P[0][0]
      float X[KR];
      if (fwd) {
        const int src = (s + d < S) ? lane + d : lane;
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          if (SC == 0 && k >= S) break;
          const float v = __shfl_sync(0xffffffffu, P[k] + own_py, src);
          X[k] = (s + d < S) ? v - m : NB;
        }
#pragma unroll
        for (int j = 1; j < S; ++j) {
#pragma unroll
          for (int k = 0; k < KR; ++k) {
            if (SC == 0 && k >= S) break;
            const float v = __shfl_up_sync(0xffffffffu, X[k] + own_px, 1);
            if (s == j) X[k] = lae2(X[k], v);
          }
        }
      } else {
        const int src = (s - d >= 0) ? lane - d : lane;
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          if (SC == 0 && k >= S) break;
          const float v = __shfl_sync(0xffffffffu, P[k], src);
          X[k] = (s - d >= 0) ? v + own_py - m : NB;
        }
#pragma unroll
        for (int j = S - 2; j >= 0; --j) {
#pragma unroll
          for (int k = 0; k < KR; ++k) {
            if (SC == 0 && k >= S) break;
            const float v = __shfl_down_sync(0xffffffffu, X[k], 1);
            if (s == j) X[k] = lae2(X[k], v + own_px);
          }
        }
      }
      if (act) {
#pragma unroll
        for (int k = 0; k < KR; ++k) P[k] = X[k];
        shacc += m;
      }
    }
    if (cact) {
      float* dst = Pm + ((size_t)c * S + s) * S;
      if (G > 1) {
        const uint32_t da = tc::mapa(dst, 0);
#pragma unroll
        for (int k = 0; k < KR; ++k)
          if (k < S) tc::st_cluster_f32(da + 4 * k, P[k]);
        if (s == 0) tc::st_cluster_f32(tc::mapa(&psh[c], 0), shacc);
      } else {
#pragma unroll
        for (int k = 0; k < KR; ++k)
          if (k < S) dst[k] = P[k];
        if (s == 0) psh[c] = shacc;
      }
    }
  }
  if (G > 1) tc::cluster_sync();        // every chunk matrix is in rank 0's shared memory
  else __syncthreads();
  scan_trace(2);

  // ---------------- phase B: boundary vectors (rank 0)
  // a_0 (frame 0 / T-1) by warp 0; then either warp 0 chains a_{c+1} = M_c (x) a_c over the nc chunks, or
  // (q.prefix) the whole CTA forms the prefix products Q_c = M_c (x) ... (x) M_0 in log2(nc) Hillis-Steele
  // rounds (Q_c <- Q_c (x) Q_{c-d}, every entry a log-sum-exp over S terms) and a_{c+1} = Q_c (x) a_0 --
  // the chain was ~0.27 us per chunk (c5: 11 of the scan's 27 us).  The prefix entries are not rebased
  // (relative to the summed chunk shifts they stay within a few hundred log2 units); phase C rebases
  // every frame as before.
  if (rank == 0) {
    if (warp == 0) {
      const bool sa = lane < S;
      float a = NB;
      if (fwd) {
        // frame 0: alpha(0,0) = 0, then the vertical chain
        a = (s == 0) ? 0.f : NB;
        const float own_px = sa ? PX[s] : NB;
        for (int j = 1; j < S; ++j) {
          const float v = __shfl_up_sync(0xffffffffu, a + own_px, 1);
          if (lane == j) a = v;
        }
      } else {
        // frame T-1: the terminal blank at slot sU, then the chain downwards
        const size_t o = (size_t)(Tn - 1) * S + s;
        const float own_px = sa ? PX[o] : NB;
        a = (sa && s == sU) ? PY[o] : NB;
        for (int j = S - 2; j >= 0; --j) {
          const float v = __shfl_down_sync(0xffffffffu, a, 1);
          if (lane == j) a = lae2(a, v + own_px);
        }
      }
      double sh = 0.0;
      if (sa) bv[s] = a;
      if (lane == 0) bsh[0] = 0.0;
      if (!q.prefix) {
        const long long ck0 = clock64();
        for (int c = 0; c < nc; ++c) {
          // reconverge the warp every step: after the lane-predicated stores (and the divergent set-up
          // above) the warp otherwise stays split and every shuffle takes the diverged path (measured
          // 3519 -> 538 cycles per step at c4)
          __syncwarp();
          const float m = rebase_of(__shfl_sync(0xffffffffu, a, 0));
          const float* Pc = Pm + ((size_t)c * S + (sa ? s : 0)) * S;
          float mx = NB, x[KR];
#pragma unroll
          for (int k = 0; k < KR; ++k) {
            const float ak = __shfl_sync(0xffffffffu, a, k < S ? k : 0);
            x[k] = (k < S && sa) ? (ak - m) + Pc[k] : NB;
            mx = fmaxf(mx, x[k]);
          }
          float acc = 0.f;
#pragma unroll
          for (int k = 0; k < KR; ++k)
            if (k < S) acc += ex2_approx(x[k] - mx);
          a = mx + lg2_approx(acc);
          sh += (double)m + (double)psh[c];
          if (sa) bv[(c + 1) * S + s] = a;
          if (lane == 0) bsh[c + 1] = sh;
        }
        if (g_scan_trace && lane == 0) {
          g_scan_trace[((size_t)n * 2 + blockIdx.y) * 8 + 5] = (unsigned long long)(clock64() - ck0);
          g_scan_trace[((size_t)n * 2 + blockIdx.y) * 8 + 6] = (unsigned long long)nc;
        }
      }
    }
    if (q.prefix) {
      __syncthreads();                                   // a_0 in bv[0 .. S)
      float* Qa = Pm;
      float* Qb = reinterpret_cast<float*>(pfx_base);
      double* ha = reinterpret_cast<double*>(
          (reinterpret_cast<uintptr_t>(Qb + (size_t)q.ncmax * S * S) + 15) & ~uintptr_t(15));
      double* hb = ha + q.ncmax;
      const int SS = S * S, tid = threadIdx.x, nthr = blockDim.x;
      for (int c = tid; c < nc; c += nthr) ha[c] = (double)psh[c];
      __syncthreads();
      for (int dd = 1; dd < nc; dd <<= 1) {
        for (int e = tid; e < nc * SS; e += nthr) {
          const int c = e / SS, r = e - c * SS, sr = r / S, k = r - sr * S;
          if (c >= dd) {                                 // (Q_c (x) Q_{c-dd})[sr][k]
            const float* A = Qa + (size_t)c * SS + sr * S;
            const float* B = Qa + (size_t)(c - dd) * SS + k;
            float x[KR], mx = NB;
#pragma unroll
            for (int j = 0; j < KR; ++j) {
              if (SC == 0 && j >= S) break;
              x[j] = A[j] + B[j * S];
              mx = fmaxf(mx, x[j]);
            }
            float acc = 0.f;
#pragma unroll
            for (int j = 0; j < KR; ++j) {
              if (SC == 0 && j >= S) break;
              acc += ex2_approx(x[j] - mx);
            }
            Qb[e] = mx + lg2_approx(acc);
          } else {
            Qb[e] = Qa[e];
          }
        }
        for (int c = tid; c < nc; c += nthr) hb[c] = c >= dd ? ha[c] + ha[c - dd] : ha[c];
        __syncthreads();
        float* tq = Qa; Qa = Qb; Qb = tq;
        double* th = ha; ha = hb; hb = th;
      }
      for (int e = tid; e < nc * S; e += nthr) {         // a_{c+1} = Q_c (x) a_0
        const int c = e / S, sr = e - c * S;
        const float* Q = Qa + (size_t)c * SS + sr * S;
        float x[KR], mx = NB;
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          if (SC == 0 && k >= S) break;
          x[k] = Q[k] + bv[k];
          mx = fmaxf(mx, x[k]);
        }
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          if (SC == 0 && k >= S) break;
          acc += ex2_approx(x[k] - mx);
        }
        bv[(size_t)(c + 1) * S + sr] = mx + lg2_approx(acc);
        if (sr == 0) bsh[c + 1] = ha[c];
      }
    }
  }
  if (G > 1) tc::cluster_sync();        // the boundary vectors are visible to every rank
  else __syncthreads();
  scan_trace(3);

  // ---------------- phase C: every frame of every chunk from its boundary vector
  float* outp = (fwd ? q.ap : q.bp) + rb;
  double* Fs = (fwd ? q.Af : q.Bf) + (size_t)n * q.T;
  if (warp == 0 && lane < S && rank == 0) {       // the boundary frame 0 (fwd) / T-1 (bwd) itself
    const int t0 = fwd ? 0 : Tn - 1;
    outp[(size_t)t0 * S + s] = bv[s];
    if (s == 0) Fs[t0] = 0.0;
    if (fwd && Tn == 1 && s == sU) {
      const double L = ((double)bv[s] + (double)PY[(size_t)s]) * RNNT_LN2;   // alpha + empty(T-1,U)
      q.Lp[n] = L;
      q.loss[n] = (float)(-L);
      if (!isfinite(L) || L < -1e20) set_status(q.status, n, kStatusNonFinite);
    }
  }
  for (int rd = 0; rd < rounds; ++rd) {
    const int c = rank + G * (seg + rd * nseg);
    const bool cact = on && c < nc;
    float a = NB;
    double sh = 0.0;
    if (cact) {
      if (G > 1) {
        a = tc::ld_cluster_f32(tc::mapa(&bv[(size_t)c * S + s], 0));
        sh = tc::ld_cluster_f64(tc::mapa(&bsh[c], 0));
      } else {
        a = bv[(size_t)c * S + s];
        sh = bsh[c];
      }
    }
    StepIn nx = load_step(c, 0, cact);
    for (int i = 0; i < C; ++i) {
      const StepIn in = nx;
      if (i + 1 < C) nx = load_step(c, i + 1, cact);
      __syncwarp();                                     // converged shuffles (see phase A)
      const int t = in.t;
      const bool act = in.act;
      const int d = in.d;
      const float own_py = in.py, own_px = in.px;
      const float m = rebase_of(__shfl_sync(0xffffffffu, a, base));
      float x;
      if (fwd) {
        const float v = __shfl_sync(0xffffffffu, a + own_py, (s + d < S) ? lane + d : lane);
        x = (s + d < S) ? v - m : NB;
        for (int j = 1; j < S; ++j) {
          const float w = __shfl_up_sync(0xffffffffu, x + own_px, 1);
          if (s == j) x = lae2(x, w);
        }
      } else {
        const float v = __shfl_sync(0xffffffffu, a, (s - d >= 0) ? lane - d : lane);
        x = (s - d >= 0) ? v + own_py - m : NB;
        for (int j = S - 2; j >= 0; --j) {
          const float w = __shfl_down_sync(0xffffffffu, x, 1);
          if (s == j) x = lae2(x, w + own_px);
        }
      }
      if (act) {
        a = x;
        sh += (double)m;
        outp[(size_t)t * S + s] = a;
        if (s == 0) Fs[t] = sh;
        if (fwd && t == Tn - 1 && s == sU) {
          // L_pruned = alpha(T-1,U) + empty(T-1,U) (P:167-168 on the band)
          const double L = ((double)a + (double)PY[(size_t)t * S + s] + sh) * RNNT_LN2;
          q.Lp[n] = L;
          q.loss[n] = (float)(-L);
          if (!isfinite(L) || L < -1e20) set_status(q.status, n, kStatusNonFinite);
        }
      }
    }
  }
  if (G > 1) tc::cluster_sync();        // rank 0's shared memory stays alive until every rank has read it
  else __syncthreads();
  scan_trace(4);
}

// g_l = y'_p(t,u), g_b = empty'_p(t,u) for u = p_t + s (P:273-281 on the pruned lattice), and
// the per-(row, tile) softmax scale of the logit gradient sc = gs (g_b + g_l) exp(m_tile - lse).
__global__ void pruned_combine_kernel(const float* __restrict__ px2, const float* __restrict__ py2,
                                      const float* __restrict__ ap, const float* __restrict__ bp,
                                      const double* __restrict__ Af, const double* __restrict__ Bf,
                                      const double* __restrict__ Lp, const int32_t* __restrict__ ranges,
                                      const int32_t* __restrict__ rowinfo, const float* __restrict__ mt,
                                      const float* __restrict__ lse, const int64_t* __restrict__ bnd,
                                      int N, int T, int S, int ntile, float gs, float* __restrict__ gb,
                                      float* __restrict__ gl, float4* __restrict__ gpk,
                                      const int* __restrict__ tscale, uint16_t* __restrict__ Pt, int V, int VP) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long R = (long long)N * T * S;
  if (r >= R) return;
  const int s = (int)(r % S);
  const long long nt = r / S;
  const int t = (int)(nt % T), n = (int)(nt / T);
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  float yb = 0.f, bb = 0.f;
  const double L2 = Lp[n] * RNNT_LOG2E;
  const int info = rowinfo[r];
  if (info >= 0 && isfinite(L2)) {
    const int p = ranges[(size_t)n * T + t];
    const int u = p + s;
    const double At = Af[nt];
    const float a = ap[r];
    if (u < Un && s + 1 < S)    // label arc (t,u) -> (t,u+1): both ends in frame t
      yb = ex2_approx(a + px2[r] + bp[r + 1] + (float)(At + Bf[nt] - L2));
    if (t < Tn - 1) {            // blank arc (t,u) -> (t+1,u)
      const int s2 = u - ranges[(size_t)n * T + t + 1];
      if (s2 >= 0 && s2 < S) bb = ex2_approx(a + py2[r] + bp[r + S + (s2 - s)] + (float)(At + Bf[nt + 1] - L2));
    } else if (u == Un) {        // terminal blank
      bb = ex2_approx(a + py2[r] + (float)(At - L2));
    }
  }
  gb[r] = bb;
  gl[r] = yb;
  // packed per (V tile, row) operand scalars of the joiner backward (joiner_bwd.cu):
  // {gs (g_b + g_l) exp(m_tile - lse), gs g_b, gs g_l, label}; dead rows {0, 0, 0, -1}.  With one P~
  // offset per row (plain mode, D20) every tile's entry is tile 0's and only tile 0's is read (c4: 63
  // tiles x 160k rows of 16 B and an expf each were 220 us of this kernel)
  const float l = lse[r];
  const int ntw = *tscale == 0 ? 1 : ntile;
  for (int tl = 0; tl < ntw; ++tl) {
    float4 qv = make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
    if (info >= 0) qv = make_float4(gs * (bb + yb) * expf(mt[r * ntile + tl] - l), gs * bb, gs * yb, __int_as_float(info));
    gpk[(size_t)tl * R + r] = qv;
  }
  // One P~ offset per row (tscale == 0): the logit gradient is dz = sc P~' with the row scalar
  // sc = gs (g_b + g_l) e^{m_ref - lse} once the two picks are folded into P~ itself,
  //   P~'[r,0] = P~[r,0] - g_b / (g_b + g_l) e^{lse - m_ref},  P~'[r,y] = P~[r,y] - g_l / (...) e^{...},
  // so the joiner backward runs as plain GEMMs on P~' (K10: dh = sc (P~' W); K11: d_w = P~'^T (sc h)).
  if (*tscale == 0 && info >= 0) {
    const float occ = bb + yb;
    if (occ > 0.f) {
      const float e = expf(l - mt[r * ntile]);
      uint16_t* row = Pt + (size_t)r * VP;
      if (bb > 0.f) row[0] = f_to_bf16_bits_rn(bf16_bits_to_f(row[0]) - (bb / occ) * e);
      if (yb > 0.f && info < V) row[info] = f_to_bf16_bits_rn(bf16_bits_to_f(row[info]) - (yb / occ) * e);
    }
  }
}

__global__ void split_reduce_kernel(const float* __restrict__ part, int splits, long long M,
                                    float* __restrict__ out) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  float acc = 0.f;
  for (int z = 0; z < splits; ++z) acc += part[(size_t)z * M + i];
  out[i] = acc;
}
// float4 variant (M % 4 == 0): eight split loads in flight per thread, added in split order (the same
// order as the scalar kernel: bit-identical), instead of one dependent load per split
__global__ void split_reduce4_kernel(const float4* __restrict__ part, int splits, long long M4,
                                     float4* __restrict__ out) {
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
  out[i] = acc;
}

// ------------------------------------------------------------------ host drivers
cudaError_t prune_launch(const Dims& d, const float* enc, const float* dec, const int32_t* ranges,
                         const int64_t* bnd, uint16_t* h, cudaStream_t st) {
  const int J8 = d.J / 8;                          // J % 8 == 0 (rnnt_check_dims)
  const int fpb = std::max(1, 256 / J8);           // frames per block
  const long long NT = (long long)d.N * d.T;
  if (NT >= (1LL << 31)) return cudaErrorInvalidValue;   // (32-bit frame index in the kernel)
  RNNT_LAUNCH(KID_PRUNE, st, launch_pdl(prune_kernel, (unsigned)((NT + fpb - 1) / fpb), dim3(J8, fpb), 0, st, 
      enc, dec, ranges, bnd, d.N, d.T, d.U, d.J, d.S, h));
  return cudaGetLastError();
}

// Chunk length of the pruned scan: about sqrt(T) frames (phase B is T/C sequential steps, phase
// C is C), raised until the chunk matrices fit in shared memory.
static long long scan_mat_bytes(const Dims& d, int c) {
  const long long nc = (d.T + c - 1) / c + 1;
  return ((nc * d.S * d.S + nc + (nc + 1) * d.S) * 4 + 15) / 16 * 16 + (nc + 1) * 8;
}
// CTAs per (utterance, direction) of the scan: 4 for wide bands (phase A is bound by the MUFU work
// of S (S-1) LogAdds per lane and frame), else 2
static int scan_cluster(const Dims& d) { return d.S >= 8 ? 4 : 2; }
// Chunk length: the chain is A (C frames) + B (T/C steps, ~0.23 us each) + C (C frames, where a
// frame of A + C costs ~1 us at S = 5): C ~ sqrt(T / 5), raised until every chunk has a segment in
// one round over the cluster (nseg = 8 (32 / S) per CTA) and the matrices fit in shared memory.
static int scan_chunk(const Dims& d) {
  const int nseg = 8 * (32 / std::max(1, std::min(d.S, 32))) * scan_cluster(d);
  int C = 4;
  while ((long long)C * C * 5 < d.T) ++C;
  while ((d.T + C - 1) / C > nseg) ++C;
  while (scan_mat_bytes(d, C) > 32 * 1024) C *= 2;
  return C;
}
// chunk matrices + the staged arcs (2 T S floats) and bounds (T ints)
static long long scan_prefix_bytes(const Dims& d);
static bool scan_staged(const Dims& d) {
  return scan_mat_bytes(d, scan_chunk(d)) + (long long)d.T * d.S * 8 + (long long)d.T * 4 + scan_prefix_bytes(d) <=
         200 * 1024;
}
// phase B as a parallel prefix for narrow bands (c5 / c3: S = 5); wide bands keep the chain (the prefix's
// S^2 log-sum-exps per matrix and round outgrow it)
static bool scan_prefix(const Dims& d) { return d.S <= 8; }
static long long scan_prefix_bytes(const Dims& d) {
  const long long nc = (d.T + scan_chunk(d) - 1) / scan_chunk(d) + 1;
  return scan_prefix(d) ? 16 + nc * d.S * d.S * 4 + 16 + 2 * nc * 8 : 0;   // (16-B alignment of both parts)
}
size_t pruned_recursion_smem(const Dims& d) {
  const long long mat = scan_mat_bytes(d, scan_chunk(d));
  return (size_t)((scan_staged(d) ? mat + (long long)d.T * d.S * 8 + (long long)d.T * 4 : mat) + scan_prefix_bytes(d));
}

template <int SMAX, int SC>
static cudaError_t launch_scan(const Dims& d, const ScanParams& q, size_t sm, cudaStream_t st) {
  cudaFuncSetAttribute(pruned_scan_kernel<SMAX, SC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(d.N * q.G), 2);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)q.G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  RNNT_LAUNCH(KID_PALPHA, st, cudaLaunchKernelEx(&cfg, pruned_scan_kernel<SMAX, SC>, q));
  return cudaGetLastError();
}

// The plain joiner backward (no per-tile rescale of P~) needs the CTA-pair forward (one P~ offset per
// row) and the wide d_w kernel; RNNT_PLAIN=0 turns it off (A/B).
bool plain_backward_capable(const Dims& d) {
  static const int plain = env_int("RNNT_PLAIN", 1), pair = env_int("RNNT_FWD_PAIR", 1);
  return plain != 0 && pair != 0 && dw_wide(d);
}

cudaError_t rowinfo_launch(const Dims& d, const PrunedWS& w, const int32_t* ranges, const int64_t* sym,
                           const int64_t* bnd, const uint16_t* b, float gs, cudaStream_t st) {
  const long long R = d.rows();
  RNNT_LAUNCH(KID_ROWINFO, st, launch_pdl(rowinfo_kernel, (unsigned)((R + 255) / 256 + 1), 256, 0, st, 
      ranges, sym, bnd, d.N, d.T, d.U, d.V, d.S, w.rowinfo, w.urange, b, d.VP(), w.bias, w.bmax, w.tlive, w.tcounter,
      plain_backward_capable(d) ? 0 : 1, gs, w.dhlive));
  return cudaGetLastError();
}

// Forward: per-row info, K8 joiner with fused log-softmax, K9 recursion, the occupancies and the
// packed backward scalars.
cudaError_t pruned_fwd_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, const uint16_t* W,
                              const uint16_t* b, const int64_t* sym, const int32_t* ranges, const int64_t* bnd,
                              float gs, float* loss, int32_t* status, cudaStream_t st, bool do_rowinfo) {
  cudaError_t e;
  const long long R = d.rows();
  const int nt = d.ntile();
  if (do_rowinfo && (e = rowinfo_launch(d, w, ranges, sym, bnd, b, gs, st)) != cudaSuccess) return e;
  if ((e = joiner_fwd_launch(d, w, h, W, b, st)) != cudaSuccess) return e;
  {
    const size_t sm = pruned_recursion_smem(d);
    const int C = scan_chunk(d);
    ScanParams q{w.px2, w.py2, ranges, bnd, d.T, d.S, C, (d.T + C - 1) / C + 1, w.ap, w.bp, w.Af, w.Bf, w.Lp, loss,
                 status, scan_cluster(d), scan_staged(d) ? 1 : 0, scan_prefix(d) ? 1 : 0};
    switch (d.S) {   // band widths of the BASELINE configs (and the tests) get a compile-time S
      case 2: e = launch_scan<2, 2>(d, q, sm, st); break;
      case 3: e = launch_scan<3, 3>(d, q, sm, st); break;
      case 4: e = launch_scan<4, 4>(d, q, sm, st); break;
      case 5: e = launch_scan<5, 5>(d, q, sm, st); break;
      case 6: e = launch_scan<6, 6>(d, q, sm, st); break;
      case 8: e = launch_scan<8, 8>(d, q, sm, st); break;
      case 10: e = launch_scan<10, 10>(d, q, sm, st); break;
      default:
        e = d.S <= 8 ? launch_scan<8, 0>(d, q, sm, st)
                     : d.S <= 16 ? launch_scan<16, 0>(d, q, sm, st) : launch_scan<32, 0>(d, q, sm, st);
    }
    if (e != cudaSuccess) return e;
  }
  RNNT_LAUNCH(KID_PCOMBINE, st, launch_pdl(pruned_combine_kernel, (unsigned)((R + 255) / 256), 256, 0, st, 
      w.px2, w.py2, w.ap, w.bp, w.Af, w.Bf, w.Lp, ranges, w.rowinfo, w.mt, w.lse, bnd, d.N, d.T, d.S, nt, gs, w.gb,
      w.gl, w.gpk, w.tscale, w.Pt, d.V, d.VP()));
  return cudaGetLastError();
}

// Backward to the joiner input: K10 dh (and dpre), then d_enc / d_dec reductions.
// Backward to the joiner input: K10 dpre = (dz W) (1 - h^2) per band row (joiner_bwd.cu), then the
// band reductions
//   d_enc[n,t,:] = sum_{s: p_t + s <= U_n} dpre[(n,t,s),:]
//   d_dec[n,u,:] = sum_{t: p_t <= u < p_t + S} dpre[(n,t,u - p_t),:]      (frames [lo(u), hi(u)), Eq. 9)
// in two balanced passes (a band stuck at p = 0 or p = Umax covers one u with hundreds of frames, so a
// plain per-u gather is badly imbalanced):
//   A (block per chunk of kBandCH frames): the chunk's d_enc rows, and for every u its frames cover the
//     partial sum over the chunk's frames, stored at row p_{t0} + c S + (u - p_{t0}) of the utterance's
//     partial buffer (U + 1 + S ceil(T / CH) rows: chunk c's rows lie below chunk c+1's since p is
//     monotone);
//   B (a warp per (u, 128 columns)): d_dec[u] = the partials of the chunks covering u, in chunk order.
// Every output row is a fixed-order sum (deterministic).  The dpre rows are fp16 dpre / gs
// (joiner_dh_tc_kernel): the sums are taken in fp32 and scaled by gs when the outputs are written.
// Padded rows and infeasible utterances get 0.  (A single pass whose last-arriving chunk finishes each
// shared u measured slower: 68-77 vs 37 + 18 us at c5, the arrival fences and atomics sit on every
// warp's critical path.)
__device__ __forceinline__ float4 h4_to_f4(uint2 v) {
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&v.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&v.y));
  return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ float4 f4_scale(float4 a, float g) { return make_float4(a.x * g, a.y * g, a.z * g, a.w * g); }
__device__ __forceinline__ float gs_mult(const float* gsp) {   // the scale the fp16 rows were divided by
  const float g = *gsp;
  return (g != 0.f && isfinite(g)) ? g : 1.f;
}
// A: a warp per (chunk of kBandCH frames, utterance, 32-float4 column segment), lane = 4 columns: it
// walks the chunk's frames in order, loading the frame's S rows once (the next frames' rows are in
// flight meanwhile), adds them into d_enc[t] and into a window win[k] = partial of u = base + k (base
// = p_t; p is monotone, so a window entry is complete once p passes it: it is stored then and the
// window shifts).  SW >= S (compile time) bounds the window.
template <int SW>
__global__ void __launch_bounds__(256) band_chunk_kernel(const uint16_t* __restrict__ dpre,
                                                         const int32_t* __restrict__ ranges,
                                                         const int64_t* __restrict__ bnd, int N, int T, int U, int S,
                                                         int J, float* __restrict__ d_enc, float* __restrict__ part,
                                                         const float* __restrict__ gsp) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  const int J4 = J / 4, nseg = band_nseg(J);
  const int nch = (T + kBandCH - 1) / kBandCH;
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);   // < 2^31 (checked by the launcher)
  if (w >= N * nch * nseg) return;
  const int lane = threadIdx.x & 31;
  const int nc = w / nseg, seg = w - nc * nseg;
  const int n = nc / nch, c = nc - n * nch;
  const int q = seg * 32 + lane;
  const bool qok = q < J4;
  const int t0 = c * kBandCH, t1 = min(T, t0 + kBandCH);
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  const bool feas = (long long)Un <= (long long)Tn * (S - 1);
  const int te = feas ? min(t1, Tn) : t0;                  // live frames [t0, te)
  const int32_t* pr = ranges + (size_t)n * T;
  const uint2* D = reinterpret_cast<const uint2*>(dpre) + (size_t)n * T * S * J4;
  float4* E = reinterpret_cast<float4*>(d_enc) + (size_t)n * T * J4;
  float4* P = reinterpret_cast<float4*>(part) + ((size_t)n * band_part_rows(T, U, S) + (size_t)c * S) * J4;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  if (d_enc && qok)
    for (int t = max(t0, te); t < t1; ++t) E[(size_t)t * J4 + q] = z;          // padded / infeasible frames
  if (te <= t0) return;
  const float gm = gs_mult(gsp);
  float4 win[SW];
#pragma unroll
  for (int k = 0; k < SW; ++k) win[k] = z;
  int base = pr[t0];
  auto flush = [&]() {                                     // u = base is complete
    if (part && qok && base <= Un) P[(size_t)base * J4 + q] = win[0];
#pragma unroll
    for (int k = 0; k + 1 < SW; ++k) win[k] = win[k + 1];
    win[SW - 1] = z;
    ++base;
  };
  // FB frames per batch: all their rows' loads in flight together
  constexpr int FB = SW <= 5 ? 4 : (SW <= 10 ? 2 : 1);
  for (int tb = t0; tb < te; tb += FB) {
    uint2 x[FB][SW];                                       // raw fp16 x 4 (converted at use)
    int pf[FB];
#pragma unroll
    for (int f = 0; f < FB; ++f) {
      const int t = tb + f;
      pf[f] = t < te ? pr[t] : 0;
      const int ns = t < te ? min(S, Un - pf[f] + 1) : 0;
#pragma unroll
      for (int s = 0; s < SW; ++s) x[f][s] = (s < ns && qok) ? D[((size_t)t * S + s) * J4 + q] : make_uint2(0u, 0u);
    }
#pragma unroll
    for (int f = 0; f < FB; ++f) {
      const int t = tb + f;
      if (t >= te) break;
      while (base < pf[f]) flush();
      float4 e = z;
#pragma unroll
      for (int s = 0; s < SW; ++s) {
        const float4 xv = h4_to_f4(x[f][s]);
        e.x += xv.x; e.y += xv.y; e.z += xv.z; e.w += xv.w;
        win[s].x += xv.x; win[s].y += xv.y; win[s].z += xv.z; win[s].w += xv.w;
      }
      if (d_enc && qok) E[(size_t)t * J4 + q] = f4_scale(e, gm);
    }
  }
  const int ue = min(Un, pr[te - 1] + S - 1);
  while (base <= ue) flush();
}
// B: a warp per (utterance, u, 32-float4 column segment): the partials of the chunks covering u, in chunk
// order, eight chunks' loads in flight (a u under a band stuck for hundreds of frames spans tens of
// chunks: a chunk per round trip measured 24-36 us at c5); 32-bit index math (64-bit divisions were most of
// its issue slots).
__global__ void __launch_bounds__(256) band_dec_kernel(const float* __restrict__ part, const int2* __restrict__ urange,
                                                       const int64_t* __restrict__ bnd, int N, int T, int U, int S,
                                                       int J, float* __restrict__ d_dec, const float* __restrict__ gsp) {
  RNNT_GDC();   // programmatic dependent launch: wait for the producer grid, release ours
  const int J4 = J / 4, nseg = band_nseg(J);
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);   // < 2^31 (checked by the launcher)
  const int lane = threadIdx.x & 31;
  if (w >= N * (U + 1) * nseg) return;
  const int nu = w / nseg;
  const int q = (w - nu * nseg) * 32 + lane;
  const int n = nu / (U + 1), u = nu - n * (U + 1);
  const int2 cv = urange[nu];                              // (issued with the length loads: one round trip)
  const float gm = gs_mult(gsp);
  const int Tn = utt_T(bnd, n), Un = utt_U(bnd, n);
  const bool feas = (long long)Un <= (long long)Tn * (S - 1);
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
  if (feas && u <= Un) {                                   // frames [lo, hi) cover u
    const int c0 = cv.x / kBandCH, c1 = (cv.y - 1) / kBandCH;
    const float4* P = reinterpret_cast<const float4*>(part) + ((size_t)n * band_part_rows(T, U, S) + u) * J4 + q;
    const int cstride = S * J4;
    for (int cb = c0; cb <= c1; cb += 8) {
      float4 x[8];
#pragma unroll
      for (int m = 0; m < 8; ++m)
        x[m] = (cb + m <= c1 && q < J4) ? P[(cb + m) * cstride] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int m = 0; m < 8; ++m) { a.x += x[m].x; a.y += x[m].y; a.z += x[m].z; a.w += x[m].w; }
    }
    a = f4_scale(a, gm);
  }
  if (q < J4) reinterpret_cast<float4*>(d_dec + (size_t)nu * J)[q] = a;
}

cudaError_t pruned_bwd_input_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, const uint16_t* W,
                                    const int32_t* ranges, const int64_t* bnd, float* d_enc, float* d_dec,
                                    cudaStream_t st) {
  cudaError_t e;
  GradSrc g{w.Pt, w.gpk, w.rowinfo, d.rows(), d.V, d.VP(), d.ntile()};
  if (!d_enc && !d_dec) return cudaSuccess;
  const long long ntiles = (d.rows() + 127) / 128;   // (the live-tile list: built by the forward)
  if ((e = joiner_dh_launch(d, g, h, W, w.dhlive, w.dhlive + ntiles, ntiles, w.dpre, w.tscale, w.gsp, st)) !=
      cudaSuccess)
    return e;
  {
    const long long nwarp = (long long)d.N * ((d.T + kBandCH - 1) / kBandCH) * band_nseg(d.J);
    if (nwarp >= (1LL << 31) || (long long)d.N * d.U1() * band_nseg(d.J) >= (1LL << 31)) return cudaErrorInvalidValue;
    const unsigned nb = (unsigned)((nwarp + 7) / 8);
    float* pp = d_dec ? w.bpart : nullptr;
#define RNNT_BAND(SWV) launch_pdl(band_chunk_kernel<SWV>, nb, 256, 0, st, reinterpret_cast<const uint16_t*>(w.dpre), \
                                  ranges, bnd, d.N, d.T, d.U, d.S, d.J, d_enc, pp, w.gsp)
    switch (d.S) {   // the window is exactly S wide for the common band widths
      case 1: RNNT_LAUNCH(KID_DENC, st, RNNT_BAND(1)); break;
      case 2: RNNT_LAUNCH(KID_DENC, st, RNNT_BAND(2)); break;
      case 3: RNNT_LAUNCH(KID_DENC, st, RNNT_BAND(3)); break;
      case 4: RNNT_LAUNCH(KID_DENC, st, RNNT_BAND(4)); break;
      case 5: RNNT_LAUNCH(KID_DENC, st, RNNT_BAND(5)); break;
      case 6: RNNT_LAUNCH(KID_DENC, st, RNNT_BAND(6)); break;
      case 7: case 8: RNNT_LAUNCH(KID_DENC, st, RNNT_BAND(8)); break;
      case 9: case 10: RNNT_LAUNCH(KID_DENC, st, RNNT_BAND(10)); break;
      default:
        if (d.S <= 16) RNNT_LAUNCH(KID_DENC, st, RNNT_BAND(16));
        else RNNT_LAUNCH(KID_DENC, st, RNNT_BAND(32));
    }
#undef RNNT_BAND
  }
  if (d_dec) {
    const long long nw = (long long)d.N * d.U1() * band_nseg(d.J);
    RNNT_LAUNCH(KID_DDEC, st, launch_pdl(band_dec_kernel, (unsigned)((nw + 7) / 8), 256, 0, st,
                                         w.bpart, w.urange, bnd, d.N, d.T, d.U, d.S, d.J, d_dec, w.gsp));
  }
  return cudaGetLastError();
}

cudaError_t split_reduce_acc_launch(const float* part, int splits, long long M, float* out, int mode, int kid,
                                    cudaStream_t st);

// Backward to the joiner weights: K11 dW (split-K) + db, deterministic split reduction.  mode > 0: the
// reduced d_w / d_b are ADDED into the targets (exchange.cu: red.global.add, or multimem.red.add on an
// NVLS multicast address).
cudaError_t pruned_bwd_weight_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, float* d_w, float* d_b,
                                     cudaStream_t st, int mode) {
  cudaError_t e;
  GradSrc g{w.Pt, w.gpk, w.rowinfo, d.rows(), d.V, d.VP(), d.ntile()};
  const long long ntiles = (d.rows() + 127) / 128;
  const int* ts = w.plain ? w.tscale : nullptr;   // (the full loss: always the rescaling path)
  if (ts && w.Hs && (e = scale_rows_launch(d, g, h, ts, w.dhlive, w.dhlive + ntiles, ntiles, w.Hs, st)) != cudaSuccess)
    return e;
  if ((e = joiner_dw_launch(d, g, h, w.Hs, ts, w.dhlive, w.dhlive + ntiles, w.dWp, w.dbp, w.splits, st)) !=
      cudaSuccess)
    return e;
  if (mode != 0) {
    if ((e = split_reduce_acc_launch(w.dWp, w.splits, (long long)d.V * d.J, d_w, mode, KID_DW_REDUCE, st)) !=
        cudaSuccess)
      return e;
    return split_reduce_acc_launch(w.dbp, w.splits, d.V, d_b, mode, KID_DB_REDUCE, st);
  }
  const long long M = (long long)d.V * d.J;
  if (M % 4 == 0 && reinterpret_cast<uintptr_t>(d_w) % 16 == 0)
    RNNT_LAUNCH(KID_DW_REDUCE, st, launch_pdl(split_reduce4_kernel, (unsigned)((M / 4 + 255) / 256), 256, 0, st, 
        reinterpret_cast<const float4*>(w.dWp), w.splits, M / 4, reinterpret_cast<float4*>(d_w)));
  else
    RNNT_LAUNCH(KID_DW_REDUCE, st, launch_pdl(split_reduce_kernel, (unsigned)((M + 255) / 256), 256, 0, st, w.dWp, w.splits, M, d_w));
  RNNT_LAUNCH(KID_DB_REDUCE, st, launch_pdl(split_reduce_kernel, (unsigned)((d.V + 255) / 256), 256, 0, st, w.dbp, w.splits, d.V, d_b));
  return cudaGetLastError();
}

cudaError_t pruned_loss_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, const uint16_t* W,
                               const uint16_t* b, const int64_t* sym, const int32_t* ranges,
                               const int64_t* bnd, float gs, float* loss, float* d_enc, float* d_dec,
                               float* d_w, float* d_b, int32_t* status, cudaStream_t st) {
  cudaError_t e;
  if ((e = pruned_fwd_launch(d, w, h, W, b, sym, ranges, bnd, gs, loss, status, st, true)) != cudaSuccess) return e;
  if ((e = pruned_bwd_input_launch(d, w, h, W, ranges, bnd, d_enc, d_dec, st)) != cudaSuccess) return e;
  return pruned_bwd_weight_launch(d, w, h, d_w, d_b, st, 0);
}

}  // namespace rnnt
