/*
 * rnnt.h — C-ABI of the B200 pruned RNN-T loss hot path (arXiv 2206.13236).
 *
 * Citations: P:<n> = line n of the paper source;
 * D<k> = the reading of the paper recorded in DESIGN.md "Readings".
 *
 * The four entry points follow the paper's statement of the problem
 * ("computing the core recursion ... twice"):
 *   rnnt_simple_loss  : trivial joiner (Eq. 5-6) + recursion (Eq. 3)
 *                       + occupancies y', empty' + am/lm gradients
 *   rnnt_get_ranges   : locally optimal bounds (Eq. 8) + consistency
 *                       adjustment (Eq. 9-10; algorithm D3)
 *   rnnt_prune        : gather of the joiner input at the T*S band pairs
 *   rnnt_pruned_loss  : full joiner W_out*tanh(.)+b on the band, log-softmax, pick and
 *                       logit gradient fused (function merging), pruned
 *                       recursion, all gradients.
 *
 * Conventions (all entry points):
 *  - Every pointer is a DEVICE pointer unless stated; the caller owns every buffer.
 *    The library never allocates device memory: scratch comes from `workspace`
 *    (size from rnnt_workspace_bytes).  No global mutable state: calls on distinct
 *    streams with distinct workspaces may run concurrently.
 *  - Every call only ENQUEUES work on `stream` (a cudaStream_t passed as void*;
 *    NULL = legacy default stream) and never synchronises the host.
 *  - Layouts are dense row-major with the padded batch maxima of rnnt_dims_t:
 *    T = max_n T_n, U = max_n U_n.  Values at padded positions of inputs are never
 *    read; all outputs at padded positions are written as exactly 0 (ranges: Umax_n).
 *  - boundary is int64 (N,4) {0, 0, U_n, T_n} (begin_symbol, begin_frame,
 *    end_symbol, end_frame); nonzero begins are not supported (RNNT_ERR_UNSUPPORTED
 *    cannot be detected without a sync, so they are reported in status bit 4).
 *  - symbols is int64 (N,U): y_1..y_{U_n} in [1,V) (D1); blank id is 0.
 *  - bf16 tensors are passed as uint16_t bit patterns.
 *  - Synchronous errors (returned): null pointer, dims out of range, misaligned
 *    pointer (16 B), workspace too small, CUDA launch failure.  Nothing is launched
 *    when an argument error is returned.
 *  - Data-dependent errors go to the optional device `status` (N) int32 bitmask:
 *      bit0  infeasible band: U_n > T_n (S-1) (no band-respecting path; D3)
 *      bit1  non-finite loss
 *      bit2  symbol outside [1,V)
 *      bit3  normaliser underflow (sum_v exp(...) == 0 after offsets; D7)
 *      bit4  nonzero begin_symbol / begin_frame in boundary
 *    status is OR-ed into (callers zero it once per step).
 *  - Gradients are grad_scale * d(sum_n loss_n)/dx, overwritten (not accumulated).
 *    Pass 0.5 for the simple loss and 1.0 for the pruned loss.
 */
#ifndef RNNT_B200_H
#define RNNT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RNNT_OK = 0,
  RNNT_ERR_INVALID_ARG = 1,
  RNNT_ERR_UNSUPPORTED = 2,
  RNNT_ERR_WORKSPACE = 3,
  RNNT_ERR_CUDA = 4
} rnnt_status_t;

/* Padded problem sizes. T, U are the batch maxima; V includes the blank id 0;
 * J is the joiner hidden size; S the band width (s_range).
 * Limits: 1 <= N, 1 <= T <= 65536, 0 <= U <= 1023 and U < T*64, 2 <= V, 8 <= J <= 4096 and
 * J % 8 == 0, 1 <= S <= 32.  U <= 1023 because the simple-lattice wavefront holds a row of U+1
 * cells in at most 4 warps x 32 lanes x 8 registers.  Long utterances are supported: the pruned
 * recursion stages an utterance's band arcs in shared memory when they fit and reads them from L2
 * otherwise.  Outside these limits the calls return RNNT_ERR_UNSUPPORTED (or RNNT_ERR_INVALID_ARG for
 * the argument ranges) and launch nothing. */
typedef struct {
  int32_t N, T, U, V, J, S;
} rnnt_dims_t;

/* Bytes of device scratch needed by rnnt_simple_loss and rnnt_pruned_loss for these
 * dims (one workspace may be reused by consecutive calls on the same stream). */
size_t rnnt_workspace_bytes(const rnnt_dims_t* dims);

/* Human-readable name of a status code (static string, never NULL). */
const char* rnnt_status_string(rnnt_status_t s);

/* Library build string: kernels compiled and the sm target. */
const char* rnnt_version(void);

/* The CUDA error string behind the last RNNT_ERR_CUDA returned to the calling host thread
 * (static string, never NULL; "no error" before any). */
const char* rnnt_last_cuda_error(void);

/* ---- Diagnostics (bench.py; not needed for computing the loss) ----
 * rnnt_launch_count: number of kernels the library has launched from the calling host
 *   thread (monotone counter).
 * rnnt_kernel_count / rnnt_kernel_name: ids 1..count-1 of the library's kernel launch sites.
 * rnnt_profile_kernel: from the calling thread on, every launch of kernel `kernel_id` is
 *   bracketed by cudaEventRecord(start_event) / cudaEventRecord(stop_event) on the launch
 *   stream (events are cudaEvent_t passed as void*, owned by the caller); id 0 disarms.
 *   Returns RNNT_ERR_INVALID_ARG for an unknown id. */
uint64_t rnnt_launch_count(void);
/* rnnt_pruned_backward_mode: after rnnt_pruned_loss_forward was enqueued on `stream` with this
 *   workspace, synchronises the stream and writes to *plain 1 if the forward stored every row's P~
 *   with one offset (the joiner backward then runs as plain GEMMs on P~ with the picks folded in), 0 if
 *   some row needed per-tile offsets (a logit more than 60 above the row's reference; the backward then
 *   rescales P~ per (row, tile) in shared memory), D20. */
rnnt_status_t rnnt_pruned_backward_mode(const rnnt_dims_t* dims, const void* workspace, size_t workspace_bytes,
                                        int32_t* plain, void* stream);
int32_t rnnt_kernel_count(void);
const char* rnnt_kernel_name(int32_t id);
rnnt_status_t rnnt_profile_kernel(int32_t kernel_id, void* start_event, void* stop_event);

/*
 * Trivial-joiner loss, occupancies and gradients.
 *   am  (N,T,V) fp32   L_enc(t,v)
 *   lm  (N,U+1,V) fp32 L_dec(u,v)
 *   L_norm(t,u) = log sum_v exp(am[t,v]+lm[u,v]) is evaluated as a max-shifted
 *   contraction (Eq. 6, "after first applying offsets") without
 *   materialising (T,U+1,V).
 * Outputs:
 *   loss    (N) fp32      -L_tot,n  (L_tot = alpha(T-1,U)+empty(T-1,U))
 *   px_grad (N,T,U+1) fp32  y'(t,u)     = dL_tot/dy(t,u)      (unscaled, in [0,1])
 *   py_grad (N,T,U+1) fp32  empty'(t,u) = dL_tot/dempty(t,u)  (unscaled, in [0,1])
 *   am_grad (N,T,V) fp32, lm_grad (N,U+1,V) fp32 : grad_scale * d(sum loss)/d(am|lm);
 *           either may be NULL to skip it.
 *   status  (N) int32, nullable.
 */
rnnt_status_t rnnt_simple_loss(const float* am, const float* lm, const int64_t* symbols,
                               const int64_t* boundary, const rnnt_dims_t* dims, float grad_scale,
                               float* loss, float* px_grad, float* py_grad, float* am_grad,
                               float* lm_grad, int32_t* status, void* workspace,
                               size_t workspace_bytes, void* stream);

/*
 * The am/lm gradients of rnnt_simple_loss as a separate call, so that a caller can run them on a
 * second stream concurrently with rnnt_get_ranges / rnnt_prune / rnnt_pruned_loss (they depend on
 * nothing downstream).  Precondition: rnnt_simple_loss was enqueued earlier, in stream order, with
 * the same dims and workspace (it leaves the normaliser operands and G~ = (y'+empty')/S in the
 * simple-loss region of the workspace, which rnnt_pruned_loss never touches), and px_grad /
 * py_grad are its outputs.  rnnt_simple_loss(..., am_grad = lm_grad = NULL, ...) followed by this
 * call computes exactly what rnnt_simple_loss with both gradient pointers computes.
 *   am_grad (N,T,V), lm_grad (N,U+1,V) fp32: grad_scale * d(sum loss)/d(am|lm); one may be NULL.
 */
rnnt_status_t rnnt_simple_loss_backward(const float* am, const float* lm, const float* px_grad,
                                        const float* py_grad, const int64_t* symbols,
                                        const int64_t* boundary, const rnnt_dims_t* dims,
                                        float grad_scale, float* am_grad, float* lm_grad,
                                        void* workspace, size_t workspace_bytes, void* stream);

/*
 * Smoothed trivial joiner (Eq. 11-15): rnnt_simple_loss on the lattice of
 *   L_smoothed(t,u,v) = (1 - a_lm - a_ac) L_trivial(t,u,v) + a_lm L_lm(u,v) + a_ac L_acoustic(t,v)
 * with L_trivial = LogSoftmax_v(am[t,v] + lm[u,v]) (Eq. 12), L_lm = LogSoftmax_v lm[u,v] (Eq. 14),
 * L_acoustic = LogSoftmax_v(am[t,v] + L_dec^avg(v)) (Eq. 13) and the per-utterance unigram prior
 * L_dec^avg(v) = log (1/(U_n+1)) sum_{u<=U_n} Softmax_v lm[u,v] (Eq. 15).  Eq. 11 as printed repeats
 * L_lm in its third term; it is read as L_acoustic (D18).
 *   lm_only_scale = a_lm, am_only_scale = a_ac (finite; 0, 0 gives exactly rnnt_simple_loss).
 * Every other argument, output and convention is that of rnnt_simple_loss /
 * rnnt_simple_loss_backward; am_grad / lm_grad include the derivatives through all three terms
 * (the L_dec^avg prior couples lm to every frame).  The backward needs the workspace of the
 * forward call with the same scales.
 */
rnnt_status_t rnnt_simple_loss_smoothed(const float* am, const float* lm, const int64_t* symbols,
                                        const int64_t* boundary, const rnnt_dims_t* dims,
                                        float lm_only_scale, float am_only_scale, float grad_scale,
                                        float* loss, float* px_grad, float* py_grad, float* am_grad,
                                        float* lm_grad, int32_t* status, void* workspace,
                                        size_t workspace_bytes, void* stream);
rnnt_status_t rnnt_simple_loss_smoothed_backward(const float* am, const float* lm, const float* px_grad,
                                                 const float* py_grad, const int64_t* symbols,
                                                 const int64_t* boundary, const rnnt_dims_t* dims,
                                                 float lm_only_scale, float am_only_scale,
                                                 float grad_scale, float* am_grad, float* lm_grad,
                                                 void* workspace, size_t workspace_bytes, void* stream);

/*
 * Pruning bounds.  For every frame t < T_n:
 *   raw_t = argmax_{p=0..max(0,U_n-S+1)} ( -y'(t,p-1) + sum_{u=p}^{p+S-1} empty'(t,u) )  (Eq. 8)
 * evaluated in fp64 from the fp32 inputs in a fixed order (u ascending, then the
 * subtraction; D5) with ties to the smallest p — bit-exact w.r.t. the oracle on
 * identical inputs.  Then the ADJ-scan adjustment (D3) enforces Eq. 9-10 plus
 * p_0 = 0, p_{T_n-1} = Umax_n.  ranges (N,T) int32; padded frames get Umax_n;
 * infeasible utterances (status bit0) get all-zero ranges.
 * Uses dims N, T, U, S (V, J ignored).  No workspace.
 */
rnnt_status_t rnnt_get_ranges(const float* px_grad, const float* py_grad, const int64_t* boundary,
                              const rnnt_dims_t* dims, int32_t* ranges, int32_t* status,
                              void* stream);

/*
 * Joiner input on the band (joiner form D13):
 *   h[n,t,s,:] = bf16_rn( tanh(enc_proj[n,t,:] + dec_proj[n,p_t+s,:]) )
 * for t < T_n and p_t+s <= U_n; every other row (masked slot or padded frame) is 0.
 *   enc_proj (N,T,J) fp32, dec_proj (N,U+1,J) fp32, ranges (N,T) int32,
 *   h (N,T,S,J) bf16 (uint16 bits).
 */
rnnt_status_t rnnt_prune(const float* enc_proj, const float* dec_proj, const int32_t* ranges,
                         const int64_t* boundary, const rnnt_dims_t* dims, uint16_t* h,
                         void* stream);

/*
 * Pruned loss and gradients.
 *   z[n,t,s,:] = W_out h[n,t,s,:] + b_out  (V), L(t,p_t+s,.) = log_softmax(z)
 *   empty_p(t,u) = L(t,u,0), y_p(t,u) = L(t,u,y_{u+1}) (-inf at u=U_n), -inf off-band;
 *   Eq. 3 recursion over the band -> loss (N) = -L_pruned,n (+inf if infeasible).
 * Gradients (function merging): dz = gs((g_b+g_l) softmax(z) - g_b[v=0] - g_l[v=y]),
 *   d_w (V,J) fp32 = sum dz h^T,  d_b (V) fp32 = sum dz  (overwritten, this batch only),
 *   d_enc (N,T,J) fp32 = sum_s dpre, d_dec (N,U+1,J) fp32 = sum over band rows of dpre,
 *   dpre = (W^T dz) * (1 - h^2).  d_enc / d_dec may be NULL.
 *   w_out (V,J) bf16, b_out (V) bf16.
 */
rnnt_status_t rnnt_pruned_loss(const uint16_t* h, const uint16_t* w_out, const uint16_t* b_out,
                               const int64_t* symbols, const int32_t* ranges,
                               const int64_t* boundary, const rnnt_dims_t* dims, float grad_scale,
                               float* loss, float* d_enc, float* d_dec, float* d_w, float* d_b,
                               int32_t* status, void* workspace, size_t workspace_bytes,
                               void* stream);

/*
 * rnnt_pruned_loss as three calls (forward, backward to the joiner input, backward to the joiner
 * weights), so that the two backward halves — which only read what the forward left in the
 * pruned-loss region of the workspace and write disjoint outputs — can run on two streams.
 * In stream order: forward, then backward_input and backward_weight (in either order or
 * concurrently); together they compute exactly what rnnt_pruned_loss computes.
 *   rnnt_pruned_loss_forward:          loss (N), status; leaves P~, the tile maxima and the
 *                                      occupancies (times grad_scale) in the workspace.
 *   rnnt_pruned_loss_backward_input:   d_enc (N,T,J) and/or d_dec (N,U+1,J) (one may be NULL).
 *   rnnt_pruned_loss_backward_weight:  d_w (V,J), d_b (V).
 */
rnnt_status_t rnnt_pruned_loss_forward(const uint16_t* h, const uint16_t* w_out, const uint16_t* b_out,
                                       const int64_t* symbols, const int32_t* ranges,
                                       const int64_t* boundary, const rnnt_dims_t* dims,
                                       float grad_scale, float* loss, int32_t* status, void* workspace,
                                       size_t workspace_bytes, void* stream);
/*
 * rnnt_pruned_loss_forward split in two so that its first step can overlap the gather (rnnt_prune): it
 * does not read h.  rnnt_pruned_loss_prepare (ranges, symbols, boundary, b_out, grad_scale -> per band row
 * label info, the frames covering each token position, the fp32 bias and its tile maxima, the live
 * 128-row tiles, the loss scale; all in the workspace) followed in stream order by
 * rnnt_pruned_loss_forward_prepared (the same arguments as rnnt_pruned_loss_forward; grad_scale must be
 * the prepare call's) computes exactly what rnnt_pruned_loss_forward computes.
 * Same argument rules and errors as rnnt_pruned_loss_forward; the workspace is the pruned region.
 */
rnnt_status_t rnnt_pruned_loss_prepare(const int32_t* ranges, const int64_t* symbols, const int64_t* boundary,
                                       const rnnt_dims_t* dims, const uint16_t* b_out, float grad_scale,
                                       void* workspace, size_t workspace_bytes, void* stream);
rnnt_status_t rnnt_pruned_loss_forward_prepared(const uint16_t* h, const uint16_t* w_out, const uint16_t* b_out,
                                                const int64_t* symbols, const int32_t* ranges,
                                                const int64_t* boundary, const rnnt_dims_t* dims, float grad_scale,
                                                float* loss, int32_t* status, void* workspace,
                                                size_t workspace_bytes, void* stream);
rnnt_status_t rnnt_pruned_loss_backward_input(const uint16_t* h, const uint16_t* w_out,
                                              const int32_t* ranges, const int64_t* boundary,
                                              const rnnt_dims_t* dims, float* d_enc, float* d_dec,
                                              void* workspace, size_t workspace_bytes, void* stream);
rnnt_status_t rnnt_pruned_loss_backward_weight(const uint16_t* h, const rnnt_dims_t* dims, float* d_w,
                                               float* d_b, void* workspace, size_t workspace_bytes,
                                               void* stream);

/*
 * Data-parallel exchange.  The only cross-GPU reduction of a step is the sum of
 * d_w, d_b and the two batch losses over ranks.  A caller keeps them in one flat fp32 buffer
 *   acc = [ d_w (V*J) | d_b (V) | loss sums (2) ]
 * and chooses how each contribution reaches it:
 *   RNNT_EXCHANGE_STORE     plain stores (this rank's values; an all_reduce, e.g. NCCL, follows);
 *   RNNT_EXCHANGE_RED       red.global.add into a device buffer the caller zeroed (several shards of
 *                           one batch, or several launches, summed in place; fp32 addition order is
 *                           not fixed, so results agree to rounding, not bit for bit);
 *   RNNT_EXCHANGE_MULTIMEM  multimem.red.add on an NVLink-SHARP (NVLS) multicast address of a
 *                           symmetric buffer: every rank's copy receives the sum over ranks inside the
 *                           NVSwitch.  The pointers must be multicast addresses (e.g. torch symmetric
 *                           memory's multicast_ptr); the caller zeroes the buffer before the first add
 *                           and barriers across ranks before reading it.
 */
typedef enum {
  RNNT_EXCHANGE_STORE = 0,
  RNNT_EXCHANGE_RED = 1,
  RNNT_EXCHANGE_MULTIMEM = 2
} rnnt_exchange_mode_t;

/* rnnt_pruned_loss_backward_weight with the reduced d_w (V,J) / d_b (V) delivered by `mode`
 * (STORE: identical to rnnt_pruned_loss_backward_weight).  Same preconditions. */
rnnt_status_t rnnt_pruned_loss_backward_weight_exchange(const uint16_t* h, const rnnt_dims_t* dims,
                                                        int32_t mode, float* d_w, float* d_b,
                                                        void* workspace, size_t workspace_bytes,
                                                        void* stream);

/* Fixed-order sum of `nparts` contiguous fp32 vectors of length M (parts[k*M + i], k ascending),
 * delivered into out[0..M) by `mode`: e.g. the exchange buffers of several sub-batches of one step
 * (deterministic for any nparts), or a rank's partials before a multimem exchange. */
rnnt_status_t rnnt_exchange_sum(const float* parts, int32_t nparts, int64_t M, int32_t mode, float* out,
                                void* stream);

/* Batch loss combination (D12, D16):
 *   out[0] = simple_scale * sum_n loss_simple[n],
 *   out[1] = pruned_scale * sum_n loss_pruned[n] over the utterances whose status bit0 (infeasible)
 *            is clear — an infeasible utterance's +inf stays visible in loss_pruned[n] but does not
 *            poison the sum (status may be NULL: nothing masked).
 * fp64 accumulation in a fixed order; delivered by `mode` as above.  N >= 1. */
rnnt_status_t rnnt_loss_sums(const float* loss_simple, const float* loss_pruned, const int32_t* status,
                             int32_t N, float simple_scale, float pruned_scale, int32_t mode,
                             float* out, void* stream);

/*
 * Full (unpruned) transducer loss with the same non-linear joiner (the comparison
 * class of P:44-52, P:171-176 and Tables 1-2): the band widened to every token position
 * (S = U_n + 1, all bounds 0), so the joiner runs on all (N, T, U+1) lattice nodes:
 *   h = bf16(tanh(enc_proj[t] + dec_proj[u])), z = W_out h + b, L = log_softmax(z) (D13),
 *   loss[n] = -log P(y | x) of the full lattice (Eq. 3 with the joiner's arcs),
 *   d_enc / d_dec / d_w / d_b = grad_scale * d(sum loss)/d(.) (d_enc, d_dec nullable).
 * dims.S is ignored.  Memory grows as N T (U+1) (J + V) — the cost the pruned loss avoids; size the
 * workspace with rnnt_full_workspace_bytes.  Same conventions as rnnt_pruned_loss otherwise.
 */
size_t rnnt_full_workspace_bytes(const rnnt_dims_t* dims);
rnnt_status_t rnnt_full_loss(const float* enc_proj, const float* dec_proj, const uint16_t* w_out,
                             const uint16_t* b_out, const int64_t* symbols, const int64_t* boundary,
                             const rnnt_dims_t* dims, float grad_scale, float* loss, float* d_enc,
                             float* d_dec, float* d_w, float* d_b, int32_t* status, void* workspace,
                             size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RNNT_B200_H */
