// api.cu — the C-ABI entry points of include/rnnt.h: argument validation, workspace
// carving and launch sequencing.  Every call only enqueues on the caller's stream.
#include <cuda_runtime.h>
#include <stdint.h>

#include <nvtx3/nvToolsExt.h>

#include "../../include/rnnt.h"
#include "launch.h"
#include "workspace.h"

// NVTX range around every C-ABI call (the enqueue, not the kernels: those are async), so a profiler's
// timeline groups the launches by stage (SURVEY 5 "Profiling").  NVTX3 is header-only; without an
// attached tool each call is one predicted branch.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

namespace rnnt {
cudaError_t simple_loss_launch(const Dims& d, const SimpleWS& w, const float* am, const float* lm,
                               const int64_t* sym, const int64_t* bnd, float gs, float* loss,
                               float* px_grad, float* py_grad, float* am_grad, float* lm_grad,
                               int32_t* status, Smooth sm, cudaStream_t st);
cudaError_t get_ranges_launch(const Dims& d, const float* px_grad, const float* py_grad, const int64_t* bnd,
                              int32_t* ranges, int32_t* status, cudaStream_t st);
cudaError_t prune_launch(const Dims& d, const float* enc, const float* dec, const int32_t* ranges,
                         const int64_t* bnd, uint16_t* h, cudaStream_t st);
cudaError_t simple_grads_launch(const Dims& d, const SimpleWS& w, const float* am, const float* lm,
                                const float* px_grad, const float* py_grad, const int64_t* sym, const int64_t* bnd,
                                float gs, float* am_grad, float* lm_grad, Smooth sm, cudaStream_t st);
size_t pruned_recursion_smem(const Dims& d);
cudaError_t rowinfo_launch(const Dims& d, const PrunedWS& w, const int32_t* ranges, const int64_t* sym,
                           const int64_t* bnd, const uint16_t* b, float gs, cudaStream_t st);
cudaError_t pruned_fwd_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, const uint16_t* W,
                              const uint16_t* b, const int64_t* sym, const int32_t* ranges, const int64_t* bnd,
                              float gs, float* loss, int32_t* status, cudaStream_t st, bool do_rowinfo);
cudaError_t pruned_bwd_input_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, const uint16_t* W,
                                    const int32_t* ranges, const int64_t* bnd, float* d_enc, float* d_dec,
                                    cudaStream_t st);
cudaError_t pruned_bwd_weight_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, float* d_w, float* d_b,
                                     cudaStream_t st, int mode);
cudaError_t loss_sums_launch(const float* ls, const float* lp, const int32_t* status, int N, float s_scale,
                             float p_scale, float* out, int mode, cudaStream_t st);
cudaError_t split_reduce_acc_launch(const float* part, int splits, long long M, float* out, int mode, int kid,
                                    cudaStream_t st);
cudaError_t full_loss_launch(const Dims& d, void* base, const float* enc, const float* dec, const uint16_t* W,
                             const uint16_t* b, const int64_t* sym, const int64_t* bnd, float gs, float* loss,
                             float* d_enc, float* d_dec, float* d_w, float* d_b, int32_t* status, cudaStream_t st);
cudaError_t pruned_loss_launch(const Dims& d, const PrunedWS& w, const uint16_t* h, const uint16_t* W,
                               const uint16_t* b, const int64_t* sym, const int32_t* ranges,
                               const int64_t* bnd, float gs, float* loss, float* d_enc, float* d_dec,
                               float* d_w, float* d_b, int32_t* status, cudaStream_t st);
}  // namespace rnnt

namespace rnnt {
void set_timeline(void* buf);
void set_fwd_trace(void* buf);
void set_dh_trace(void* buf);
void set_scan_trace(void* buf);
static thread_local unsigned long long g_launches = 0;
static thread_local int g_prof_id = 0;
static thread_local cudaEvent_t g_prof_start = nullptr, g_prof_stop = nullptr;

static const char* const kNames[KID_COUNT] = {
    "none", "validate", "simple_prep", "unused_exp_split_lm", "simple_norm_gemm", "skew_fill", "lattice_fb",
    "lattice_combine", "simple_am_grad_gemm", "unused_am_picks", "simple_lm_grad_gemm", "unused_lm_picks",
    "ranges_raw", "ranges_adjust", "prune_gather", "pruned_rowinfo", "joiner_fwd_gemm", "joiner_softmax",
    "pruned_fb", "pruned_unused", "pruned_combine", "joiner_dh_gemm", "joiner_band_chunk", "joiner_band_dec",
    "joiner_dw_gemm", "joiner_db", "joiner_dw_reduce", "joiner_db_reduce", "bias_pad", "occ_sums",
    "smooth_lm_avg", "smooth_ac_lse", "smooth_avg_grad", "smooth_q", "full_scatter", "full_pack", "full_live",
    "full_dgrad", "loss_sums", "exchange_sum", "joiner_scale_rows"};

bool pdl_enabled() {
  static const bool on = env_int("RNNT_PDL", 1) != 0;
  return on;
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

const char* kernel_name(int id) { return (id >= 0 && id < KID_COUNT) ? kNames[id] : "unknown"; }

void launch_begin(int id, cudaStream_t st) {
  if (id == g_prof_id && g_prof_start) cudaEventRecord(g_prof_start, st);
}
void launch_end(int id, cudaStream_t st) {
  ++g_launches;
  if (id == g_prof_id && g_prof_stop) cudaEventRecord(g_prof_stop, st);
}
}  // namespace rnnt

using namespace rnnt;

static bool aligned16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

static rnnt_status_t check_dims(const rnnt_dims_t* dims, Dims* d) {
  if (!dims) return RNNT_ERR_INVALID_ARG;
  d->N = dims->N; d->T = dims->T; d->U = dims->U; d->V = dims->V; d->J = dims->J; d->S = dims->S;
  if (d->N < 1 || d->T < 1 || d->T > 65536 || d->U < 0 || d->V < 2 || d->S < 1 || d->S > 32)
    return RNNT_ERR_INVALID_ARG;
  if ((long long)d->U >= (long long)d->T * 64) return RNNT_ERR_INVALID_ARG;
  if (d->J < 8 || d->J > 4096 || d->J % 8) return RNNT_ERR_INVALID_ARG;
  if (d->lat_R() == 0) return RNNT_ERR_UNSUPPORTED;   // recursion kernel: one warp x <= 32 columns per lane
  return RNNT_OK;
}

static thread_local const char* g_last_cuda_error = "no error";
static rnnt_status_t cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return RNNT_OK;
  g_last_cuda_error = cudaGetErrorString(e);
  return RNNT_ERR_CUDA;
}

extern "C" {

size_t rnnt_workspace_bytes(const rnnt_dims_t* dims) {
  Dims d;
  if (check_dims(dims, &d) != RNNT_OK) return 0;
  return carve(d, nullptr, nullptr, nullptr);
}

// dims of the full (unpruned) loss: S is ignored (the band is every token position)
static rnnt_status_t check_full_dims(const rnnt_dims_t* dims, Dims* d) {
  if (!dims) return RNNT_ERR_INVALID_ARG;
  rnnt_dims_t x = *dims;
  x.S = 1;
  rnnt_status_t rs = check_dims(&x, d);
  if (rs != RNNT_OK) return rs;
  Dims df = *d;
  df.S = d->U + 1;
  *d = df;
  return RNNT_OK;
}

size_t rnnt_full_workspace_bytes(const rnnt_dims_t* dims) {
  Dims d;
  if (check_full_dims(dims, &d) != RNNT_OK) return 0;
  return carve_full(d, nullptr, nullptr, nullptr, nullptr);
}

const char* rnnt_status_string(rnnt_status_t s) {
  switch (s) {
    case RNNT_OK: return "RNNT_OK";
    case RNNT_ERR_INVALID_ARG: return "RNNT_ERR_INVALID_ARG";
    case RNNT_ERR_UNSUPPORTED: return "RNNT_ERR_UNSUPPORTED";
    case RNNT_ERR_WORKSPACE: return "RNNT_ERR_WORKSPACE";
    case RNNT_ERR_CUDA: return "RNNT_ERR_CUDA";
  }
  return "RNNT_ERR_UNKNOWN";
}

uint64_t rnnt_launch_count(void) { return g_launches; }

const char* rnnt_last_cuda_error(void) { return g_last_cuda_error; }

int32_t rnnt_kernel_count(void) { return KID_COUNT; }

const char* rnnt_kernel_name(int32_t id) { return kernel_name(id); }

rnnt_status_t rnnt_profile_kernel(int32_t kernel_id, void* start_event, void* stop_event) {
  if (kernel_id < 0 || kernel_id >= KID_COUNT) return RNNT_ERR_INVALID_ARG;
  g_prof_id = kernel_id;
  g_prof_start = (cudaEvent_t)start_event;
  g_prof_stop = (cudaEvent_t)stop_event;
  return RNNT_OK;
}

const char* rnnt_version(void) { return "rnnt-b200 0.2 sm_100a (all contractions tcgen05: simple bf16x3, joiner bf16)"; }

static void* align_ws(void* ws) {
  uintptr_t p = reinterpret_cast<uintptr_t>(ws);
  return reinterpret_cast<void*>((p + 255) & ~uintptr_t(255));
}

static rnnt_status_t simple_loss_impl(const float* am, const float* lm, const int64_t* symbols,
                                      const int64_t* boundary, const rnnt_dims_t* dims, Smooth sm, float grad_scale,
                                      float* loss, float* px_grad, float* py_grad, float* am_grad, float* lm_grad,
                                      int32_t* status, void* workspace, size_t workspace_bytes, void* stream) {
  Dims d;
  rnnt_status_t rs = check_dims(dims, &d);
  if (rs != RNNT_OK) return rs;
  if (!am || !lm || !boundary || !loss || !px_grad || !py_grad || !workspace) return RNNT_ERR_INVALID_ARG;
  if (d.U > 0 && !symbols) return RNNT_ERR_INVALID_ARG;
  if (!aligned16(am) || !aligned16(lm)) return RNNT_ERR_INVALID_ARG;
  if (!(sm.a_lm == sm.a_lm) || !(sm.a_ac == sm.a_ac)) return RNNT_ERR_INVALID_ARG;   // NaN scales
  if (workspace_bytes < carve(d, nullptr, nullptr, nullptr)) return RNNT_ERR_WORKSPACE;
  SimpleWS sw;
  PrunedWS pw;
  carve(d, align_ws(workspace), &sw, &pw);
  return cuda_status(simple_loss_launch(d, sw, am, lm, symbols, boundary, grad_scale, loss, px_grad, py_grad,
                                        am_grad, lm_grad, status, sm, (cudaStream_t)stream));
}

static rnnt_status_t simple_backward_impl(const float* am, const float* lm, const float* px_grad,
                                          const float* py_grad, const int64_t* symbols, const int64_t* boundary,
                                          const rnnt_dims_t* dims, Smooth sm, float grad_scale, float* am_grad,
                                          float* lm_grad, void* workspace, size_t workspace_bytes, void* stream) {
  Dims d;
  rnnt_status_t rs = check_dims(dims, &d);
  if (rs != RNNT_OK) return rs;
  if (!am || !lm || !px_grad || !py_grad || !boundary || !workspace) return RNNT_ERR_INVALID_ARG;
  if (!am_grad && !lm_grad) return RNNT_ERR_INVALID_ARG;
  if (d.U > 0 && !symbols) return RNNT_ERR_INVALID_ARG;
  if (!aligned16(am) || !aligned16(lm) || !aligned16(am_grad) || !aligned16(lm_grad)) return RNNT_ERR_INVALID_ARG;
  if (!(sm.a_lm == sm.a_lm) || !(sm.a_ac == sm.a_ac)) return RNNT_ERR_INVALID_ARG;
  if (workspace_bytes < carve(d, nullptr, nullptr, nullptr)) return RNNT_ERR_WORKSPACE;
  SimpleWS sw;
  PrunedWS pw;
  carve(d, align_ws(workspace), &sw, &pw);
  return cuda_status(simple_grads_launch(d, sw, am, lm, px_grad, py_grad, symbols, boundary, grad_scale, am_grad,
                                         lm_grad, sm, (cudaStream_t)stream));
}

rnnt_status_t rnnt_simple_loss(const float* am, const float* lm, const int64_t* symbols,
                               const int64_t* boundary, const rnnt_dims_t* dims, float grad_scale,
                               float* loss, float* px_grad, float* py_grad, float* am_grad,
                               float* lm_grad, int32_t* status, void* workspace,
                               size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("rnnt_simple_loss");   // (profiler range; a no-op without an attached tool)
  return simple_loss_impl(am, lm, symbols, boundary, dims, Smooth{}, grad_scale, loss, px_grad, py_grad, am_grad,
                          lm_grad, status, workspace, workspace_bytes, stream);
}

rnnt_status_t rnnt_simple_loss_backward(const float* am, const float* lm, const float* px_grad,
                                        const float* py_grad, const int64_t* symbols, const int64_t* boundary,
                                        const rnnt_dims_t* dims, float grad_scale, float* am_grad, float* lm_grad,
                                        void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("rnnt_simple_loss_backward");   // (profiler range; a no-op without an attached tool)
  return simple_backward_impl(am, lm, px_grad, py_grad, symbols, boundary, dims, Smooth{}, grad_scale, am_grad,
                              lm_grad, workspace, workspace_bytes, stream);
}

rnnt_status_t rnnt_simple_loss_smoothed(const float* am, const float* lm, const int64_t* symbols,
                                        const int64_t* boundary, const rnnt_dims_t* dims, float lm_only_scale,
                                        float am_only_scale, float grad_scale, float* loss, float* px_grad,
                                        float* py_grad, float* am_grad, float* lm_grad, int32_t* status,
                                        void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("rnnt_simple_loss_smoothed");   // (profiler range; a no-op without an attached tool)
  return simple_loss_impl(am, lm, symbols, boundary, dims, Smooth{lm_only_scale, am_only_scale}, grad_scale, loss,
                          px_grad, py_grad, am_grad, lm_grad, status, workspace, workspace_bytes, stream);
}

rnnt_status_t rnnt_simple_loss_smoothed_backward(const float* am, const float* lm, const float* px_grad,
                                                 const float* py_grad, const int64_t* symbols,
                                                 const int64_t* boundary, const rnnt_dims_t* dims,
                                                 float lm_only_scale, float am_only_scale, float grad_scale,
                                                 float* am_grad, float* lm_grad, void* workspace,
                                                 size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("rnnt_simple_loss_smoothed_backward");   // (profiler range; a no-op without an attached tool)
  return simple_backward_impl(am, lm, px_grad, py_grad, symbols, boundary, dims, Smooth{lm_only_scale, am_only_scale},
                              grad_scale, am_grad, lm_grad, workspace, workspace_bytes, stream);
}

rnnt_status_t rnnt_get_ranges(const float* px_grad, const float* py_grad, const int64_t* boundary,
                              const rnnt_dims_t* dims, int32_t* ranges, int32_t* status, void* stream) {
  NvtxRange nvtx_("rnnt_get_ranges");   // (profiler range; a no-op without an attached tool)
  Dims d;
  rnnt_status_t rs = check_dims(dims, &d);
  if (rs != RNNT_OK) return rs;
  if (!px_grad || !py_grad || !boundary || !ranges) return RNNT_ERR_INVALID_ARG;
  return cuda_status(get_ranges_launch(d, px_grad, py_grad, boundary, ranges, status, (cudaStream_t)stream));
}

rnnt_status_t rnnt_prune(const float* enc_proj, const float* dec_proj, const int32_t* ranges,
                         const int64_t* boundary, const rnnt_dims_t* dims, uint16_t* h, void* stream) {
  NvtxRange nvtx_("rnnt_prune");   // (profiler range; a no-op without an attached tool)
  Dims d;
  rnnt_status_t rs = check_dims(dims, &d);
  if (rs != RNNT_OK) return rs;
  if (!enc_proj || !dec_proj || !ranges || !boundary || !h) return RNNT_ERR_INVALID_ARG;
  if (!aligned16(enc_proj) || !aligned16(dec_proj) || !aligned16(h)) return RNNT_ERR_INVALID_ARG;
  return cuda_status(prune_launch(d, enc_proj, dec_proj, ranges, boundary, h, (cudaStream_t)stream));
}

rnnt_status_t rnnt_pruned_loss(const uint16_t* h, const uint16_t* w_out, const uint16_t* b_out,
                               const int64_t* symbols, const int32_t* ranges,
                               const int64_t* boundary, const rnnt_dims_t* dims, float grad_scale,
                               float* loss, float* d_enc, float* d_dec, float* d_w, float* d_b,
                               int32_t* status, void* workspace, size_t workspace_bytes,
                               void* stream) {
  NvtxRange nvtx_("rnnt_pruned_loss");   // (profiler range; a no-op without an attached tool)
  Dims d;
  rnnt_status_t rs = check_dims(dims, &d);
  if (rs != RNNT_OK) return rs;
  if (!h || !w_out || !b_out || !ranges || !boundary || !loss || !d_w || !d_b || !workspace)
    return RNNT_ERR_INVALID_ARG;
  if (d.U > 0 && !symbols) return RNNT_ERR_INVALID_ARG;
  if (!aligned16(h) || !aligned16(w_out)) return RNNT_ERR_INVALID_ARG;
  if (workspace_bytes < carve(d, nullptr, nullptr, nullptr)) return RNNT_ERR_WORKSPACE;
  if (pruned_recursion_smem(d) > 224 * 1024) return RNNT_ERR_UNSUPPORTED;
  SimpleWS sw;
  PrunedWS pw;
  carve(d, align_ws(workspace), &sw, &pw);
  return cuda_status(pruned_loss_launch(d, pw, h, w_out, b_out, symbols, ranges, boundary, grad_scale, loss,
                                        d_enc, d_dec, d_w, d_b, status, (cudaStream_t)stream));
}

rnnt_status_t rnnt_full_loss(const float* enc_proj, const float* dec_proj, const uint16_t* w_out,
                             const uint16_t* b_out, const int64_t* symbols, const int64_t* boundary,
                             const rnnt_dims_t* dims, float grad_scale, float* loss, float* d_enc, float* d_dec,
                             float* d_w, float* d_b, int32_t* status, void* workspace, size_t workspace_bytes,
                             void* stream) {
  NvtxRange nvtx_("rnnt_full_loss");   // (profiler range; a no-op without an attached tool)
  Dims d;
  rnnt_status_t rs = check_full_dims(dims, &d);
  if (rs != RNNT_OK) return rs;
  if (!enc_proj || !dec_proj || !w_out || !b_out || !boundary || !loss || !d_w || !d_b || !workspace)
    return RNNT_ERR_INVALID_ARG;
  if (d.U > 0 && !symbols) return RNNT_ERR_INVALID_ARG;
  if (!aligned16(enc_proj) || !aligned16(dec_proj) || !aligned16(w_out) || !aligned16(d_enc) || !aligned16(d_dec))
    return RNNT_ERR_INVALID_ARG;
  if (workspace_bytes < carve_full(d, nullptr, nullptr, nullptr, nullptr)) return RNNT_ERR_WORKSPACE;
  Dims d0 = d;
  d0.S = 1;
  return cuda_status(full_loss_launch(d0, align_ws(workspace), enc_proj, dec_proj, w_out, b_out, symbols, boundary,
                                      grad_scale, loss, d_enc, d_dec, d_w, d_b, status, (cudaStream_t)stream));
}

rnnt_status_t rnnt_pruned_loss_forward(const uint16_t* h, const uint16_t* w_out, const uint16_t* b_out,
                                       const int64_t* symbols, const int32_t* ranges, const int64_t* boundary,
                                       const rnnt_dims_t* dims, float grad_scale, float* loss, int32_t* status,
                                       void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("rnnt_pruned_loss_forward");   // (profiler range; a no-op without an attached tool)
  Dims d;
  rnnt_status_t rs = check_dims(dims, &d);
  if (rs != RNNT_OK) return rs;
  if (!h || !w_out || !b_out || !ranges || !boundary || !loss || !workspace) return RNNT_ERR_INVALID_ARG;
  if (d.U > 0 && !symbols) return RNNT_ERR_INVALID_ARG;
  if (!aligned16(h) || !aligned16(w_out)) return RNNT_ERR_INVALID_ARG;
  if (workspace_bytes < carve(d, nullptr, nullptr, nullptr)) return RNNT_ERR_WORKSPACE;
  if (pruned_recursion_smem(d) > 224 * 1024) return RNNT_ERR_UNSUPPORTED;
  SimpleWS sw;
  PrunedWS pw;
  carve(d, align_ws(workspace), &sw, &pw);
  return cuda_status(pruned_fwd_launch(d, pw, h, w_out, b_out, symbols, ranges, boundary, grad_scale, loss, status,
                                       (cudaStream_t)stream, true));
}

rnnt_status_t rnnt_pruned_loss_prepare(const int32_t* ranges, const int64_t* symbols, const int64_t* boundary,
                                       const rnnt_dims_t* dims, const uint16_t* b_out, float grad_scale,
                                       void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("rnnt_pruned_loss_prepare");   // (profiler range; a no-op without an attached tool)
  Dims d;
  rnnt_status_t rs = check_dims(dims, &d);
  if (rs != RNNT_OK) return rs;
  if (!ranges || !boundary || !b_out || !workspace) return RNNT_ERR_INVALID_ARG;
  if (d.U > 0 && !symbols) return RNNT_ERR_INVALID_ARG;
  if (workspace_bytes < carve(d, nullptr, nullptr, nullptr)) return RNNT_ERR_WORKSPACE;
  SimpleWS sw;
  PrunedWS pw;
  carve(d, align_ws(workspace), &sw, &pw);
  return cuda_status(rowinfo_launch(d, pw, ranges, symbols, boundary, b_out, grad_scale, (cudaStream_t)stream));
}

rnnt_status_t rnnt_pruned_loss_forward_prepared(const uint16_t* h, const uint16_t* w_out, const uint16_t* b_out,
                                                const int64_t* symbols, const int32_t* ranges,
                                                const int64_t* boundary, const rnnt_dims_t* dims, float grad_scale,
                                                float* loss, int32_t* status, void* workspace,
                                                size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("rnnt_pruned_loss_forward_prepared");   // (profiler range; a no-op without an attached tool)
  Dims d;
  rnnt_status_t rs = check_dims(dims, &d);
  if (rs != RNNT_OK) return rs;
  if (!h || !w_out || !b_out || !ranges || !boundary || !loss || !workspace) return RNNT_ERR_INVALID_ARG;
  if (d.U > 0 && !symbols) return RNNT_ERR_INVALID_ARG;
  if (!aligned16(h) || !aligned16(w_out)) return RNNT_ERR_INVALID_ARG;
  if (workspace_bytes < carve(d, nullptr, nullptr, nullptr)) return RNNT_ERR_WORKSPACE;
  if (pruned_recursion_smem(d) > 224 * 1024) return RNNT_ERR_UNSUPPORTED;
  SimpleWS sw;
  PrunedWS pw;
  carve(d, align_ws(workspace), &sw, &pw);
  return cuda_status(pruned_fwd_launch(d, pw, h, w_out, b_out, symbols, ranges, boundary, grad_scale, loss, status,
                                       (cudaStream_t)stream, false));
}

rnnt_status_t rnnt_pruned_loss_backward_input(const uint16_t* h, const uint16_t* w_out, const int32_t* ranges,
                                              const int64_t* boundary, const rnnt_dims_t* dims, float* d_enc,
                                              float* d_dec, void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("rnnt_pruned_loss_backward_input");   // (profiler range; a no-op without an attached tool)
  Dims d;
  rnnt_status_t rs = check_dims(dims, &d);
  if (rs != RNNT_OK) return rs;
  if (!h || !w_out || !ranges || !boundary || !workspace || (!d_enc && !d_dec)) return RNNT_ERR_INVALID_ARG;
  if (!aligned16(h) || !aligned16(w_out) || !aligned16(d_enc) || !aligned16(d_dec)) return RNNT_ERR_INVALID_ARG;
  if (workspace_bytes < carve(d, nullptr, nullptr, nullptr)) return RNNT_ERR_WORKSPACE;
  SimpleWS sw;
  PrunedWS pw;
  carve(d, align_ws(workspace), &sw, &pw);
  return cuda_status(pruned_bwd_input_launch(d, pw, h, w_out, ranges, boundary, d_enc, d_dec, (cudaStream_t)stream));
}

rnnt_status_t rnnt_pruned_loss_backward_weight(const uint16_t* h, const rnnt_dims_t* dims, float* d_w, float* d_b,
                                               void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("rnnt_pruned_loss_backward_weight");   // (profiler range; a no-op without an attached tool)
  Dims d;
  rnnt_status_t rs = check_dims(dims, &d);
  if (rs != RNNT_OK) return rs;
  if (!h || !d_w || !d_b || !workspace) return RNNT_ERR_INVALID_ARG;
  if (!aligned16(h) || !aligned16(d_w)) return RNNT_ERR_INVALID_ARG;
  if (workspace_bytes < carve(d, nullptr, nullptr, nullptr)) return RNNT_ERR_WORKSPACE;
  SimpleWS sw;
  PrunedWS pw;
  carve(d, align_ws(workspace), &sw, &pw);
  return cuda_status(pruned_bwd_weight_launch(d, pw, h, d_w, d_b, (cudaStream_t)stream, 0));
}

rnnt_status_t rnnt_pruned_backward_mode(const rnnt_dims_t* dims, const void* workspace, size_t workspace_bytes,
                                        int32_t* plain, void* stream) {
  Dims d;
  rnnt_status_t rs = check_dims(dims, &d);
  if (rs != RNNT_OK) return rs;
  if (!workspace || !plain) return RNNT_ERR_INVALID_ARG;
  if (workspace_bytes < carve(d, nullptr, nullptr, nullptr)) return RNNT_ERR_WORKSPACE;
  SimpleWS sw;
  PrunedWS pw;
  carve(d, align_ws(const_cast<void*>(workspace)), &sw, &pw);
  int32_t v = 1;
  cudaError_t e = cudaMemcpyAsync(&v, pw.tscale, 4, cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  *plain = v == 0 ? 1 : 0;
  return cuda_status(e);
}

rnnt_status_t rnnt_pruned_loss_backward_weight_exchange(const uint16_t* h, const rnnt_dims_t* dims, int32_t mode,
                                                        float* d_w, float* d_b, void* workspace,
                                                        size_t workspace_bytes, void* stream) {
  NvtxRange nvtx_("rnnt_pruned_loss_backward_weight_exchange");   // (profiler range; a no-op without an attached tool)
  Dims d;
  rnnt_status_t rs = check_dims(dims, &d);
  if (rs != RNNT_OK) return rs;
  if (mode < RNNT_EXCHANGE_STORE || mode > RNNT_EXCHANGE_MULTIMEM) return RNNT_ERR_INVALID_ARG;
  if (!h || !d_w || !d_b || !workspace) return RNNT_ERR_INVALID_ARG;
  if (!aligned16(h) || !aligned16(d_w)) return RNNT_ERR_INVALID_ARG;
  if (workspace_bytes < carve(d, nullptr, nullptr, nullptr)) return RNNT_ERR_WORKSPACE;
  SimpleWS sw;
  PrunedWS pw;
  carve(d, align_ws(workspace), &sw, &pw);
  return cuda_status(pruned_bwd_weight_launch(d, pw, h, d_w, d_b, (cudaStream_t)stream, mode));
}

rnnt_status_t rnnt_exchange_sum(const float* parts, int32_t nparts, int64_t M, int32_t mode, float* out,
                                void* stream) {
  NvtxRange nvtx_("rnnt_exchange_sum");   // (profiler range; a no-op without an attached tool)
  if (!parts || !out || nparts < 1 || M < 1) return RNNT_ERR_INVALID_ARG;
  if (mode < RNNT_EXCHANGE_STORE || mode > RNNT_EXCHANGE_MULTIMEM) return RNNT_ERR_INVALID_ARG;
  return cuda_status(split_reduce_acc_launch(parts, nparts, (long long)M, out, mode, KID_EXCHANGE_SUM,
                                             (cudaStream_t)stream));
}

rnnt_status_t rnnt_loss_sums(const float* loss_simple, const float* loss_pruned, const int32_t* status, int32_t N,
                             float simple_scale, float pruned_scale, int32_t mode, float* out, void* stream) {
  NvtxRange nvtx_("rnnt_loss_sums");   // (profiler range; a no-op without an attached tool)
  if (!loss_simple || !loss_pruned || !out || N < 1) return RNNT_ERR_INVALID_ARG;
  if (mode < RNNT_EXCHANGE_STORE || mode > RNNT_EXCHANGE_MULTIMEM) return RNNT_ERR_INVALID_ARG;
  return cuda_status(loss_sums_launch(loss_simple, loss_pruned, status, N, simple_scale, pruned_scale, out, mode,
                                      (cudaStream_t)stream));
}

#ifdef RNNT_DIAGNOSTICS
/* diagnostics builds only (-DRNNT_DIAGNOSTICS, not in rnnt.h): per-CTA phase timestamps of the
   simple-loss GEMMs, joiner_dh and the pruned scan into buf (process-global, never in the product) */
void rnnt_debug_timeline(void* buf) {
  rnnt::set_timeline(buf);
  rnnt::set_dh_trace(buf ? static_cast<char*>(buf) + (4u << 20) : nullptr);   // joiner_dh trace 4 MiB in
  rnnt::set_scan_trace(buf ? static_cast<char*>(buf) + (6u << 20) : nullptr); // pruned scan trace 6 MiB in
  rnnt::set_fwd_trace(buf ? static_cast<char*>(buf) + (7u << 20) : nullptr);  // joiner forward trace 7 MiB in
}
#endif

}  // extern "C"
