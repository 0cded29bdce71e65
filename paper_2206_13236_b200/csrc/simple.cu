// simple.cu — stage 1: the trivial ("simple") joiner loss, its lattice
// recursion (Eq. 3) and occupancies, and the am/lm gradients.
//
// Sequence (all on the caller's stream):
//   K1 simple_prep (simple_tc.cu)      one launch: row maxima (Eq. 6 offsets), bf16 hi/lo
//                                      of e^{x-m}, amy gather, one-hot rows, sentinels in the invalid
//                                      skewed cells, symbol / boundary validation -> status
//   K2 norm gemm3 (simple_tc.cu)       S(t,u) on tcgen05, epilogue: skewed arcs px2/py2 and 1/S
//   K3/K4 (lattice.cu)                 alpha || beta wavefronts, occupancies, G~
//   K5 am/lm grad gemm3 (simple_tc.cu) d(-L)/d am, d(-L)/d lm (chain rule through Eq. 5-6)
#include "common.cuh"
#include "launch.h"
#include "workspace.h"

namespace rnnt {

// ------------------------------------------------------------------ host driver
cudaError_t lattice_launch(const Dims& d, const SimpleWS& w, const int64_t* bnd, float* loss, float* px_grad,
                           float* py_grad, int32_t* status, cudaStream_t st);

cudaError_t simple_prep_launch(const Dims& d, const SimpleWS& w, const float* am, const float* lm, const int64_t* sym,
                               const int64_t* bnd, int32_t* status, cudaStream_t st);
cudaError_t norm_gemm_launch(const Dims& d, const SimpleWS& w, const float* am, const float* lm, const int64_t* sym,
                             const int64_t* bnd, int32_t* status, Smooth sm, cudaStream_t st);
cudaError_t simple_grads_launch(const Dims& d, const SimpleWS& w, const float* am, const float* lm,
                                const float* px_grad, const float* py_grad, const int64_t* sym, const int64_t* bnd,
                                float gs, float* am_grad, float* lm_grad, Smooth sm, cudaStream_t st);

cudaError_t simple_loss_launch(const Dims& d, const SimpleWS& w, const float* am, const float* lm,
                               const int64_t* sym, const int64_t* bnd, float gs, float* loss,
                               float* px_grad, float* py_grad, float* am_grad, float* lm_grad,
                               int32_t* status, Smooth sm, cudaStream_t st) {
  cudaError_t e;
  if ((e = simple_prep_launch(d, w, am, lm, sym, bnd, status, st)) != cudaSuccess) return e;
  if ((e = norm_gemm_launch(d, w, am, lm, sym, bnd, status, sm, st)) != cudaSuccess) return e;
  if ((e = lattice_launch(d, w, bnd, loss, px_grad, py_grad, status, st)) != cudaSuccess) return e;
  if ((e = simple_grads_launch(d, w, am, lm, px_grad, py_grad, sym, bnd, gs, am_grad, lm_grad, sm, st)) != cudaSuccess)
    return e;
  return cudaGetLastError();
}

}  // namespace rnnt
