// tmap.h — host-side TMA descriptor encoding (cuTensorMapEncodeTiled through the runtime's
// driver entry point, so the library does not link libcuda directly).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rnnt {

// 2-D bf16 tensor [outer][inner] with row pitch `row_bytes`; box = box_inner x box_outer,
// SWIZZLE_128B (box_inner * 2 must be 128), out-of-bounds elements read as zero.
bool make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                       uint32_t box_inner, uint32_t box_outer);

}  // namespace rnnt
