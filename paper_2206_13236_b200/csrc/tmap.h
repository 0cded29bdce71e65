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

// 3-D bf16 tensor [d2][d1][d0] (row pitch stride1 bytes, plane pitch stride2 bytes); box =
// box0 x box1 x 1, SWIZZLE_128B (box0 * 2 == 128), out-of-bounds elements (also past d1 within a
// plane) read as zero — used for per-utterance operands so a box never spills into the next one.
bool make_tmap_bf16_3d(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1,
                       uint64_t stride2, uint32_t box0, uint32_t box1, uint32_t box2 = 1);

// 3-D fp32 tensor, box = box0 (32 -> 128 B rows) x box1 x 1, SWIZZLE_128B (loads and stores).
bool make_tmap_f32_3d(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1,
                      uint64_t stride2, uint32_t box0, uint32_t box1);

// 3-D fp16 tensor, box = box0 (32 -> 64 B rows) x box1 x 1, SWIZZLE_64B (stores of the fp16 dpre rows).
bool make_tmap_f16_3d(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1,
                      uint64_t stride2, uint32_t box0, uint32_t box1);

}  // namespace rnnt
