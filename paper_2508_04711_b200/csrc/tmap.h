// Host-side TMA tensor-map encoding (driver entry point fetched through the
// runtime, so the library does not link libcuda directly).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace jh {

// 2-D bf16 row-major matrix [rows x cols] with row stride `ld` elements.
// Box = 64 columns (128 B) x box_rows rows, 128B swizzle, OOB rows/cols
// zero-filled.  Returns 0 on success.
int make_tmap_bf16_2d(CUtensorMap* out, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                      uint32_t box_rows);

// 1-D int64 vector [n] (timestamps), box of `box` elements, OOB zero-filled.
int make_tmap_i64_1d(CUtensorMap* out, const void* base, uint64_t n, uint32_t box);

}  // namespace jh
