// adg_tma.cuh -- host-side TMA tensor-map encoding shared by the kernels.
#pragma once
#include <cuda.h>

#include "adg_internal.cuh"

namespace adg {

// 2-D row-major tensor [outer][inner] of `elem` type with row pitch
// `row_bytes`; box = box_inner x box_outer elements; out-of-bounds reads fill 0.
CUtensorMap make_tensor_map_2d(const void* base, CUtensorMapDataType elem, uint64_t inner,
                               uint64_t outer, uint64_t row_bytes, uint32_t box_inner,
                               uint32_t box_outer, CUtensorMapSwizzle swizzle);

}  // namespace adg
