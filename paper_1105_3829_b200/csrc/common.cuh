// common.cuh -- shared parameter block and helpers for the rank-filter kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mtb {

// One launch = one slab (rows [row_begin,row_end) of a global H x W image)
// for each of gridDim.z images.  See include/medtree_b200.h for semantics.
struct SlabParams {
    const void *src;          // device, element type = pixel type
    int64_t src_pitch;        // elements
    int64_t src_img_stride;   // elements between batch images
    int32_t src_row0;         // global row held in src row 0
    int32_t src_rows;
    void *dst;
    int64_t dst_pitch;
    int64_t dst_img_stride;
    int32_t H, W;             // global image
    int32_t row_begin, row_end;
    int32_t radius;
    uint32_t rank;            // 1-based
    const void *lut;          // optional value map (2^d entries) or nullptr
    int32_t rows_per_cta;     // slab height handled by one CTA row
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

template <typename P>
__device__ __forceinline__ const P *src_row(const SlabParams &p, const P *base, int g) {
    return base + (int64_t)(g - p.src_row0) * p.src_pitch;
}

}  // namespace mtb
