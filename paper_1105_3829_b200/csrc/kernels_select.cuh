// kernels_select.cuh -- independent exact rank selection, O(d * n^2) per
// pixel: the package's own cross-check (the reference's oracle filters,
// oracles.py:23-66, serve the CLI `compare` command and tests; here they run
// on the GPU with an algorithm that shares nothing with the fast kernels).
//
// Per output pixel: the rank-th smallest window value is the largest v with
// count(window < v) < rank; its bits are decided from the top, each by one
// counting pass over the n x n (replicate-clamped) window.
#pragma once
#include "common.cuh"

namespace mtb {

template <typename P, int D>
__global__ void k_select_brute(const P *__restrict__ src, int64_t src_pitch, P *__restrict__ dst,
                               int64_t dst_pitch, int H, int W, int r, uint32_t rank) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= W || y >= H) return;
    unsigned ans = 0;
    for (int b = D - 1; b >= 0; --b) {
        const unsigned t = ans | (1u << b);
        uint32_t below = 0;
        for (int j = -r; j <= r; ++j) {
            const P *row = src + (int64_t)clampi(y + j, 0, H - 1) * src_pitch;
            for (int i = -r; i <= r; ++i) below += __ldg(row + clampi(x + i, 0, W - 1)) < t ? 1u : 0u;
        }
        if (below < rank) ans = t;
    }
    dst[(int64_t)y * dst_pitch + x] = (P)ans;
}

}  // namespace mtb
