// run_colhist4p.cuh -- launcher template of the pair-record kernel
// (k_colhist4p_u8), shared by run_colhist4p.cu and run_colhist4q.cu (the
// PL = 4 compile-time window sides, a separate translation unit so the two
// compile in parallel).
#pragma once
#include <algorithm>

#include "host.h"
#include "kernels_colhist.cuh"

namespace mtb {

template <int T, int G, int M, int PL, int NF = 0>
inline int run_colhist4p_u8_gm(SlabParams p, int B, cudaStream_t s, const char *name) {
    const size_t smem = (size_t)colhist4q_bytes(T, p.radius, PL);
    auto kern = p.in_rows ? k_colhist4p_u8<T, G, M, PL, true, NF> : k_colhist4p_u8<T, G, M, PL, false, NF>;
    if (int rc = set_smem(kern, smem)) return rc;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem);
    if (per_sm < 1) per_sm = 1;
    const int bx = (p.W + T - 1) / T;
    p.rows_per_cta = rows_per_cta(p, bx, B, per_sm);
    dim3 grid(bx, (p.row_end - p.row_begin + p.rows_per_cta - 1) / p.rows_per_cta, B);
    return launch(kern, grid, T, smem, s, p, name);
}

}  // namespace mtb
