// run_hi16.cuh -- launcher template of the pair-record kernel keyed by the
// high byte of 16-bit pixels (k_colhist4p_u8<..., uint16_t>: first pass of
// the candidate-list path, run_lowsel16.cu), compile-time window sides split
// over run_hi16_a.cu / run_hi16_b.cu so that they compile in parallel.
#pragma once
#include <algorithm>

#include "host.h"
#include "kernels_colhist.cuh"

namespace mtb {

constexpr int HI16_NOT_COVERED = 1;  // (MTB status codes are 0 or negative)

// pair levels as in the 8-bit dispatch (run_colhist.cu): level-2 singles up
// to r = 16, derived from level 3 above
constexpr int hi16_pair_levels(int r) { return r <= 16 ? 3 : 4; }

template <int NLO, int NHI>
inline int run_hi16_fixed(SlabParams p, int B, cudaStream_t s) {
    const int n = 2 * p.radius + 1;
    if (n < NLO || n > NHI) return HI16_NOT_COVERED;
    return with_fixed_n<NLO, NHI>(n, [&](auto nf) {
        constexpr int NF = decltype(nf)::value;
        if constexpr (NF == 0) {
            return HI16_NOT_COVERED;
        } else {
            constexpr int T = 256, G = carry_free_group(NF), PL = hi16_pair_levels(NF / 2);
            const size_t smem = (size_t)colhist4q_bytes(T, NF / 2, PL);
            auto kern = k_colhist4p_u8<T, G, NF % G, PL, false, NF, uint16_t>;
            if (int rc = set_smem(kern, smem)) return rc;
            int per_sm = 1;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem);
            if (per_sm < 1) per_sm = 1;
            const int bx = (p.W + T - 1) / T;
            p.rows_per_cta = rows_per_cta(p, bx, B, per_sm);
            dim3 grid(bx, (p.row_end - p.row_begin + p.rows_per_cta - 1) / p.rows_per_cta, B);
            return launch(kern, grid, T, smem, s, p, "k_colhist4p_u8<256,u16 high byte>");
        }
    });
}

}  // namespace mtb
