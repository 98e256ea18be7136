// run_wk16.cuh -- launcher template of the pair-record kernel in window-key
// mode (k_colhist4p_u8<..., uint16_t, 1>: compact 16-bit data as one 8-bit
// problem per tile, run_lowsel16.cu), compile-time window sides split over
// run_wk16_a.cu / run_wk16_b.cu so that they compile in parallel.
#pragma once
#include <algorithm>

#include "host.h"
#include "kernels_colhist.cuh"

namespace mtb {

constexpr int WK16_NOT_COVERED = 1;  // (MTB status codes are 0 or negative)

template <int NLO, int NHI>
inline int run_wk16_fixed(SlabParams p, int B, cudaStream_t s) {
    const int n = 2 * p.radius + 1;
    if (n < NLO || n > NHI) return WK16_NOT_COVERED;
    return with_fixed_n<NLO, NHI>(n, [&](auto nf) {
        constexpr int NF = decltype(nf)::value;
        if constexpr (NF == 0) {
            return WK16_NOT_COVERED;
        } else {
            // pair levels as in the 8-bit dispatch (run_colhist.cu)
            constexpr int T = 256, G = carry_free_group(NF), PL = NF / 2 <= 16 ? 3 : 4;
            const size_t smem = (size_t)colhist4q_bytes(T, NF / 2, PL);
            auto kern = k_colhist4p_u8<T, G, NF % G, PL, false, NF, uint16_t, 1>;
            if (int rc = set_smem(kern, smem)) return rc;
            int per_sm = 1;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem);
            if (per_sm < 1) per_sm = 1;
            const int bx = (p.W + T - 1) / T;
            // four rounds of shorter slabs (eight from r = 56): a tile's window follows its own
            // median (config 4 r = 47: 8.2 / 5.8 / 7.4 ms at 2 / 4 / 8 rounds, r = 63: 10.8 / 11.6 / 8.9)
            p.rows_per_cta = rows_per_cta(p, bx, B, per_sm, env_int("MTB_WK16_WAVES", p.radius >= 56 ? 8 : 4));
            dim3 grid(bx, (p.row_end - p.row_begin + p.rows_per_cta - 1) / p.rows_per_cta, B);
            return launch(kern, grid, T, smem, s, p, "k_colhist4p_u8<256,u16 window key>");
        }
    });
}

}  // namespace mtb
