// run_colhist16c.cu -- launcher of k_colhist16c_u16 (16-bit, widely spread
// data: high byte by pair records, low byte by candidates).
#include <algorithm>

#include "host.h"
#include "kernels_colhist16c.cuh"

namespace mtb {

constexpr int CH16C_T = 128;
constexpr int CH16C_CMAX = 32;

template <int G, int M, int PL, int NF = 0>
static int run_colhist16c_gm(SlabParams p, int B, cudaStream_t s) {
    constexpr int T = CH16C_T;
    const size_t smem = (size_t)ch16c_bytes(T, p.radius, PL, CH16C_CMAX);
    if (smem > 227 * 1024) return run_colhist16_u16(p, B, s, 0);  // spans too large: two-phase kernel
    auto kern = p.in_rows ? k_colhist16c_u16<T, G, M, PL, CH16C_CMAX, true, NF>
                          : k_colhist16c_u16<T, G, M, PL, CH16C_CMAX, false, NF>;
    if (int rc = set_smem(kern, smem)) return rc;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem);
    if (per_sm < 1) per_sm = 1;
    const int n = 2 * p.radius + 1;
    const int bx = (p.W + T - 1) / T;
    // short slabs (~2n rows, many waves): the per-row work varies with the
    // data from CTA to CTA, and short slabs even it out -- config 3 r = 15
    // 3.17 -> 2.66 ms, r = 7 1.72 -> 1.46 ms against two waves of ~150-row
    // slabs, despite the extra span builds
    p.rows_per_cta = std::max(rows_per_cta(p, bx, B, per_sm, 16), std::min(2 * n, p.row_end - p.row_begin));
    dim3 grid(bx, (p.row_end - p.row_begin + p.rows_per_cta - 1) / p.rows_per_cta, B);
    return launch(kern, grid, T, smem, s, p, "k_colhist16c_u16");
}

template <int PL>
static int run_colhist16c_pl(SlabParams p, int B, cudaStream_t s) {
    const int n = 2 * p.radius + 1;
    if (8 * n <= 255) {
        switch (n % 8) {
            case 1: return run_colhist16c_gm<8, 1, PL>(p, B, s);
            case 3: return run_colhist16c_gm<8, 3, PL>(p, B, s);
            case 5: return run_colhist16c_gm<8, 5, PL>(p, B, s);
            default: return run_colhist16c_gm<8, 7, PL>(p, B, s);
        }
    }
    if (4 * n <= 255) return n % 4 == 1 ? run_colhist16c_gm<4, 1, PL>(p, B, s) : run_colhist16c_gm<4, 3, PL>(p, B, s);
    return run_colhist16c_gm<2, 1, PL>(p, B, s);
}

// n <= 127 (pair counts <= 2n fit u8)
int run_colhist16c_u16(SlabParams p, int B, cudaStream_t s) {
    const int n = 2 * p.radius + 1;
    if (n > 127) return run_colhist16_u16(p, B, s, 0);
    if (n >= 5 && n <= 47) {  // compile-time window side for the radii this kernel serves (r <= 23)
        return with_fixed_n<5, 47>(n, [&](auto nf) {
            constexpr int NF = decltype(nf)::value, G = carry_free_group(NF);
            constexpr int PL = ch16c_pair_levels(CH16C_T, NF / 2, CH16C_CMAX);
            return run_colhist16c_gm<G, NF % G, PL, NF>(p, B, s);
        });
    }
    return ch16c_pair_levels(CH16C_T, p.radius, CH16C_CMAX) == 3 ? run_colhist16c_pl<3>(p, B, s)
                                                                   : run_colhist16c_pl<2>(p, B, s);
}

}  // namespace mtb
