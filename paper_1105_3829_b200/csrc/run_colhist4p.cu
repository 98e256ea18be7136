// run_colhist4p.cu -- launchers of the radix-4 column-histogram kernel with
// pair records (k_colhist4p_u8); see run_colhist.cu for the dispatch.
#include <algorithm>

#include "host.h"
#include "kernels_colhist.cuh"

namespace mtb {

template <int T, int G, int M, int PL, int NF = 0>
static int run_colhist4p_u8_gm(SlabParams p, int B, cudaStream_t s, const char *name) {
    const size_t smem = (size_t)colhist4p_bytes(T, p.radius, PL);
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

// pair records (G even: n <= 127); PL pair levels
template <int T, int PL>
static int run_colhist4p_u8(SlabParams p, int B, cudaStream_t s, const char *name) {
    const int n = 2 * p.radius + 1;
    // compile-time window side for the radii each variant serves (PL = 3:
    // r = 11..15, PL = 2: r = 16..32; run_colhist.cu)
    if (PL == 3 && n >= 5 && n <= 37)
        return with_fixed_n<5, 37>(n, [&](auto nf) {
            constexpr int NF = decltype(nf)::value, G = carry_free_group(NF);  // even: n <= 127
            return run_colhist4p_u8_gm<T, G, NF % G, PL, NF>(p, B, s, name);
        });
    if (PL == 2 && n >= 29 && n <= 65)
        return with_fixed_n<29, 65>(n, [&](auto nf) {
            constexpr int NF = decltype(nf)::value, G = carry_free_group(NF);  // even: n <= 127
            return run_colhist4p_u8_gm<T, G, NF % G, PL, NF>(p, B, s, name);
        });
    if (8 * n <= 255) {
        switch (n % 8) {
            case 1: return run_colhist4p_u8_gm<T, 8, 1, PL>(p, B, s, name);
            case 3: return run_colhist4p_u8_gm<T, 8, 3, PL>(p, B, s, name);
            case 5: return run_colhist4p_u8_gm<T, 8, 5, PL>(p, B, s, name);
            default: return run_colhist4p_u8_gm<T, 8, 7, PL>(p, B, s, name);
        }
    }
    if (4 * n <= 255) return n % 4 == 1 ? run_colhist4p_u8_gm<T, 4, 1, PL>(p, B, s, name)
                                        : run_colhist4p_u8_gm<T, 4, 3, PL>(p, B, s, name);
    if (2 * n <= 255) return run_colhist4p_u8_gm<T, 2, 1, PL>(p, B, s, name);
    return run_colhist4_256(p, B, s);  // pair counts would overflow u8
}

int run_colhist4p_256(SlabParams p, int B, cudaStream_t s, int pl) {
    switch (pl) {
        case 3: return run_colhist4p_u8<256, 3>(p, B, s, "k_colhist4p_u8<256,3>");
        case 2: return run_colhist4p_u8<256, 2>(p, B, s, "k_colhist4p_u8<256,2>");
        default: return run_colhist4p_u8<256, 1>(p, B, s, "k_colhist4p_u8<256,1>");
    }
}

}  // namespace mtb
