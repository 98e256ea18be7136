// run_colhist.cu -- launchers of the 8-bit column-histogram gather kernels
// (kernels_colhist.cuh); see medtree_b200.cu for the dispatch.
#include <algorithm>

#include "host.h"
#include "kernels_colhist.cuh"

namespace mtb {

template <int T, int S, int G, int M, int NF = 0>
static int run_colhist_u8_gm(SlabParams p, int B, cudaStream_t s, const char *name) {
    const ColhistGeom g = colhist_geom(T, S, p.radius);
    const size_t smem = (size_t)g.bytes;
    auto kern = k_colhist_u8<T, S, G, M, NF>;
    if (int rc = set_smem(kern, smem)) return rc;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem);
    if (per_sm < 1) per_sm = 1;
    const int bx = (p.W + g.TW - 1) / g.TW;
    p.rows_per_cta = rows_per_cta(p, bx, B, per_sm);
    dim3 grid(bx, (p.row_end - p.row_begin + p.rows_per_cta - 1) / p.rows_per_cta, B);
    return launch(kern, grid, T, smem, s, p, name);
}

// n is odd, so the tail n mod G is odd for G > 1 and 0 for G = 1
template <int T, int S, int G>
static int run_colhist_u8_g(SlabParams p, int B, cudaStream_t s, const char *name) {
    switch ((2 * p.radius + 1) % G) {
        case 1: return run_colhist_u8_gm<T, S, G, (G > 1 ? 1 : 0)>(p, B, s, name);
        case 3: return run_colhist_u8_gm<T, S, G, (G > 3 ? 3 : 0)>(p, B, s, name);
        case 5: return run_colhist_u8_gm<T, S, G, (G > 5 ? 5 : 0)>(p, B, s, name);
        case 7: return run_colhist_u8_gm<T, S, G, (G > 7 ? 7 : 0)>(p, B, s, name);
        default: return run_colhist_u8_gm<T, S, G, 0>(p, B, s, name);
    }
}

// carry-free group size: G columns of counts <= n sum to <= 255 per u8 lane
template <int T, int S>
static int run_colhist_u8_ts(SlabParams p, int B, cudaStream_t s, const char *name) {
    const int n = 2 * p.radius + 1;
    if (S == 1 && n <= 11) {  // compile-time window side for the radii this kernel serves
        return with_fixed_n<3, 11>(n, [&](auto nf) {
            constexpr int NF = decltype(nf)::value, G = carry_free_group(NF);
            return run_colhist_u8_gm<T, S, G, NF % G, NF>(p, B, s, name);
        });
    }
    if (8 * n <= 255) return run_colhist_u8_g<T, S, 8>(p, B, s, name);
    if (4 * n <= 255) return run_colhist_u8_g<T, S, 4>(p, B, s, name);
    if (2 * n <= 255) return run_colhist_u8_g<T, S, 2>(p, B, s, name);
    return run_colhist_u8_g<T, S, 1>(p, B, s, name);
}

template <int T, int G, int M, int NF = 0>
static int run_colhist4_u8_gm(SlabParams p, int B, cudaStream_t s, const char *name) {
    const size_t smem = (size_t)colhist4_bytes(T, p.radius);
    auto kern = p.in_rows ? k_colhist4_u8<T, G, M, true, NF> : k_colhist4_u8<T, G, M, false, NF>;
    if (int rc = set_smem(kern, smem)) return rc;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem);
    if (per_sm < 1) per_sm = 1;
    const int bx = (p.W + T - 1) / T;
    p.rows_per_cta = rows_per_cta(p, bx, B, per_sm);
    dim3 grid(bx, (p.row_end - p.row_begin + p.rows_per_cta - 1) / p.rows_per_cta, B);
    return launch(kern, grid, T, smem, s, p, name);
}

template <int T, int G>
static int run_colhist4_u8_g(SlabParams p, int B, cudaStream_t s, const char *name) {
    switch ((2 * p.radius + 1) % G) {
        case 1: return run_colhist4_u8_gm<T, G, (G > 1 ? 1 : 0)>(p, B, s, name);
        case 3: return run_colhist4_u8_gm<T, G, (G > 3 ? 3 : 0)>(p, B, s, name);
        case 5: return run_colhist4_u8_gm<T, G, (G > 5 ? 5 : 0)>(p, B, s, name);
        case 7: return run_colhist4_u8_gm<T, G, (G > 7 ? 7 : 0)>(p, B, s, name);
        default: return run_colhist4_u8_gm<T, G, 0>(p, B, s, name);
    }
}

template <int T>
static int run_colhist4_u8(SlabParams p, int B, cudaStream_t s, const char *name) {
    const int n = 2 * p.radius + 1;
    if (n >= 7 && n <= 21) {  // compile-time window side for the radii this kernel may serve (3..10)
        return with_fixed_n<7, 21>(n, [&](auto nf) {
            constexpr int NF = decltype(nf)::value, G = carry_free_group(NF);
            return run_colhist4_u8_gm<T, G, NF % G, NF>(p, B, s, name);
        });
    }
    if (8 * n <= 255) return run_colhist4_u8_g<T, 8>(p, B, s, name);
    if (4 * n <= 255) return run_colhist4_u8_g<T, 4>(p, B, s, name);
    if (2 * n <= 255) return run_colhist4_u8_g<T, 2>(p, B, s, name);
    return run_colhist4_u8_g<T, 1>(p, B, s, name);
}

// radix-4 records, 256 threads (also the pair kernels' wide-window fallback)
int run_colhist4_256(SlabParams p, int B, cudaStream_t s) { return run_colhist4_u8<256>(p, B, s, "k_colhist4_u8<256>"); }

// 8-bit column-histogram gather kernels; the variant by radius is below.
// MTB_CH_VAR forces one.
int run_colhist_u8(SlabParams p, int B, cudaStream_t s) {
    int var = env_int("MTB_CH_VAR", -1);
    if (var < 0) {
        // measured on config 2 with compile-time window sides and atomic
        // record updates (tools/probe.py sweep, DESIGN.md sections 3.1b,
        // 3.3): 16-bin records for r <= 2; from r = 3 radix-4 records with
        // pair records for the three upper levels -- with the level-2
        // single records (var 30) up to r = 16, derived from level 3
        // (var 32, PL = 4: two CTAs per SM up to r = 48) above.  Plain
        // radix-4 (var 12/13) trails by 3-15% over r = 3..10.
        const int r = p.radius, lim = 113 * 1024;
        var = r <= 2 ? 0
              : (r <= 16 && colhist4p_bytes(256, r, 3) <= lim) ? 30
              : colhist4q_bytes(256, r, 4) <= lim ? 32
              : colhist4p_bytes(256, r, 2) <= lim ? 31
                                                   : 12;
    }
    switch (var) {
        case 0: return run_colhist_u8_ts<128, 1>(p, B, s, "k_colhist_u8<128,1>");
        case 2: return run_colhist_u8_ts<128, 2>(p, B, s, "k_colhist_u8<128,2>");
        case 30: return run_colhist4p_256(p, B, s, 3);
        case 31: return run_colhist4p_256(p, B, s, 2);
        case 34: return run_colhist4p_256(p, B, s, 1);
        case 32: return run_colhist4p_256(p, B, s, 4);
        case 13: return run_colhist4_u8<128>(p, B, s, "k_colhist4_u8<128>");
        default: return run_colhist4_u8<256>(p, B, s, "k_colhist4_u8<256>");
    }
}

}  // namespace mtb
