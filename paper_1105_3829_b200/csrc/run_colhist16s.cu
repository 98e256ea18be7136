// run_colhist16s.cu -- launcher of k_colhist16s_u16 (16-bit, widely spread
// data: high byte from column records, low byte from sorted columns).
#include <algorithm>

#include "host.h"
#include "kernels_colhist.cuh"

namespace mtb {

template <int T, int G, int M, int NF = 0>
static int run_colhist16s_u16_gm(SlabParams p, int B, cudaStream_t s) {
    const int n = 2 * p.radius + 1, NCOL = T + 2 * p.radius;
    const size_t smem = (size_t)colhist4_bytes(T, p.radius) + 16 * T * 2 + ((size_t)(n * T + 15) & ~(size_t)15) +
                        ((size_t)NCOL * n + 7) / 8 * 16 + (size_t)CH16S_CMAX * T;
    if (smem > 220 * 1024) return run_colhist16_u16(p, B, s, 0);  // sorted columns too large: two-phase kernel
    auto kern = k_colhist16s_u16<T, G, M, NF>;
    if (int rc = set_smem(kern, smem)) return rc;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem);
    if (per_sm < 1) per_sm = 1;
    const int bx = (p.W + T - 1) / T;
    p.rows_per_cta = rows_per_cta(p, bx, B, per_sm);
    if (p.rows_per_cta < 2 * n) p.rows_per_cta = std::min(2 * n, p.row_end - p.row_begin);
    dim3 grid(bx, (p.row_end - p.row_begin + p.rows_per_cta - 1) / p.rows_per_cta, B);
    return launch(kern, grid, T, smem, s, p, "k_colhist16s_u16");
}

template <int T, int G>
static int run_colhist16s_u16_g(SlabParams p, int B, cudaStream_t s) {
    switch ((2 * p.radius + 1) % G) {
        case 1: return run_colhist16s_u16_gm<T, G, (G > 1 ? 1 : 0)>(p, B, s);
        case 3: return run_colhist16s_u16_gm<T, G, (G > 3 ? 3 : 0)>(p, B, s);
        case 5: return run_colhist16s_u16_gm<T, G, (G > 5 ? 5 : 0)>(p, B, s);
        case 7: return run_colhist16s_u16_gm<T, G, (G > 7 ? 7 : 0)>(p, B, s);
        default: return run_colhist16s_u16_gm<T, G, 0>(p, B, s);
    }
}

// widely spread 16-bit data; sorted columns need n <= 255 (u8 run starts)
int run_colhist16s_u16(SlabParams p, int B, cudaStream_t s) {
    const int n = 2 * p.radius + 1;
    if (n >= 5 && n <= 33) {  // compile-time window side for the radii this kernel serves (r <= 16)
        return with_fixed_n<5, 33>(n, [&](auto nf) {
            constexpr int NF = decltype(nf)::value, G = carry_free_group(NF);
            return run_colhist16s_u16_gm<128, G, NF % G, NF>(p, B, s);
        });
    }
    if (8 * n <= 255) return run_colhist16s_u16_g<128, 8>(p, B, s);
    if (4 * n <= 255) return run_colhist16s_u16_g<128, 4>(p, B, s);
    if (2 * n <= 255) return run_colhist16s_u16_g<128, 2>(p, B, s);
    return run_colhist16s_u16_g<128, 1>(p, B, s);
}

}  // namespace mtb
