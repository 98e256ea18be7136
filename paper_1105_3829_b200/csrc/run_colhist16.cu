// run_colhist16.cu -- launchers of the 16-bit column-histogram kernels
// (k_colhist16_u16 two-phase, k_colhist16s_u16 sorted-column low byte).
#include "run_colhist16.cuh"

namespace mtb {

template <int T, int G, int PL>
static int run_colhist16_u16_g(SlabParams p, int B, cudaStream_t s, int wk) {
    switch ((2 * p.radius + 1) % G) {
        case 1: return run_colhist16_u16_gm<T, G, (G > 1 ? 1 : 0), PL>(p, B, s, wk);
        case 3: return run_colhist16_u16_gm<T, G, (G > 3 ? 3 : 0), PL>(p, B, s, wk);
        case 5: return run_colhist16_u16_gm<T, G, (G > 5 ? 5 : 0), PL>(p, B, s, wk);
        case 7: return run_colhist16_u16_gm<T, G, (G > 7 ? 7 : 0), PL>(p, B, s, wk);
        default: return run_colhist16_u16_gm<T, G, 0, PL>(p, B, s, wk);
    }
}

int run_colhist16_u16(SlabParams p, int B, cudaStream_t s, int wk) {
    const int n = 2 * p.radius + 1;
    {  // compile-time window sides r = 3..31 (run_colhist16_f*.cu)
        int rc = run_colhist16_fixed_a(p, B, s, wk);
        if (rc == NOT_COVERED) rc = run_colhist16_fixed_b(p, B, s, wk);
        if (rc == NOT_COVERED) rc = run_colhist16_fixed_c(p, B, s, wk);
        if (rc != NOT_COVERED) return rc;
    }
    const int pl = ch16_pair_levels(p.radius, wk == 1);
    if (8 * n <= 255) {
        if (pl == 3) return run_colhist16_u16_g<256, 8, 3>(p, B, s, wk);
        if (pl == 4) return run_colhist16_u16_g<256, 8, 4>(p, B, s, wk);
        if (pl == 2) return run_colhist16_u16_g<256, 8, 2>(p, B, s, wk);
        return run_colhist16_u16_g<256, 8, 0>(p, B, s, wk);
    }
    if (4 * n <= 255)
        return pl == 4 ? run_colhist16_u16_g<256, 4, 4>(p, B, s, wk)
                       : (pl >= 2 ? run_colhist16_u16_g<256, 4, 2>(p, B, s, wk) : run_colhist16_u16_g<256, 4, 0>(p, B, s, wk));
    if (2 * n <= 255) return run_colhist16_u16_g<256, 2, 0>(p, B, s, wk);
    return run_colhist16_u16_g<256, 1, 0>(p, B, s, wk);
}


}  // namespace mtb
