// run_colhist4p.cu -- launchers of the radix-4 column-histogram kernel with
// pair records (k_colhist4p_u8); see run_colhist.cu for the dispatch.
#include <algorithm>

#include "run_colhist4p.cuh"

namespace mtb {

int run_colhist4q_fixed(SlabParams p, int B, cudaStream_t s);

// pair records (G even: n <= 127); PL pair levels
template <int T, int PL>
static int run_colhist4p_u8(SlabParams p, int B, cudaStream_t s, const char *name) {
    const int n = 2 * p.radius + 1;
    // compile-time window side for the radii each variant serves (PL = 3:
    // r = 2..18, PL = 4: r = 16..48; run_colhist.cu)
    if (PL == 4 && T == 256 && n >= 33 && n <= 97) {  // compile-time window sides r = 16..48 (run_colhist4q.cu)
        const int rc = run_colhist4q_fixed(p, B, s);
        if (rc != 1) return rc;
    }
    if (PL == 3 && n >= 5 && n <= 37)
        return with_fixed_n<5, 37>(n, [&](auto nf) {
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
        case 4: return run_colhist4p_u8<256, 4>(p, B, s, "k_colhist4p_u8<256,4>");
        case 3: return run_colhist4p_u8<256, 3>(p, B, s, "k_colhist4p_u8<256,3>");
        case 2: return run_colhist4p_u8<256, 2>(p, B, s, "k_colhist4p_u8<256,2>");
        default: return run_colhist4p_u8<256, 1>(p, B, s, "k_colhist4p_u8<256,1>");
    }
}

}  // namespace mtb
