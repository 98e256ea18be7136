// run_colhist4q.cu -- k_colhist4p_u8 with three pair levels and derived
// level-2 singles (PL = 4) at compile-time window sides n = 33..97
// (r = 16..48, the radii run_colhist.cu sends to it).
#include "run_colhist4p.cuh"

namespace mtb {

// 1 when n is outside the range (MTB status codes are 0 or negative)
int run_colhist4q_fixed(SlabParams p, int B, cudaStream_t s) {
    const int n = 2 * p.radius + 1;
    if (n < 33 || n > 97) return 1;
    return with_fixed_n<33, 97>(n, [&](auto nf) {
        constexpr int NF = decltype(nf)::value, G = carry_free_group(NF);  // even: n <= 127
        if constexpr (NF == 0) {
            return 1;
        } else {
            return run_colhist4p_u8_gm<256, G, NF % G, 4, NF>(p, B, s, "k_colhist4p_u8<256,4>");
        }
    });
}

}  // namespace mtb
