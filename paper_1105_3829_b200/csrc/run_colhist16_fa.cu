// run_colhist16_fa.cu -- k_colhist16_u16 with compile-time window sides
// n = 7..27 (one translation unit per range: parallel builds).
#include "run_colhist16.cuh"

namespace mtb {

int run_colhist16_fixed_a(SlabParams p, int B, cudaStream_t s, int wk) {
    return run_colhist16_fixed<7, 27>(p, B, s, wk);
}

}  // namespace mtb
