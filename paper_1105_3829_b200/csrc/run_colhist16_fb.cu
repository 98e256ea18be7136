// run_colhist16_fb.cu -- k_colhist16_u16 with compile-time window sides
// n = 29..45 (one translation unit per range: parallel builds).
#include "run_colhist16.cuh"

namespace mtb {

int run_colhist16_fixed_b(SlabParams p, int B, cudaStream_t s, int wk) {
    return run_colhist16_fixed<29, 45>(p, B, s, wk);
}

}  // namespace mtb
