// run_wk16_b.cu -- window-key pass of compact 16-bit data, window sides n = 65..127 (see run_wk16.cuh).
#include "run_wk16.cuh"

namespace mtb {
int run_wk16_fixed_b(SlabParams p, int B, cudaStream_t s) { return run_wk16_fixed<65, 127>(p, B, s); }
}  // namespace mtb
