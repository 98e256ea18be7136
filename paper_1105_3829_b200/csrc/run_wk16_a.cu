// run_wk16_a.cu -- window-key pass of compact 16-bit data, window sides n = 7..63 (see run_wk16.cuh).
#include "run_wk16.cuh"

namespace mtb {
int run_wk16_fixed_a(SlabParams p, int B, cudaStream_t s) { return run_wk16_fixed<7, 63>(p, B, s); }
}  // namespace mtb
