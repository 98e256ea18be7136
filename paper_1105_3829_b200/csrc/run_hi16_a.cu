// run_hi16_a.cu -- high-byte pair-record pass of the 16-bit candidate-list
// path, window sides n = 7..63 (see run_hi16.cuh).
#include "run_hi16.cuh"

namespace mtb {
int run_hi16_fixed_a(SlabParams p, int B, cudaStream_t s) { return run_hi16_fixed<7, 63>(p, B, s); }
}  // namespace mtb
