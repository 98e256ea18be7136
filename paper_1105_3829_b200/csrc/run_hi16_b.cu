// run_hi16_b.cu -- high-byte pair-record pass of the 16-bit candidate-list
// path, window sides n = 65..127 (see run_hi16.cuh).
#include "run_hi16.cuh"

namespace mtb {
int run_hi16_fixed_b(SlabParams p, int B, cudaStream_t s) { return run_hi16_fixed<65, 127>(p, B, s); }
}  // namespace mtb
