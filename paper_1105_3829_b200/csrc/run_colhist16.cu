// run_colhist16.cu -- launchers of the 16-bit column-histogram kernels
// (k_colhist16_u16 two-phase, k_colhist16s_u16 sorted-column low byte).
#include <algorithm>

#include "host.h"
#include "kernels_colhist.cuh"

namespace mtb {

template <int T, int G, int M, int PL>
static int run_colhist16_u16_gm(SlabParams p, int B, cudaStream_t s, bool wk) {
    // window-keyed first sweep (compact data); MTB_CH16_WK=0/1 forces
    wk = env_int("MTB_CH16_WK", wk ? 1 : 0) != 0;
    const int ncp = PL > 0 ? colhist4p_ncolp(T, p.radius) : ch4_stride(T + 2 * p.radius);
    const size_t smem = (PL > 0 ? (size_t)colhist4p_bytes(T, p.radius, PL) : (size_t)colhist4_bytes(T, p.radius)) +
                        (size_t)ncp * 4 + (2 * 256 + 2) * sizeof(int);
    auto kern = k_colhist16_u16<T, G, M, PL>;
    if (int rc = set_smem(kern, smem)) return rc;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem);
    if (per_sm < 1) per_sm = 1;
    const int bx = (p.W + T - 1) / T;
    p.rows_per_cta = rows_per_cta(p, bx, B, per_sm);
    dim3 grid(bx, (p.row_end - p.row_begin + p.rows_per_cta - 1) / p.rows_per_cta, B);
    // per-pixel high-byte plane (stream-ordered pool allocation, kept cached)
    uint8_t *hplane = nullptr;
    keep_pool_memory();
    const size_t hbytes = (size_t)(p.row_end - p.row_begin) * p.W * B;
    if (cudaMallocAsync(reinterpret_cast<void **>(&hplane), hbytes, s) != cudaSuccess)
        return fail(MTB_E_CUDA, "k_colhist16_u16: scratch allocation failed");
    if (int rc = set_smem(kern, smem)) return rc;
    kern<<<grid, T, smem, s>>>(p, hplane, wk);
    cudaError_t e = cudaGetLastError();
    cudaFreeAsync(hplane, s);
    if (e != cudaSuccess) return fail(MTB_E_CUDA, std::string("k_colhist16_u16: ") + cudaGetErrorString(e));
    g_kernel = "k_colhist16_u16";
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return MTB_OK;
}

template <int T, int G, int PL>
static int run_colhist16_u16_g(SlabParams p, int B, cudaStream_t s, bool wk) {
    switch ((2 * p.radius + 1) % G) {
        case 1: return run_colhist16_u16_gm<T, G, (G > 1 ? 1 : 0), PL>(p, B, s, wk);
        case 3: return run_colhist16_u16_gm<T, G, (G > 3 ? 3 : 0), PL>(p, B, s, wk);
        case 5: return run_colhist16_u16_gm<T, G, (G > 5 ? 5 : 0), PL>(p, B, s, wk);
        case 7: return run_colhist16_u16_gm<T, G, (G > 7 ? 7 : 0), PL>(p, B, s, wk);
        default: return run_colhist16_u16_gm<T, G, 0, PL>(p, B, s, wk);
    }
}

int run_colhist16_u16(SlabParams p, int B, cudaStream_t s, bool wk) {
    const int n = 2 * p.radius + 1;
    // pair records (upper levels) where two 256-thread CTAs per SM still fit
    const int lim = 113 * 1024 - (2 * 256 + 2) * (int)sizeof(int) - ch4_stride(256 + 2 * p.radius) * 4;
    const int pl = env_int("MTB_CH16_PL", colhist4p_bytes(256, p.radius, 3) <= lim ? 3
                                          : colhist4p_bytes(256, p.radius, 2) <= lim ? 2 : 0);
    if (8 * n <= 255) {
        if (pl == 3) return run_colhist16_u16_g<256, 8, 3>(p, B, s, wk);
        if (pl == 2) return run_colhist16_u16_g<256, 8, 2>(p, B, s, wk);
        return run_colhist16_u16_g<256, 8, 0>(p, B, s, wk);
    }
    if (4 * n <= 255) return pl >= 2 ? run_colhist16_u16_g<256, 4, 2>(p, B, s, wk) : run_colhist16_u16_g<256, 4, 0>(p, B, s, wk);
    if (2 * n <= 255) return run_colhist16_u16_g<256, 2, 0>(p, B, s, wk);
    return run_colhist16_u16_g<256, 1, 0>(p, B, s, wk);
}


}  // namespace mtb
