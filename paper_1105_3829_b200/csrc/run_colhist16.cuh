// run_colhist16.cuh -- launcher template of the two-phase 16-bit kernel
// (k_colhist16_u16), shared by run_colhist16.cu (runtime window side and
// dispatch) and run_colhist16_f*.cu (compile-time window sides, split
// across translation units so they compile in parallel).
#pragma once
#include <algorithm>

#include "host.h"
#include "kernels_colhist.cuh"

namespace mtb {

template <int T, int G, int M, int PL, int NF = 0>
inline int run_colhist16_u16_gm(SlabParams p, int B, cudaStream_t s, int wk) {
    // window-keyed first sweep (compact data); MTB_CH16_WK=0/1 forces
    wk = env_int("MTB_CH16_WK", wk);
    const int ncp = PL > 0 ? colhist4p_ncolp(T, p.radius) : ch4_stride(T + 2 * p.radius);
    const size_t smem = (PL > 0 ? (size_t)colhist4q_bytes(T, p.radius, PL) : (size_t)colhist4_bytes(T, p.radius)) +
                        (size_t)ncp * 4 + (2 * 256 + 2) * sizeof(int);
    auto kern = k_colhist16_u16<T, G, M, PL, NF>;
    if (int rc = set_smem(kern, smem)) return rc;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem);
    if (per_sm < 1) per_sm = 1;
    const int bx = (p.W + T - 1) / T;
    // four waves of shorter slabs: the tiles' phase-B / window-keyed work
    // varies with the data, and shorter slabs balance it (config 4 r = 15
    // 2.53 -> 1.92 ms, r = 31 3.73 -> 2.83; config 3 r = 31 8.3 -> 6.8)
    p.rows_per_cta = rows_per_cta(p, bx, B, per_sm, 4);
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

// pair-record levels where two 256-thread CTAs per SM still fit (the
// window-keyed sweep's per-column word and the H bookkeeping included).
// allow4: three pair levels with derived level-2 singles (PL = 4) -- for
// the window-keyed sweep on compact data (one or two sweeps per tile:
// config 4 r = 31 3.84 -> 3.72 ms); on spread data the per-H phase-B
// sweeps (~10 per tile) each re-derive the level-2 pairs, and PL = 2 stays
// faster (config 3 r = 31 8.31 against 9.66 ms).
constexpr int ch16_pair_levels(int r, bool allow4 = false) {
    const int lim = 113 * 1024 - (2 * 256 + 2) * (int)sizeof(int) - ch4_stride(256 + 2 * r) * 4;
    return colhist4p_bytes(256, r, 3) <= lim                 ? 3
           : (allow4 && colhist4q_bytes(256, r, 4) <= lim) ? 4
           : colhist4p_bytes(256, r, 2) <= lim              ? 2
                                                             : 0;
}

// compile-time window sides NLO..NHI (odd); NOT_COVERED when n is outside
constexpr int NOT_COVERED = 1;  // (MTB status codes are 0 or negative)
template <int NLO, int NHI>
inline int run_colhist16_fixed(SlabParams p, int B, cudaStream_t s, int wk) {
    const int n = 2 * p.radius + 1;
    if (n < NLO || n > NHI) return NOT_COVERED;
    return with_fixed_n<NLO, NHI>(n, [&](auto nf) {
        constexpr int NF = decltype(nf)::value;
        if constexpr (NF == 0) {
            return NOT_COVERED;
        } else {
            constexpr int G = carry_free_group(NF);
            constexpr int pl = ch16_pair_levels(NF / 2), pl4 = ch16_pair_levels(NF / 2, true);
            constexpr int PL = G == 8 ? pl : (G == 4 && pl >= 2 ? 2 : 0);
            constexpr int PL4 = G == 8 ? pl4 : (G == 4 && pl4 >= 2 ? (pl4 == 4 ? 4 : 2) : 0);
            if constexpr (PL4 != PL) {
                if (wk == 1) return run_colhist16_u16_gm<256, G, NF % G, PL4, NF>(p, B, s, wk);
            }
            return run_colhist16_u16_gm<256, G, NF % G, PL, NF>(p, B, s, wk);
        }
    });
}

}  // namespace mtb
