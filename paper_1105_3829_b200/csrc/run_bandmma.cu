// run_bandmma.cu -- launcher of the band-matrix tensor-core kernel
// (kernels_bandmma.cuh).
#include <algorithm>

#include "host.h"
#include "kernels_bandmma.cuh"

namespace mtb {

template <int NK, int NT>
static int run_bandmma_nk(SlabParams p, int B, cudaStream_t s, int TW, int warps) {
    const size_t smem = bm_smem(TW, p.radius, warps, NT);
    auto kern = p.in_rows ? k_bandmma_u8<NK, NT, true> : k_bandmma_u8<NK, NT, false>;
    if (int rc = set_smem(kern, smem)) return rc;
    const int bx = (p.W + TW - 1) / TW;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, warps * 32, smem);
    if (per_sm < 1) per_sm = 1;
    // row slabs: as many CTAs as fit `waves` whole rounds of the resident slots
    // (never one more: a straggler round would double the time)
    const int waves = env_int("MTB_BM_WAVES", 1), rows = p.row_end - p.row_begin;
    int64_t slabs = (int64_t)sm_count() * per_sm * waves / ((int64_t)bx * B);
    slabs = std::max<int64_t>(1, std::min<int64_t>(slabs, rows));
    int rpc = (int)((rows + slabs - 1) / slabs);
    rpc = std::max(rpc, std::min(rows, p.radius / 2 + 8));  // keep the column build a small share
    p.rows_per_cta = rpc;
    dim3 grid(bx, (p.row_end - p.row_begin + p.rows_per_cta - 1) / p.rows_per_cta, B);
    p.gate = env_int("MTB_BM_DBG", 0);
    kern<<<grid, warps * 32, smem, s>>>(p, TW);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(MTB_E_CUDA, std::string("k_bandmma_u8: ") + cudaGetErrorString(e));
    g_kernel = NT == 4 ? "k_bandmma_u8<32>" : "k_bandmma_u8<48>";
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return MTB_OK;
}

template <int NT>
static int run_bandmma_nt(SlabParams p, int B, cudaStream_t s) {
    const int r = p.radius;
    // stripe width: the widest multiple of 64 whose planes fit one SM's shared
    // memory with one warp per 32 output columns (at most BM_MAXT threads),
    // then evened out over the stripes the image needs
    const int smem_max = 227 * 1024;
    int twmax = 64;
    for (int tw = 64; tw <= 32 * (BM_MAXT / 32); tw += 64)
        if (bm_smem(tw, r, tw / 32, NT) <= (size_t)smem_max) twmax = tw;
    twmax = std::min(twmax, std::max(64, env_int("MTB_BM_TW", twmax) / 64 * 64));
    const int stripes = (p.W + twmax - 1) / twmax;
    int TW = ((p.W + stripes - 1) / stripes + 63) / 64 * 64;
    if (TW > twmax) TW = twmax;
    const int warps = TW / 32;
    switch (bm_nk(r)) {
        case 1: return run_bandmma_nk<1, NT>(p, B, s, TW, warps);
        case 2: return run_bandmma_nk<2, NT>(p, B, s, TW, warps);
        case 3: return run_bandmma_nk<3, NT>(p, B, s, TW, warps);
        case 4: return run_bandmma_nk<4, NT>(p, B, s, TW, warps);
        case 5: return run_bandmma_nk<5, NT>(p, B, s, TW, warps);
        default: break;
    }
    if constexpr (NT == 4) {
        switch (bm_nk(r)) {
            case 6: return run_bandmma_nk<6, 4>(p, B, s, TW, warps);
            case 7: return run_bandmma_nk<7, 4>(p, B, s, TW, warps);
            case 8: return run_bandmma_nk<8, 4>(p, B, s, TW, warps);
            default: return run_bandmma_nk<9, 4>(p, B, s, TW, warps);
        }
    }
    return fail(MTB_E_INVAL, "k_bandmma_u8: radius outside the 48-plane variant");
}

// 8-bit, 1 <= r <= 127, any rank.  Keyed window: 48 planes below r = 48 (the
// median of a smaller window moves faster from row to row), 32 above.
int run_bandmma_u8(SlabParams p, int B, cudaStream_t s) {
    const int nt = env_int("MTB_BM_NT", p.radius >= 48 ? 4 : 6);
    if (nt == 6 && bm_nk(p.radius) <= 5) return run_bandmma_nt<6>(p, B, s);
    return run_bandmma_nt<4>(p, B, s);
}

}  // namespace mtb
