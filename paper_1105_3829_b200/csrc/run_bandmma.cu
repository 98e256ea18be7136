// run_bandmma.cu -- launcher of the band-matrix tensor-core kernel
// (kernels_bandmma.cuh).
#include <algorithm>

#include "host.h"
#include "kernels_bandmma.cuh"

namespace mtb {

// the geometry the dispatch relies on: 512-column stripes fit one SM up to r = 72, every radius has a stripe
static_assert(bm_smem(512, 63) <= 227 * 1024 && bm_smem(512, 72) <= 227 * 1024, "512-column stripes at r <= 72");
static_assert(bm_smem(16, 127) <= 227 * 1024, "a stripe at the largest radius");
static_assert(bm_pitch(512, 63) % 64 == 32 && bm_pitch(512, 63) >= 512 + 126 && bm_pitch(512, 63) >= 512 + 32 * bm_nk(63) - 16,
              "plane pitch: bank rule, halo'd columns, last k-tile");

template <int NK, typename PX = uint8_t>
static int run_bandmma_nk(SlabParams p, int B, cudaStream_t s, int TW) {
    constexpr bool HI16 = sizeof(PX) == 2;  // 16-bit coarse keys (never a streaming launch)
    const size_t smem = bm_smem(TW, p.radius);
    const int threads = 32 * (TW / 16);
    auto kern = (p.in_rows && !HI16) ? k_bandmma_u8<NK, !HI16, PX> : k_bandmma_u8<NK, false, PX>;
    if (int rc = set_smem(kern, smem)) return rc;
    const int bx = (p.W + TW - 1) / TW;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (per_sm < 1) per_sm = 1;
    // row slabs: as many CTAs as fit `waves` whole rounds of the resident slots
    // (never one more: a straggler round would double the time)
    const int waves = env_int("MTB_BM_WAVES", 2), rows = p.row_end - p.row_begin;  // (two: evens out data-dependent rows, costs nothing)
    int64_t slabs = (int64_t)sm_count() * per_sm * waves / ((int64_t)bx * B);
    slabs = std::max<int64_t>(1, std::min<int64_t>(slabs, rows));
    int rpc = (int)((rows + slabs - 1) / slabs);
    rpc = std::max(rpc, std::min(rows, p.radius / 2 + 8));  // keep the column build a small share
    p.rows_per_cta = rpc;
    dim3 grid(bx, (rows + rpc - 1) / rpc, B);
    if (!HI16) p.gate = env_int("MTB_BM_DBG", 0);  // (only read by a -DBM_TIMING build)
    kern<<<grid, threads, smem, s>>>(p, TW);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(MTB_E_CUDA, std::string("k_bandmma_u8: ") + cudaGetErrorString(e));
    g_kernel = HI16 ? "k_bandmma_u8<u16 coarse key>" : "k_bandmma_u8";
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return MTB_OK;
}

template <typename PX>
static int run_bandmma_px(SlabParams p, int B, cudaStream_t s) {
    const int r = p.radius;
    // stripe width: the widest multiple of 16 whose planes fit one SM's shared
    // memory with one warp per 16 output columns (at most BM_MAXT threads),
    // then evened out over the stripes the image needs
    const int smem_max = 227 * 1024;
    int twmax = 16;
    for (int tw = 16; tw <= 16 * (BM_MAXT / 32); tw += 16)
        if (bm_smem(tw, r) <= (size_t)smem_max) twmax = tw;
    twmax = std::min(twmax, std::max(16, env_int("MTB_BM_TW", twmax) / 16 * 16));
    const int stripes = (p.W + twmax - 1) / twmax;
    int TW = ((p.W + stripes - 1) / stripes + 15) / 16 * 16;
    if (TW > twmax) TW = twmax;
    switch (bm_nk(r)) {
        case 1: return run_bandmma_nk<1, PX>(p, B, s, TW);
        case 2: return run_bandmma_nk<2, PX>(p, B, s, TW);
        case 3: return run_bandmma_nk<3, PX>(p, B, s, TW);
        case 4: return run_bandmma_nk<4, PX>(p, B, s, TW);
        case 5: return run_bandmma_nk<5, PX>(p, B, s, TW);
        case 6: return run_bandmma_nk<6, PX>(p, B, s, TW);
        case 7: return run_bandmma_nk<7, PX>(p, B, s, TW);
        case 8: return run_bandmma_nk<8, PX>(p, B, s, TW);
        default: return run_bandmma_nk<9, PX>(p, B, s, TW);
    }
}

// 8-bit, 1 <= r <= 127, any rank
int run_bandmma_u8(SlabParams p, int B, cudaStream_t s) { return run_bandmma_px<uint8_t>(p, B, s); }

// 16-bit coarse keys -> (key, rank within it) words (first pass of the candidate-bucket path)
int run_bandmma_hi16(SlabParams p, int B, cudaStream_t s) { return run_bandmma_px<uint16_t>(p, B, s); }

}  // namespace mtb
