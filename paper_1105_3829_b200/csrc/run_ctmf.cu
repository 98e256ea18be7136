// run_ctmf.cu -- launcher of the CTMF tile kernel (kernels_ctmf.cuh).
#include "host.h"
#include "kernels_ctmf.cuh"

namespace mtb {

// use_pre: snapshots from k_ctmf_pre_u8 (the PRE kernel: 4 CTAs per SM);
// if their workspace cannot be allocated, the per-tile scans instead
template <int S, int MF = -1>
static int run_ctmf_u8_s(SlabParams p, int B, cudaStream_t s, bool use_pre) {
    const CtmfGeom g = ctmf_geom(S, p.radius, use_pre ? 2 : CT_STAGE_ROWS);
    const int rows = p.row_end - p.row_begin;
    const int tiles_x = (p.W + g.TW - 1) / g.TW;
    const size_t smem = (size_t)g.warp_bytes * CT_WARPS;
    const bool ctb4 = use_pre && p.radius >= env_int("MTB_CT_CTB4_R", 80);
    auto kern = ctb4 ? k_ctmf_u8<S, MF, true, 4> : (use_pre ? k_ctmf_u8<S, MF, true, 3> : k_ctmf_u8<S, MF, false, 3>);
    if (int rc = set_smem(kern, smem)) return rc;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, CT_WARPS * 32, smem);
    if (per_sm < 1) per_sm = 1;
    // Tile height: near max(24, n/3) rows, adjusted so that the tiles divide
    // evenly over the resident warps (k full rounds, no ragged last round).
    const int n = 2 * p.radius + 1;
    const int64_t warps = (int64_t)sm_count() * per_sm * CT_WARPS;
    const double per_stripe = (double)warps / ((double)tiles_x * B);  // warps per column stripe
    // (with up-front snapshots a tile's init is two loads per column: from
    // n >= 97 shorter tiles balance better -- r = 63 0.82 -> 0.79 ms)
    const int target = (use_pre && n >= 97) ? 24 : (n / 3 > 24 ? n / 3 : 24);
    int th;
    if (per_stripe >= 1.0) {
        int k = (int)((double)rows / (target * per_stripe) + 0.5);
        if (k < 1) k = 1;
        th = (int)((rows + (int64_t)(k * per_stripe) - 1) / (int64_t)(k * per_stripe));
    } else {
        th = target;
    }
    if (th < 8) th = 8 < rows ? 8 : rows;
    if (th > rows) th = rows;
    p.rows_per_cta = th;
    const int tiles_y = (rows + th - 1) / th;
    const int tiles = tiles_x * tiles_y;
    // persistent grid: as many CTAs as are resident at once (per image)
    int ctas = (tiles + CT_WARPS - 1) / CT_WARPS;
    const int resident = (int)((sm_count() * per_sm + B - 1) / B);
    if (ctas > resident) ctas = resident > 0 ? resident : 1;
    dim3 grid(ctas, 1, B);
    // span snapshots of every tile row, computed up front (k_ctmf_pre_u8);
    // MTB_CT_PRE=0: per-warp snapshot scans inside the tiles instead
    uint4 *pre = nullptr;
    if (use_pre) {
        keep_pool_memory();
        const size_t pre_bytes = (size_t)B * tiles_y * p.W * 17 * sizeof(uint4);
        if (cudaMallocAsync(reinterpret_cast<void **>(&pre), pre_bytes, s) != cudaSuccess) {
            cudaGetLastError();
            return run_ctmf_u8_s<S, MF>(p, B, s, false);
        } else {
            const int seg = 2;  // tile rows per pre-pass thread segment
            dim3 pg((p.W + CTP_T - 1) / CTP_T, (tiles_y + seg - 1) / seg, B);
            k_ctmf_pre_u8<CTP_T><<<pg, CTP_T, 0, s>>>(p, tiles_y, seg, pre);
            g_launches.fetch_add(1, std::memory_order_relaxed);
        }
    }
    // per-tile column snapshots (stream-ordered pool allocation, kept cached)
    uint8_t *snap = nullptr;
    const size_t snap_bytes = (size_t)ctas * CT_WARPS * B * ((((size_t)g.NCP * 18 + 15) & ~(size_t)15) + (size_t)g.NCP * 256);
    if (!pre) {
        keep_pool_memory();
        if (cudaMallocAsync(reinterpret_cast<void **>(&snap), snap_bytes, s) != cudaSuccess) {
            cudaGetLastError();
            snap = nullptr;  // fall back to rescanning the spans
        }
    }
    kern<<<grid, CT_WARPS * 32, smem, s>>>(p, tiles_x, tiles_y, snap, 1, pre);
    cudaError_t e = cudaGetLastError();
    if (snap) cudaFreeAsync(snap, s);
    if (pre) cudaFreeAsync(pre, s);
    if (e != cudaSuccess) return fail(MTB_E_CUDA, std::string("k_ctmf_u8: ") + cudaGetErrorString(e));
    g_kernel = S == 8 ? "k_ctmf_u8<8>" : "k_ctmf_u8<16>";
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return MTB_OK;
}

int run_ctmf_u8(SlabParams p, int B, cudaStream_t s) {
    // MTB_CT_PRE=0: per-tile snapshot scans instead of the up-front pre-pass
    const bool pre = env_int("MTB_CT_PRE", 1) != 0;
    switch ((2 * p.radius + 1) % 8) {  // n mod 8 as a compile-time constant (n odd)
        case 1: return run_ctmf_u8_s<8, 1>(p, B, s, pre);
        case 3: return run_ctmf_u8_s<8, 3>(p, B, s, pre);
        case 5: return run_ctmf_u8_s<8, 5>(p, B, s, pre);
        default: return run_ctmf_u8_s<8, 7>(p, B, s, pre);
    }
}


}  // namespace mtb
