// run_lowsel16.cu -- 16-bit, widely spread data: the candidate-list path.
//   pass 1  k_colhist4p_u8<..., uint16_t>   high byte H and rank k' within it, per pixel
//   pass 2  k_lowsel_u16                    low byte from a per-block candidate list
//   pass 3  k_colhist16_u16 (todo-gated)    the blocks pass 2 flagged (locally compact data)
// All three on the caller's stream; the scratch planes come from the
// stream-ordered pool.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "host.h"
#include "kernels_lowsel16.cuh"

namespace mtb {

int run_hi16_fixed_a(SlabParams p, int B, cudaStream_t s);
int run_hi16_fixed_b(SlabParams p, int B, cudaStream_t s);
int run_wk16_fixed_a(SlabParams p, int B, cudaStream_t s);
int run_wk16_fixed_b(SlabParams p, int B, cudaStream_t s);

bool lowsel16_applies(const SlabParams &p) {
    return !p.in_rows && p.radius >= LOWSEL_MIN_R && p.radius <= LOWSEL_MAX_R;
}

template <int PH, int NI>
static int launch_lowsel_ni(const SlabParams &p, int B, cudaStream_t s, const uint32_t *hk) {
    // a CTA takes `seg` vertically adjacent block rows.  One block row per CTA schedules best
    // (config 3 r = 31: 1.38 / 1.43 / 1.57 ms at seg = 1 / 2 / 4: the blocks' costs vary); larger
    // launches take more, so that a gated launch with nothing to do (compact data, device-selected
    // dispatch) stays at <= 16 K CTAs to retire
    const int gx = (p.todo_nbx + LS_WARPS - 1) / LS_WARPS;
    const int64_t want = 16384;
    const int seg = std::max(1, env_int("MTB_LS_SEG", (int)(((int64_t)gx * p.todo_nby * B + want - 1) / want)));
    dim3 grid(gx, (p.todo_nby + seg - 1) / seg, B);
    k_lowsel_u16<PH, NI><<<grid, 32 * LS_WARPS, 0, s>>>(p, hk, seg);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(MTB_E_CUDA, std::string("k_lowsel_u16: ") + cudaGetErrorString(e));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return MTB_OK;
}

template <int PH>
static int launch_lowsel(const SlabParams &p, int B, cudaStream_t s, const uint32_t *hk) {
    switch ((32 + 2 * p.radius + 31) / 32) {  // column steps of the scan
        case 2: return launch_lowsel_ni<PH, 2>(p, B, s, hk);
        case 3: return launch_lowsel_ni<PH, 3>(p, B, s, hk);
        case 4: return launch_lowsel_ni<PH, 4>(p, B, s, hk);
        default: return launch_lowsel_ni<PH, 5>(p, B, s, hk);
    }
}

int run_lowsel16_u16(SlabParams p, int B, cudaStream_t s) {
    if (!lowsel16_applies(p)) return run_colhist16_u16(p, B, s, 0);
    const int rows = p.row_end - p.row_begin;
    // block height: taller blocks share the scan among more pixels but widen the blocks' key ranges
    // and lengthen the buckets.  16 rows (config 3, 8 / 16 / 24 / 32 rows: r = 7 0.67 / 0.62 / 0.62 /
    // 0.69 ms, r = 15 0.87 / 0.76 / 0.77 / 0.86, r = 31 1.39 / 1.20 / 1.21 / 1.26).  Heights above 8
    // run the variant that keeps the block's (H, k') words out of registers.
    const int ph_env = env_int("MTB_LS_PH", 16);
    const int PH = ph_env > 8 ? std::min(ph_env, 64) : (ph_env >= 8 ? 8 : 4);
    p.todo_bh = PH;
    p.todo_nbx = (p.W + 31) / 32;
    p.todo_nby = (rows + PH - 1) / PH;
    const size_t hk_bytes = (size_t)rows * p.W * B * sizeof(uint32_t);
    const size_t flag_bytes = (size_t)p.todo_nbx * p.todo_nby * B;
    unsigned char *scratch = nullptr;
    keep_pool_memory();
    if (cudaMallocAsync(reinterpret_cast<void **>(&scratch), hk_bytes + flag_bytes, s) != cudaSuccess) {
        // no room for the 4-byte-per-pixel plane: the two-phase kernel (1 byte per pixel) instead
        cudaGetLastError();
        p.todo = nullptr;
        return run_colhist16_u16(p, B, s, 0);
    }
    uint32_t *hk = reinterpret_cast<uint32_t *>(scratch);
    p.todo = scratch + hk_bytes;
    if (cudaMemsetAsync(p.todo, 0, flag_bytes, s) != cudaSuccess) {
        cudaFreeAsync(scratch, s);
        return fail(MTB_E_CUDA, "k_lowsel_u16: clearing the block flags failed");
    }

    SlabParams a = p;  // pass 1 writes H << 16 | k' words
    a.dst = hk;
    a.dst_pitch = p.W;
    a.dst_img_stride = (int64_t)rows * p.W;
    a.lut = nullptr;
    a.todo = nullptr;
    // pass 1: pair records up to r = 30, band-matrix products on the tensor cores from r = 31
    // (config 3, whole path, pair / mma: r = 23 1.14 / 1.17 ms, r = 31 1.33 / 1.31, r = 47 2.23 /
    // 1.90, r = 63 3.98 / 2.37; MTB_LS_HI=pair|mma forces)
    const std::string hi = getenv("MTB_LS_HI") ? getenv("MTB_LS_HI") : "";
    int rc = 1;
    if (hi == "mma" || (hi.empty() && p.radius >= 31)) {
        rc = run_bandmma_hi16(a, B, s);
    } else {
        rc = run_hi16_fixed_a(a, B, s);
        if (rc == 1) rc = run_hi16_fixed_b(a, B, s);
    }
    if (rc == 1) rc = fail(MTB_E_INVAL, "k_lowsel_u16: radius outside the candidate-list path");
    if (!rc) rc = PH > 8 ? launch_lowsel<0>(p, B, s, hk) : (PH == 8 ? launch_lowsel<8>(p, B, s, hk) : launch_lowsel<4>(p, B, s, hk));
    // pass 3: flagged blocks are locally compact, where the window-keyed sweep pays
    if (!rc) rc = run_colhist16_u16(p, B, s, 1);
    cudaFreeAsync(scratch, s);
    if (!rc) g_kernel = "k_lowsel_u16";
    return rc;
}

// Compact, peaked 16-bit data (config 4): pass 1 the pair-record kernel in window-key mode (one
// 8-bit problem per tile), pass 2 the two-phase kernel on the tiles holding a block pass 1 flagged.
int run_wk16_u16(SlabParams p, int B, cudaStream_t s) {
    if (!lowsel16_applies(p)) return run_colhist16_u16(p, B, s, 1);
    const int rows = p.row_end - p.row_begin;
    p.todo_bh = 8;
    p.todo_nbx = (p.W + 31) / 32;
    p.todo_nby = (rows + p.todo_bh - 1) / p.todo_bh;
    const size_t flag_bytes = (size_t)p.todo_nbx * p.todo_nby * B;
    keep_pool_memory();
    if (cudaMallocAsync(reinterpret_cast<void **>(&p.todo), flag_bytes, s) != cudaSuccess)
        return fail(MTB_E_CUDA, "window-key pass: scratch allocation failed");
    if (cudaMemsetAsync(p.todo, 0, flag_bytes, s) != cudaSuccess) {
        cudaFreeAsync(p.todo, s);
        return fail(MTB_E_CUDA, "window-key pass: clearing the block flags failed");
    }
    int rc = run_wk16_fixed_a(p, B, s);
    if (rc == 1) rc = run_wk16_fixed_b(p, B, s);
    if (rc == 1) rc = fail(MTB_E_INVAL, "window-key pass: radius outside its range");
    if (!rc) rc = run_colhist16_u16(p, B, s, 1);
    cudaFreeAsync(p.todo, s);
    if (!rc) g_kernel = "k_colhist4p_u8<256,u16 window key>";
    return rc;
}

}  // namespace mtb
