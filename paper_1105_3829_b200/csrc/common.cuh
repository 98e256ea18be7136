// common.cuh -- shared parameter block and helpers for the rank-filter kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mtb {

// One launch = one slab (rows [row_begin,row_end) of a global H x W image)
// for each of gridDim.z images.  See include/medtree_b200.h for semantics.
struct SlabParams {
    const void *src;          // device, element type = pixel type
    int64_t src_pitch;        // elements
    int64_t src_img_stride;   // elements between batch images
    int32_t src_row0;         // global row held in src row 0
    int32_t src_rows;
    void *dst;
    int64_t dst_pitch;
    int64_t dst_img_stride;
    int32_t H, W;             // global image
    int32_t row_begin, row_end;
    int32_t radius;
    uint32_t rank;            // 1-based
    const void *lut;          // optional value map (2^d entries) or nullptr
    int32_t rows_per_cta;     // slab height handled by one CTA row
    // streaming mode (host-buffer path, mtb_filter_host): the source rows
    // arrive in chunks while the kernel runs and results leave in chunks.
    // in_rows: number of global rows [0, *in_rows) already copied in;
    // out_px[c]: output pixels of rows [c*out_chunk, (c+1)*out_chunk) done.
    // Both nullptr outside streaming mode.
    const unsigned int *in_rows;
    unsigned int *out_px;
    int32_t out_chunk;
    // set to 1 by a CTA that gave up waiting for its rows (STREAM_TIMEOUT_NS)
    unsigned int *status;
    // 16-bit dispatch by value spread (medtree_b200.cu::run_u16_colhist):
    // spread = device word with the sampled number of distinct high bytes;
    // gate = GATE_WIDE / GATE_COMPACT: the kernel exits at once unless the
    // data is widely spread / compact (two launches, one does the work).
    const int *spread;
    int32_t gate;
    // candidate-bucket path: the coarse key of a 16-bit pixel is min(v >> s, 255), s = 8 unless the
    // sampled values leave the top bits empty (10- / 12-bit data in 16-bit words): then s follows the
    // occupied range.  Device-selected dispatch: s = spread[1]; host-selected: s = 8 - key_down.
    int32_t key_down;
    // 16-bit candidate-list path (kernels_lowsel16.cuh): one byte per block of
    // 32 x todo_bh output pixels ([image][block row][block column], todo_nbx
    // block columns), non-zero where the list kernel left the block to the
    // two-phase kernel.  With todo set, k_colhist16_u16 only works on tiles
    // that contain such a block.  nullptr elsewhere.
    unsigned char *todo;
    int32_t todo_bh, todo_nbx, todo_nby;
};

constexpr int SPREAD_WIDE = 24;  // > 24 distinct sampled high bytes: widely spread
constexpr int GATE_WIDE = 1, GATE_COMPACT = 2;
constexpr int WK_FROM_SPREAD = 2;  // k_colhist16_u16 wk mode: window-keyed sweep iff compact

__device__ __forceinline__ bool spread_is_wide(const SlabParams &p) {
    return *reinterpret_cast<const volatile int *>(p.spread) > SPREAD_WIDE;
}

// shift of the coarse key (candidate-bucket path)
__device__ __forceinline__ int key_shift(const SlabParams &p) {
    return p.spread ? reinterpret_cast<const volatile int *>(p.spread)[1] : 8 - p.key_down;
}

// true when a gated launch has nothing to do (uniform over the grid)
__device__ __forceinline__ bool gate_off(const SlabParams &p) {
    if (!p.gate) return false;
    return (p.gate == GATE_WIDE) != spread_is_wide(p);
}

// CTA-uniform: does the tile [x0, x0 + tw) x rows [y0, y1) contain a block
// the list kernel left undone?  (Every thread gets the same answer.)
__device__ __forceinline__ bool todo_any(const SlabParams &p, int x0, int tw, int y0, int y1) {
    const int bx0 = x0 >> 5, bx1 = min((x0 + tw + 31) >> 5, p.todo_nbx);
    const int by0 = (y0 - p.row_begin) / p.todo_bh, by1 = min((y1 - p.row_begin + p.todo_bh - 1) / p.todo_bh, p.todo_nby);
    const unsigned char *f = p.todo + (size_t)blockIdx.z * p.todo_nbx * p.todo_nby;
    const int nx = bx1 - bx0, cells = nx * (by1 - by0);
    int any = 0;
    for (int i = threadIdx.x; i < cells; i += blockDim.x) any |= f[(size_t)(by0 + i / nx) * p.todo_nbx + bx0 + i % nx];
    return __syncthreads_or(any) != 0;
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

template <typename P>
__device__ __forceinline__ const P *src_row(const SlabParams &p, const P *base, int g) {
    return base + (int64_t)(g - p.src_row0) * p.src_pitch;
}

// ---- streaming mode helpers (no-ops unless p.in_rows / p.out_px are set)

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int *a) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// A bound on the wait for source rows.  The host enqueues every copy and
// "rows arrived" write before the launch, so the wait only ever covers
// copy-engine time (a few ms per frame); if the rows never come (a broken
// caller), the CTA records the timeout in p.status and carries on, so the
// launch ends and the host reports an error instead of hanging.
constexpr uint64_t STREAM_TIMEOUT_NS = 20ull * 1000 * 1000 * 1000;

// spin (one thread) until source rows [0, need) have arrived
__device__ __forceinline__ void stream_wait_rows_1(const SlabParams &p, int need) {
    if (!p.in_rows) return;
    need = min(need, p.H);
    if ((int)ld_acquire(p.in_rows) >= need) return;
    const uint64_t t0 = globaltimer_ns();
    while ((int)ld_acquire(p.in_rows) < need) {
        __nanosleep(256);
        if (globaltimer_ns() - t0 > STREAM_TIMEOUT_NS) {
            if (p.status) atomicExch(p.status, 1u);
            return;
        }
    }
}

__device__ __forceinline__ void stream_wait_rows(const SlabParams &p, int need) {
    if (!p.in_rows) return;
    if (threadIdx.x == 0 && threadIdx.y == 0) stream_wait_rows_1(p, need);
    __syncthreads();
}

// one thread reports output rows [y0, y1) x columns [x0, x1) as written
__device__ __forceinline__ void stream_signal_1(const SlabParams &p, int y0, int y1, int x0, int x1) {
    if (!p.out_px) return;
    x1 = min(x1, p.W);
    y1 = min(y1, p.row_end);
    if (x1 <= x0 || y1 <= y0) return;
    __threadfence();
    const int C = p.out_chunk;
    for (int c = (y0 - p.row_begin) / C; c * C + p.row_begin < y1; ++c) {
        const int a = max(y0, p.row_begin + c * C), b = min(y1, p.row_begin + (c + 1) * C);
        atomicAdd(p.out_px + c, (unsigned int)((b - a) * (x1 - x0)));
    }
}

// CTA-wide: all threads' stores are done, then one thread signals
__device__ __forceinline__ void stream_signal(const SlabParams &p, int y0, int y1, int x0, int x1) {
    if (!p.out_px) return;
    __syncthreads();
    if (threadIdx.x == 0 && threadIdx.y == 0) stream_signal_1(p, y0, y1, x0, x1);
}

}  // namespace mtb
