// kernels_vert.cuh -- general rank-filter kernels, one thread per output
// column sliding DOWN a slab (any radius, any rank, 8/16-bit).
//
// Each thread owns the window histogram of its own output column as a
// hierarchy of counters in shared memory, laid out [bin][thread] so that
// the 32 lanes of a warp always hit 32 different banks.  Moving one row
// down removes the row leaving the window and adds the row entering it
// (2n single-counter updates, the reference's column-tree update of
// _kernels.py:115-127 applied to the window directly); the rank is then
// found by a coarse-to-fine counting descent (the reference's extract_u,
// _kernels.py:229-253, with 16-way instead of 2-way nodes).
//
// Cost is O(n) per output pixel.  It is the general path: every radius
// the reference accepts (validation.py:19-29, windows larger than the
// image included) and the 16-bit hierarchy.  The O(1)-in-r kernels in
// kernels_colhist.cuh take over where they apply.
#pragma once
#include "common.cuh"

namespace mtb {

// Incremental rank tracking for the vertical kernels.  m = previous output
// value, L = number of window pixels below m (kept current by the row
// updates).  Walk m down while L >= rank, up while L + h[m] < rank; the
// median moves little from row to row, so this replaces the 32-counter
// descent.  Returns false (caller falls back to the full descent) after
// `limit` steps.
template <typename FC>
__device__ __forceinline__ bool walk_rank(const FC *hf, int T, int fo, uint32_t rank, int &m,
                                          uint32_t &L, int limit) {
    int steps = 0;
    while (L >= rank) {
        if (++steps > limit) return false;
        --m;
        L -= hf[m * T + fo];
    }
    while (true) {
        const uint32_t c = hf[m * T + fo];
        if (L + c >= rank) return true;
        if (++steps > limit) return false;
        L += c;
        ++m;
    }
}

// 8-bit: coarse[16] (v>>4) + fine[256] (v) counters per thread.
template <typename CNT, int T>
__global__ void __launch_bounds__(T) k_vert_u8(SlabParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // distinct restrict pointers: the coarse and fine update chains may overlap
    CNT *__restrict__ hc = reinterpret_cast<CNT *>(smem_raw);  // [16][T]
    CNT *__restrict__ hf = reinterpret_cast<CNT *>(smem_raw) + 16 * T;  // [256][T]
    const int tid = threadIdx.x;
    const int x = blockIdx.x * T + tid;
    const int y0 = p.row_begin + blockIdx.y * p.rows_per_cta;
    if (y0 >= p.row_end || x >= p.W) return;  // no barriers below
    const int y1 = min(y0 + p.rows_per_cta, p.row_end);
    const uint8_t *src = static_cast<const uint8_t *>(p.src) + blockIdx.z * p.src_img_stride;
    uint8_t *dst = static_cast<uint8_t *>(p.dst) + blockIdx.z * p.dst_img_stride;
    const uint8_t *lut = static_cast<const uint8_t *>(p.lut);
    const int r = p.radius, H = p.H, W = p.W;
    stream_wait_rows_1(p, y1 + r);

    for (int b = 0; b < 16; ++b) hc[b * T + tid] = 0;
    for (int b = 0; b < 256; ++b) hf[b * T + tid] = 0;

    for (int j = -r; j <= r; ++j) {
        const uint8_t *row = src_row(p, src, clampi(y0 + j, 0, H - 1));
        for (int i = -r; i <= r; ++i) {
            const unsigned v = __ldg(row + clampi(x + i, 0, W - 1));
            hc[(v >> 4) * T + tid] += 1;
            hf[v * T + tid] += 1;
        }
    }
    int mprev = -1;   // previous output value (-1: none yet)
    uint32_t Lb = 0;  // window pixels below mprev
    const uint32_t rank = p.rank;
    for (int y = y0; y < y1; ++y) {
        if (y > y0) {
            const int yo = clampi(y - r - 1, 0, H - 1);
            const int yi = clampi(y + r, 0, H - 1);
            if (yo != yi) {
                const uint8_t *ro = src_row(p, src, yo);
                const uint8_t *ri = src_row(p, src, yi);
                for (int i = -r; i <= r; ++i) {
                    const int c = clampi(x + i, 0, W - 1);
                    const unsigned vo = __ldg(ro + c);
                    const unsigned vi = __ldg(ri + c);
                    Lb += ((int)vi < mprev ? 1u : 0u) - ((int)vo < mprev ? 1u : 0u);
                    hc[(vo >> 4) * T + tid] -= 1;
                    hf[vo * T + tid] -= 1;
                    hc[(vi >> 4) * T + tid] += 1;
                    hf[vi * T + tid] += 1;
                }
            }
        }
        int v = mprev;
        uint32_t L = Lb;
        if (mprev < 0 || !walk_rank(hf, T, tid, rank, v, L, 24)) {
            // coarse-to-fine counting descent
            uint32_t acc = 0;
            int b = 0;
            for (; b < 15; ++b) {
                const uint32_t c = hc[b * T + tid];
                if (acc + c >= rank) break;
                acc += c;
            }
            v = b * 16;
            for (const int e = v + 15; v < e; ++v) {
                const uint32_t c = hf[v * T + tid];
                if (acc + c >= rank) break;
                acc += c;
            }
            L = acc;
        }
        mprev = v;
        Lb = L;
        dst[(int64_t)(y - p.row_begin) * p.dst_pitch + x] = lut ? __ldg(lut + v) : (uint8_t)v;
    }
    stream_signal_1(p, y0, y1, x, x + 1);
}

// 16-bit: three-level hierarchy.  Levels 1+2 are the 8-bit hierarchy over
// the high byte (16 + 256 counters, unrestricted).  Level 3 resolves the
// low byte among window pixels whose high byte equals the selected one
// (16 + 256 counters restricted to high byte `curH`); it is maintained
// incrementally while the selected high byte stays the same and rebuilt
// from the window when it changes.
template <typename CNT, int T>
__global__ void __launch_bounds__(T) k_vert_u16(SlabParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CNT *tc = reinterpret_cast<CNT *>(smem_raw);  // [16][T]   high nibble
    CNT *tf = tc + 16 * T;                        // [256][T]  high byte
    CNT *lc = tf + 256 * T;                       // [16][T]   bits 4..7 | high byte == curH
    CNT *lf = lc + 16 * T;                        // [256][T]  low byte  | high byte == curH
    const int tid = threadIdx.x;
    const int x = blockIdx.x * T + tid;
    const int y0 = p.row_begin + blockIdx.y * p.rows_per_cta;
    if (y0 >= p.row_end || x >= p.W) return;
    const int y1 = min(y0 + p.rows_per_cta, p.row_end);
    const uint16_t *src = static_cast<const uint16_t *>(p.src) + blockIdx.z * p.src_img_stride;
    uint16_t *dst = static_cast<uint16_t *>(p.dst) + blockIdx.z * p.dst_img_stride;
    const uint16_t *lut = static_cast<const uint16_t *>(p.lut);
    const int r = p.radius, H = p.H, W = p.W;
    stream_wait_rows_1(p, y1 + r);

    for (int b = 0; b < 16; ++b) tc[b * T + tid] = 0;
    for (int b = 0; b < 256; ++b) tf[b * T + tid] = 0;
    for (int j = -r; j <= r; ++j) {
        const uint16_t *row = src_row(p, src, clampi(y0 + j, 0, H - 1));
        for (int i = -r; i <= r; ++i) {
            const unsigned v = __ldg(row + clampi(x + i, 0, W - 1));
            tc[(v >> 12) * T + tid] += 1;
            tf[(v >> 8) * T + tid] += 1;
        }
    }
    int curH = -1;
    const uint32_t rank = p.rank;
    for (int y = y0; y < y1; ++y) {
        if (y > y0) {
            const int yo = clampi(y - r - 1, 0, H - 1);
            const int yi = clampi(y + r, 0, H - 1);
            if (yo != yi) {
                const uint16_t *ro = src_row(p, src, yo);
                const uint16_t *ri = src_row(p, src, yi);
                for (int i = -r; i <= r; ++i) {
                    const int c = clampi(x + i, 0, W - 1);
                    const unsigned vo = __ldg(ro + c);
                    const unsigned vi = __ldg(ri + c);
                    tc[(vo >> 12) * T + tid] -= 1;
                    tf[(vo >> 8) * T + tid] -= 1;
                    tc[(vi >> 12) * T + tid] += 1;
                    tf[(vi >> 8) * T + tid] += 1;
                    if ((int)(vo >> 8) == curH) {
                        lc[((vo >> 4) & 15) * T + tid] -= 1;
                        lf[(vo & 255) * T + tid] -= 1;
                    }
                    if ((int)(vi >> 8) == curH) {
                        lc[((vi >> 4) & 15) * T + tid] += 1;
                        lf[(vi & 255) * T + tid] += 1;
                    }
                }
            }
        }
        uint32_t acc = 0;
        int b = 0;
        for (; b < 15; ++b) {
            const uint32_t c = tc[b * T + tid];
            if (acc + c >= rank) break;
            acc += c;
        }
        int hb = b * 16;
        for (const int e = hb + 15; hb < e; ++hb) {
            const uint32_t c = tf[hb * T + tid];
            if (acc + c >= rank) break;
            acc += c;
        }
        if (hb != curH) {  // rebuild the restricted low-byte hierarchy
            curH = hb;
            for (int k = 0; k < 16; ++k) lc[k * T + tid] = 0;
            for (int k = 0; k < 256; ++k) lf[k * T + tid] = 0;
            for (int j = -r; j <= r; ++j) {
                const uint16_t *row = src_row(p, src, clampi(y + j, 0, H - 1));
                for (int i = -r; i <= r; ++i) {
                    const unsigned v = __ldg(row + clampi(x + i, 0, W - 1));
                    if ((int)(v >> 8) == curH) {
                        lc[((v >> 4) & 15) * T + tid] += 1;
                        lf[(v & 255) * T + tid] += 1;
                    }
                }
            }
        }
        int lb = 0;
        for (; lb < 15; ++lb) {
            const uint32_t c = lc[lb * T + tid];
            if (acc + c >= rank) break;
            acc += c;
        }
        int lo = lb * 16;
        for (const int e = lo + 15; lo < e; ++lo) {
            const uint32_t c = lf[lo * T + tid];
            if (acc + c >= rank) break;
            acc += c;
        }
        const unsigned v = ((unsigned)hb << 8) | (unsigned)lo;
        dst[(int64_t)(y - p.row_begin) * p.dst_pitch + x] = lut ? __ldg(lut + v) : (uint16_t)v;
    }
    stream_signal_1(p, y0, y1, x, x + 1);
}

// U independent branchless lower_bounds over sorted arrays of the same
// length n, interleaved step by step so their shared-memory loads overlap
// (the step count depends only on n, so the loop is warp-uniform).
template <int U>
__device__ __forceinline__ void lower_bound_multi(const uint16_t *const (&a)[U], int n,
                                                  const unsigned (&v)[U], int (&out)[U]) {
    int base[U];
#pragma unroll
    for (int u = 0; u < U; ++u) base[u] = 0;
    for (int len = n; len > 1;) {
        const int half = len >> 1;
#pragma unroll
        for (int u = 0; u < U; ++u) base[u] += (a[u][base[u] + half] < v[u]) ? half : 0;
        len -= half;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) out[u] = base[u] + ((a[u][base[u]] < v[u]) ? 1 : 0);
}

}  // namespace mtb
