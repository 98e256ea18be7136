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
#include "kernels_ctmf.cuh"  // ct_stage

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

// 8-bit general path, v2: each warp stages the rows it needs (its 32
// columns + 2r halo, clamped) in shared memory with coalesced loads, so the
// 2n per-row counter updates read pixels from shared memory instead of 2n
// dependent global loads; fine counters are u8 when the window holds at
// most 255 pixels (r <= 7), halving the footprint and doubling occupancy.
template <typename FC, int T>
__global__ void __launch_bounds__(T) k_vert2_u8(SlabParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint16_t *__restrict__ hc = reinterpret_cast<uint16_t *>(smem_raw);           // [16][T]
    FC *__restrict__ hf = reinterpret_cast<FC *>(smem_raw + 16 * T * sizeof(uint16_t));  // [256][T]
    const int r = p.radius, H = p.H, W = p.W;
    const int SPW = (32 + 2 * r + 16 + 15) & ~15;               // staged row pitch
    uint8_t *stg = reinterpret_cast<uint8_t *>(hf + 256 * T) + (threadIdx.x >> 5) * 2 * SPW;
    const int tid = threadIdx.x, lane = tid & 31;
    const int x = blockIdx.x * T + tid;
    const int xw = blockIdx.x * T + (tid & ~31);                  // warp's first column
    const int y0 = p.row_begin + blockIdx.y * p.rows_per_cta;
    if (y0 >= p.row_end || xw >= W) return;                       // warp-uniform
    const int y1 = min(y0 + p.rows_per_cta, p.row_end);
    stream_wait_rows_1(p, y1 + r);
    const uint8_t *src = static_cast<const uint8_t *>(p.src) + blockIdx.z * p.src_img_stride;
    uint8_t *dst = static_cast<uint8_t *>(p.dst) + blockIdx.z * p.dst_img_stride;
    const uint8_t *lut = static_cast<const uint8_t *>(p.lut);
    const int sx0 = max(0, xw - r), sx1 = min(W, xw + 32 + r);
    const int A = ct_span_base(sx0);
    const bool aligned = ct_rows_aligned16(src, p.src_pitch);
    StageBar sbar = ct_stage_init(lane);
    // staged index of window column i (0..2r) of this thread
    auto sidx = [&](int i) { return clampi(x - r + i, 0, W - 1) - A; };
    // u8 counters: lane l of warp w at byte 4l+w, so a warp's 32 lanes hit
    // 32 different banks whatever their values
    const int fo = sizeof(FC) == 1 ? (((tid & 31) << 2) | (tid >> 5)) : tid;

    for (int b = 0; b < 16; ++b) hc[b * T + tid] = 0;
    for (int b = 0; b < 256; ++b) hf[b * T + fo] = 0;
    for (int j = -r; j <= r; ++j) {
        int g = clampi(y0 + j, 0, H - 1);
        __syncwarp();
        ct_stage(p, src, stg, SPW, &g, 1, A, sx1, aligned, lane, &sbar);
        __syncwarp();
        for (int i = 0; i <= 2 * r; ++i) {
            const unsigned v = stg[sidx(i)];
            hc[(v >> 4) * T + tid] += 1;
            hf[v * T + fo] += 1;
        }
    }
    int mprev = -1;
    uint32_t Lb = 0;
    const uint32_t rank = p.rank;
    for (int y = y0; y < y1; ++y) {
        if (y > y0) {
            int g[2] = {clampi(y - r - 1, 0, H - 1), clampi(y + r, 0, H - 1)};
            if (g[0] != g[1]) {
                __syncwarp();
                ct_stage(p, src, stg, SPW, g, 2, A, sx1, aligned, lane, &sbar);
                __syncwarp();
                for (int i = 0; i <= 2 * r; ++i) {
                    const int si = sidx(i);
                    const unsigned vo = stg[si], vi = stg[SPW + si];
                    if (vo == vi) continue;
                    Lb += ((int)vi < mprev ? 1u : 0u) - ((int)vo < mprev ? 1u : 0u);
                    if ((vo >> 4) != (vi >> 4)) {
                        hc[(vo >> 4) * T + tid] -= 1;
                        hc[(vi >> 4) * T + tid] += 1;
                    }
                    hf[vo * T + fo] -= 1;
                    hf[vi * T + fo] += 1;
                }
            }
        }
        int v = mprev;
        uint32_t L = Lb;
        if (mprev < 0 || !walk_rank(hf, T, fo, rank, v, L, 24)) {
            uint32_t acc = 0;
            int b = 0;
            for (; b < 15; ++b) {
                const uint32_t c = hc[b * T + tid];
                if (acc + c >= rank) break;
                acc += c;
            }
            v = b * 16;
            for (const int e = v + 15; v < e; ++v) {
                const uint32_t c = hf[v * T + fo];
                if (acc + c >= rank) break;
                acc += c;
            }
            L = acc;
        }
        mprev = v;
        Lb = L;
        if (x < W) dst[(int64_t)(y - p.row_begin) * p.dst_pitch + x] = lut ? __ldg(lut + v) : (uint8_t)v;
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

}  // namespace mtb

namespace mtb {

// ---------------------------------------------------------------------------
// 16-bit general path, v2.  The high byte H of the result comes from the
// same incremental per-thread counters as k_vert_u16 (16 + 256); the low
// byte comes from per-column SORTED arrays instead of a second counter
// level: the CTA keeps, for every column of its halo'd stripe, the n pixels
// of the column's current vertical span in ascending order, so the window
// values with high byte H are one run per window column, starting at
// lower_bound(256H) (2r+1 interleaved branchless binary searches, whose
// results are kept as u8 run starts for the second pass).  The low byte is
// then two counting passes over the runs (bits 4..7, then bits 0..3 of the
// selected 16-value sub-run) into 16 scratch counters.  (Moving the run
// starts incrementally instead of searching was measured slower: the walk
// is a chain of dependent loads per column, the searches overlap.)
// Moving down a row deletes the leaving value and inserts the entering one
// in each sorted column (one shift of the elements between the positions).

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

template <typename CNT, int T>
__global__ void __launch_bounds__(T) k_vert2_u16(SlabParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CNT *tc = reinterpret_cast<CNT *>(smem_raw);  // [16][T]   high nibble
    CNT *tf = tc + 16 * T;                        // [256][T]  high byte
    CNT *sc = tf + 256 * T;                       // [16][T]   scratch: nibble counts inside H
    uint16_t *scol = reinterpret_cast<uint16_t *>(sc + 16 * T);  // [NCOL][n] sorted columns
    const int tid = threadIdx.x;
    const int r = p.radius, H = p.H, W = p.W, n = 2 * r + 1;
    const int NCOL = T + 2 * r;
    uint8_t *rpos = reinterpret_cast<uint8_t *>(scol + NCOL * n);  // [n][T] run starts
    const int X0 = blockIdx.x * T;
    const int x = X0 + tid;
    const int y0 = p.row_begin + blockIdx.y * p.rows_per_cta;
    if (y0 >= p.row_end) return;  // CTA-uniform (barriers below)
    const int y1 = min(y0 + p.rows_per_cta, p.row_end);
    stream_wait_rows(p, y1 + r);
    const uint16_t *src = static_cast<const uint16_t *>(p.src) + blockIdx.z * p.src_img_stride;
    uint16_t *dst = static_cast<uint16_t *>(p.dst) + blockIdx.z * p.dst_img_stride;
    const uint16_t *lut = static_cast<const uint16_t *>(p.lut);
    const int xc = min(x, W - 1);  // threads beyond the edge compute a clamped column, store nothing
    // window column j of this thread is stripe column c0 + j (global xc - r + j, clamped)
    const uint16_t *wcol = scol + (xc - X0) * n;

    // sorted columns at row y0 (insertion sort of each column's span)
    for (int k = tid; k < NCOL; k += T) {
        uint16_t *a = scol + k * n;
        const int gx = clampi(X0 - r + k, 0, W - 1);
        for (int j = 0; j < n; ++j) {
            const uint16_t v = __ldg(src_row(p, src, clampi(y0 - r + j, 0, H - 1)) + gx);
            int i = j;
            while (i > 0 && a[i - 1] > v) {
                a[i] = a[i - 1];
                --i;
            }
            a[i] = v;
        }
    }
    for (int b = 0; b < 16; ++b) tc[b * T + tid] = 0;
    for (int b = 0; b < 256; ++b) tf[b * T + tid] = 0;
    for (int j = -r; j <= r; ++j) {
        const uint16_t *row = src_row(p, src, clampi(y0 + j, 0, H - 1));
        for (int i = -r; i <= r; ++i) {
            const unsigned v = __ldg(row + clampi(xc + i, 0, W - 1));
            tc[(v >> 12) * T + tid] += 1;
            tf[(v >> 8) * T + tid] += 1;
        }
    }
    __syncthreads();
    const uint32_t rank = p.rank;
    for (int y = y0; y < y1; ++y) {
        if (y > y0) {
            const int yo = clampi(y - r - 1, 0, H - 1);
            const int yi = clampi(y + r, 0, H - 1);
            if (yo != yi) {
                const uint16_t *ro = src_row(p, src, yo);
                const uint16_t *ri = src_row(p, src, yi);
                // window counters of this thread
                for (int i = -r; i <= r; ++i) {
                    const int c = clampi(xc + i, 0, W - 1);
                    const unsigned vo = __ldg(ro + c);
                    const unsigned vi = __ldg(ri + c);
                    if (vo == vi) continue;
                    tc[(vo >> 12) * T + tid] -= 1;
                    tf[(vo >> 8) * T + tid] -= 1;
                    tc[(vi >> 12) * T + tid] += 1;
                    tf[(vi >> 8) * T + tid] += 1;
                }
                __syncthreads();  // everyone done reading the sorted columns
                // sorted columns: delete the leaving value, insert the entering one
                for (int k = tid; k < NCOL; k += T) {
                    const int gx = clampi(X0 - r + k, 0, W - 1);
                    const unsigned vo = __ldg(ro + gx), vi = __ldg(ri + gx);
                    if (vo == vi) continue;
                    uint16_t *a = scol + k * n;
                    const uint16_t *const aa[2] = {a, a};
                    const unsigned vv[2] = {vo, vi};
                    int pos[2];
                    lower_bound_multi<2>(aa, n, vv, pos);
                    const int io = pos[0];  // a[io] == vo
                    const int ii = pos[1];
                    if (ii > io) {
                        for (int q = io; q < ii - 1; ++q) a[q] = a[q + 1];
                        a[ii - 1] = (uint16_t)vi;
                    } else {
                        for (int q = io; q > ii; --q) a[q] = a[q - 1];
                        a[ii] = (uint16_t)vi;
                    }
                }
                __syncthreads();
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
        // low byte: the (rank - acc)-th smallest window value in [vb, vb+256)
        const unsigned vb = (unsigned)hb << 8, ve = vb + 256;
#pragma unroll
        for (int q = 0; q < 16; ++q) sc[q * T + tid] = 0;
        for (int j0 = 0; j0 < n; j0 += 8) {
            const uint16_t *aa[8];
            unsigned vv[8];
            int e0[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                aa[u] = wcol + min(j0 + u, n - 1) * n;
                vv[u] = vb;
            }
            lower_bound_multi<8>(aa, n, vv, e0);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (j0 + u >= n) break;
                rpos[(j0 + u) * T + tid] = (uint8_t)e0[u];
                const uint16_t *a = aa[u];
                for (int e = e0[u]; e < n; ++e) {
                    const unsigned v = a[e];
                    if (v >= ve) break;
                    sc[((v >> 4) & 15) * T + tid] += 1;
                }
            }
        }
        int lb = 0;
        for (; lb < 15; ++lb) {
            const uint32_t c = sc[lb * T + tid];
            if (acc + c >= rank) break;
            acc += c;
        }
        // bits 0..3 inside the 16-value sub-run [vs, vs+16)
        const unsigned vs = vb + 16u * (unsigned)lb, vse = vs + 16;
#pragma unroll
        for (int q = 0; q < 16; ++q) sc[q * T + tid] = 0;
        for (int j = 0; j < n; ++j) {
            const uint16_t *a = wcol + j * n;
            for (int e = rpos[j * T + tid]; e < n; ++e) {
                const unsigned v = a[e];
                if (v >= vse) break;
                if (v >= vs) sc[(v & 15) * T + tid] += 1;
            }
        }
        int lo = lb * 16;
        for (const int e = lo + 15; lo < e; ++lo) {
            const uint32_t c = sc[(lo & 15) * T + tid];
            if (acc + c >= rank) break;
            acc += c;
        }
        const unsigned v = ((unsigned)hb << 8) | (unsigned)lo;
        if (x < W) dst[(int64_t)(y - p.row_begin) * p.dst_pitch + x] = lut ? __ldg(lut + v) : (uint16_t)v;
    }
    stream_signal(p, y0, y1, X0, X0 + T);
}

}  // namespace mtb
