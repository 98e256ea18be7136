// kernels_ctmf.cuh -- 8-bit rank filter with per-column histograms in shared
// memory and horizontal window sliding: O(1) window-histogram work per
// output pixel in the radius (the reference's per-column trees + window
// sync, _kernels.py:115-194, re-planned for a warp).
//
// Decomposition.  Each WARP owns an independent tile: output columns
// [X0, X0 + 32*S) and rows [Y0, Y1).  Lane t owns the S consecutive output
// columns x_t = X0 + t*S ... x_t + S-1 of every row.  The tile keeps one
// 16-bin histogram per column of the halo'd stripe [X0-r, X0+32S+r)
// ("column histograms", u16 counts, 32 B per column) for the current row;
// moving down one row removes the pixel leaving each column's vertical
// span and adds the one entering it (2 counter updates per column).
//
// Per row, lane t first rebuilds its window histogram at x_t from the
// column histograms (chunk sums + warp shuffles, ct_window), then slides
// right S-1 times with
//     W += C[x + r + 1] - C[x - r]       (16 bins = 8 packed u16 words, IADD3)
// and resolves the rank at every position by a 4-step binary descent over
// the 16 bins (the reference's extract_u, _kernels.py:229-253, 16-ary).
//
// Two levels (16 coarse bins of width 16, then 16 fine bins):
//   pass 1 (coarse): bins v>>4; writes the coarse bin of each output into
//           dst (scratch) and collects the set of coarse bins the tile uses;
//   pass 2 (fine), once per coarse bin B used by the tile: histograms count
//           only pixels with v>>4 == B (bins v&15) plus, per column, the
//           number of pixels below 16*B; outputs whose coarse bin is B
//           resolve their low nibble with rank - below.
// All arithmetic is exact integer counting; window counts fit u16 because
// n^2 <= 65535 is required (r <= 127; larger windows use kernels_vert).
#pragma once
#include "common.cuh"

namespace mtb {

constexpr int CT_WARPS = 4;
constexpr int CT_STAGE_ROWS = 8;  // image rows staged per batch (init); nibble counts stay < 16

struct CtmfGeom {
    int S, TW, NC, NCP;    // lane segment, tile width, halo'd columns, padded
    int colh_bytes;        // per warp: 2 chunk arrays of NCP x 16 B
    int below_bytes;       // per warp: NCP u16
    int SPB;               // staged row pitch (bytes)
    int warp_bytes;
};

__host__ __device__ inline CtmfGeom ctmf_geom(int S, int r, int stage_rows = CT_STAGE_ROWS) {
    CtmfGeom g;
    g.S = S;
    g.TW = 32 * S;
    g.NC = g.TW + 2 * r;
    g.NCP = (g.NC + 31) & ~31;
    g.colh_bytes = 2 * g.NCP * 16;
    g.below_bytes = (g.NCP + 8) * 2;  // + dummy counter
    g.SPB = (g.NC + 16 + 15) & ~15;
    g.warp_bytes = g.colh_bytes + ((g.below_bytes + 15) & ~15) + stage_rows * g.SPB;
    return g;
}

// column slot swizzle: lanes read columns S apart; XOR the low 3 bits with
// (c/S) so the 32 lanes' 16-B records spread over all 8 bank groups.
template <int S>
__device__ __forceinline__ int ct_slot(int c) {
    return c ^ ((c / S) & 7);
}

__device__ __forceinline__ uint32_t hsum16(uint32_t w) {  // lo + hi (sum < 2^16)
    return (w * 0x10001u) >> 16;
}

// Smallest bin b with cumsum(bins[0..b]) >= k; returns b and leaves in k the
// rank within bin b.  bins are 16 u16 counters packed in w[0..7].
__device__ __forceinline__ int ct_descend(const uint32_t (&w)[8], uint32_t &k) {
    uint32_t t = w[0] + w[1] + w[2] + w[3];
    uint32_t s = hsum16(t);
    const bool r1 = s < k;
    k -= r1 ? s : 0u;
    uint32_t a0 = r1 ? w[4] : w[0], a1 = r1 ? w[5] : w[1];
    uint32_t a2 = r1 ? w[6] : w[2], a3 = r1 ? w[7] : w[3];
    s = hsum16(a0 + a1);
    const bool r2 = s < k;
    k -= r2 ? s : 0u;
    uint32_t b0 = r2 ? a2 : a0, b1 = r2 ? a3 : a1;
    s = hsum16(b0);
    const bool r3 = s < k;
    k -= r3 ? s : 0u;
    const uint32_t c = r3 ? b1 : b0;
    s = c & 0xffffu;
    const bool r4 = s < k;
    k -= r4 ? s : 0u;
    return (r1 ? 8 : 0) | (r2 ? 4 : 0) | (r3 ? 2 : 0) | (r4 ? 1 : 0);
}


// Window histograms of every lane at its segment start, straight from the
// column histograms: lane t needs columns [tS, tS+2r].  Each lane sums its
// own chunk of S columns (and a second chunk when the halo'd stripe has
// more than 32 chunks), keeping the partial sum of the chunk's first m
// columns; the window is then q whole chunks plus one partial chunk,
// gathered with warp shuffles (n = qS + m).  O(S + n/S) per lane per row,
// independent of the radius' one-hot cost.
template <int S>
__device__ __forceinline__ void ct_chunk(const uint4 *colA, const uint4 *colB, const uint16_t *below,
                                         bool fine, int j, int m, int NC, uint32_t (&L)[9],
                                         uint32_t (&P)[9]) {
#pragma unroll
    for (int i = 0; i < 9; ++i) L[i] = 0;
    const int c0 = j * S;
    int c = c0;
    for (; c < c0 + m; ++c) {
        const int sl = ct_slot<S>(c);
        const uint4 a = colA[sl], b = colB[sl];
        L[0] += a.x; L[1] += a.y; L[2] += a.z; L[3] += a.w;
        L[4] += b.x; L[5] += b.y; L[6] += b.z; L[7] += b.w;
        if (fine && c < NC) L[8] += below[c];
    }
#pragma unroll
    for (int i = 0; i < 9; ++i) P[i] = L[i];
    for (; c < c0 + S; ++c) {
        const int sl = ct_slot<S>(c);
        const uint4 a = colA[sl], b = colB[sl];
        L[0] += a.x; L[1] += a.y; L[2] += a.z; L[3] += a.w;
        L[4] += b.x; L[5] += b.y; L[6] += b.z; L[7] += b.w;
        if (fine && c < NC) L[8] += below[c];
    }
}

// MF >= 0: n mod S as a compile-time constant (the partial-chunk loops unroll)
template <int S, int MF = -1>
__device__ __noinline__ void ct_window(const uint4 *colA, const uint4 *colB, const uint16_t *below,
                                          bool fine, int lane, int r, int NC, uint32_t (&ws)[8],
                                          uint32_t &wb) {
    const int n = 2 * r + 1, q = n / S, m = MF >= 0 ? MF : n - q * S;
    const int J = (NC + S - 1) / S;
    uint32_t LA[9], PA[9], LB[9], PB[9];
    ct_chunk<S>(colA, colB, below, fine, lane, m, NC, LA, PA);
    if (lane + 32 < J) {
        ct_chunk<S>(colA, colB, below, fine, lane + 32, m, NC, LB, PB);
    } else {
#pragma unroll
        for (int i = 0; i < 9; ++i) LB[i] = PB[i] = 0;
    }
    uint32_t acc[9];
    if (q >= 5 && (int64_t)NC * n < 65536) {
        // exclusive prefix I_j over the (up to 64) chunk sums, two rounds of
        // 32; window(t) = I_{t+q} + P_{t+q} - I_t.  Packed u16 lanes never
        // carry: every prefix is <= NC*n < 2^16.
        uint32_t IA[9], IB[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) {
            uint32_t a = LA[i], b = LB[i];
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t ta = __shfl_up_sync(0xffffffffu, a, d);
                const uint32_t tb = __shfl_up_sync(0xffffffffu, b, d);
                if (lane >= d) {
                    a += ta;
                    b += tb;
                }
            }
            const uint32_t totA = __shfl_sync(0xffffffffu, a, 31);
            IA[i] = a - LA[i];            // exclusive, round A
            IB[i] = b - LB[i] + totA;     // exclusive, round B
        }
        const int idx = lane + q;
        const bool hiB = idx >= 32;
        const int sl = idx & 31;
#pragma unroll
        for (int i = 0; i < 9; ++i) {
            const uint32_t xa = __shfl_sync(0xffffffffu, IA[i] + PA[i], sl);
            const uint32_t xb = __shfl_sync(0xffffffffu, IB[i] + PB[i], sl);
            acc[i] = (hiB ? xb : xa) - IA[i];
        }
    } else {
#pragma unroll
    for (int i = 0; i < 9; ++i) acc[i] = 0;
    for (int k = 0; k <= q; ++k) {
        const int idx = lane + k;
        const bool hiB = idx >= 32;
        const int sl = idx & 31;
        if (k < q) {
#pragma unroll
            for (int i = 0; i < 9; ++i) {
                const uint32_t a = __shfl_sync(0xffffffffu, LA[i], sl);
                const uint32_t b = __shfl_sync(0xffffffffu, LB[i], sl);
                acc[i] += hiB ? b : a;
            }
        } else if (m > 0) {
#pragma unroll
            for (int i = 0; i < 9; ++i) {
                const uint32_t a = __shfl_sync(0xffffffffu, PA[i], sl);
                const uint32_t b = __shfl_sync(0xffffffffu, PB[i], sl);
                acc[i] += hiB ? b : a;
            }
        }
    }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) ws[i] = acc[i];
    wb = acc[8];
}

// ---- row staging ---------------------------------------------------------
// Stage `nrows` image rows (global rows g[k]) of a tile's halo'd column span
// into shared memory: column X of staged row k lands at stage + k*SPB +
// (X - A), with A = span start rounded down to 16 bytes.
//
// TMA path (rows 16-byte aligned): lane 0 of the warp arms the warp's
// mbarrier with the byte count and issues one cp.async.bulk (global ->
// shared, completion on the mbarrier) per row for the 16-byte-aligned body;
// the other lanes load the <16-byte tail; everyone waits on the mbarrier.
// Fallback path: independent 4-byte / 1-byte loads by all lanes.
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

struct StageBar {
    uint64_t *bar;   // this warp's mbarrier
    uint32_t phase;  // parity of the next completion
};

// one mbarrier per warp; call once per warp before the first ct_stage
__device__ __forceinline__ StageBar ct_stage_init(int lane) {
    __shared__ __align__(8) uint64_t s_bar[32];
    uint64_t *bar = &s_bar[threadIdx.x >> 5];
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    return StageBar{bar, 0u};
}

__device__ __forceinline__ void ct_stage(const SlabParams &p, const uint8_t *src, uint8_t *stage,
                                         int SPB, const int *g, int nrows, int A, int sx1,
                                         bool aligned, int lane, StageBar *sb = nullptr) {
    const int nbytes = sx1 - A;
    if (sb && aligned) {
        // rows are 16-B aligned with a pitch that is a multiple of 16, so the
        // span rounded up to 16 bytes stays inside the row's pitch: one bulk
        // copy per row, no tail (bytes past sx1 are never indexed)
        const int body = (nbytes + 15) & ~15;
        if (body > 0) {
            if (lane == 0) {
                // order earlier generic-proxy reads of the stage before the TMA writes
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                             ::"r"(smem_addr(sb->bar)), "r"(body * nrows) : "memory");
                for (int k = 0; k < nrows; ++k) {
                    const uint8_t *rb = src_row(p, src, g[k]) + A;
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
                        "[%0], [%1], %2, [%3];"
                        ::"r"(smem_addr(stage + k * SPB)), "l"(rb), "r"(body),
                          "r"(smem_addr(sb->bar)) : "memory");
                }
            }
            uint32_t done = 0;
            while (!done) {
                asm volatile(
                    "{\n .reg .pred P;\n"
                    " mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n"
                    " selp.b32 %0, 1, 0, P;\n}\n"
                    : "=r"(done) : "r"(smem_addr(sb->bar)), "r"(sb->phase) : "memory");
            }
            sb->phase ^= 1u;
            return;
        }
    }
    if (aligned) {
        const int nw = nbytes >> 2;
        for (int k = 0; k < nrows; ++k) {
            const uint32_t *rw = reinterpret_cast<const uint32_t *>(src_row(p, src, g[k]) + A);
            uint32_t *sw = reinterpret_cast<uint32_t *>(stage + k * SPB);
            for (int w = lane; w < nw; w += 32) sw[w] = __ldg(rw + w);
        }
        for (int k = 0; k < nrows; ++k) {
            const uint8_t *rb = src_row(p, src, g[k]) + A;
            for (int b = (nw << 2) + lane; b < nbytes; b += 32) stage[k * SPB + b] = __ldg(rb + b);
        }
    } else {
        for (int k = 0; k < nrows; ++k) {
            const uint8_t *rb = src_row(p, src, g[k]) + A;
            for (int b = lane; b < nbytes; b += 32) stage[k * SPB + b] = __ldg(rb + b);
        }
    }
}

// span start aligned for staging; rows are TMA-eligible when 16-B aligned
__device__ __forceinline__ int ct_span_base(int sx0) { return sx0 & ~15; }
__device__ __forceinline__ bool ct_rows_aligned16(const void *src, int64_t pitch) {
    return ((reinterpret_cast<uintptr_t>(src) | (uintptr_t)pitch) & 15) == 0;
}

// MF >= 0: n mod S as a compile-time constant (measured: r = 63 1.11 -> 0.99 ms
// with the whole radius fixed; the partial-chunk loops are what unrolls)
// ---------------------------------------------------------------------------
// k_ctmf_pre_u8: every tile row's span snapshots in one pass, before the
// tiles run.  Thread = image column: it builds the 256-bin histogram of the
// span of the first tile row of its segment (rows clamp(Y0-r .. Y0+r)),
// then slides down tile row by tile row (one row out, one in per step),
// writing after each tile row the 16-B cumulative coarse counts and the 16
// fine chunks: pre[((z*tiles_y + ty)*17 + q)*W + x], q = 0 the cumulative
// counts, q = 1..16 the chunks -- component-major, so a warp's stores and
// a tile's loads of one component over consecutive columns are contiguous.
// The tiles then
// initialise every pass from two 16-B loads per column instead of scanning
// n rows per column twice (the two snapshot scans were ~25% of the CTMF
// kernel's instructions).
constexpr int CTP_T = 128;
constexpr int CTP_STRIDE = 272;  // per-thread histogram bytes (17 x 16: 16-B aligned rows)

template <int T = CTP_T>  // (a template: the header is included by several translation units)
__global__ void __launch_bounds__(T) k_ctmf_pre_u8(SlabParams p, int tiles_y, int seg, uint4 *__restrict__ pre) {
    // per thread 272 B = [cumulative coarse counts (16 B)][256 fine counts]
    __shared__ __align__(16) uint8_t hist[T * CTP_STRIDE];
    const int tid = threadIdx.x, warp0 = tid & ~31;
    const int W = p.W, H = p.H, r = p.radius, th = p.rows_per_cta;
    const int xw = blockIdx.x * T + warp0;  // the warp's first column
    const int x = xw + (tid & 31);
    const int ty0 = blockIdx.y * seg, ty1 = min(ty0 + seg, tiles_y);
    const uint8_t *src = static_cast<const uint8_t *>(p.src) + blockIdx.z * p.src_img_stride;
    if (p.in_rows) {  // streaming: the segment's rows have arrived
        stream_wait_rows(p, min(p.row_begin + ty1 * th + r, H));
    }
    if (xw >= W || ty0 >= ty1) return;  // warp-uniform (no block barriers below)
    const int xc = min(x, W - 1);  // lanes past the image edge shadow the last column
    uint8_t *rec = hist + tid * CTP_STRIDE;
    uint8_t *h = rec + 16;
    uint4 *h4 = reinterpret_cast<uint4 *>(h);
#pragma unroll
    for (int q = 0; q < 16; ++q) h4[q] = make_uint4(0, 0, 0, 0);
    const int Ya = p.row_begin + ty0 * th;
    // 16 loads in flight per thread (the rows come from L2; latency-bound otherwise)
    int j = -r;
    for (; j + 15 <= r; j += 16) {
        unsigned v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = __ldg(src_row(p, src, clampi(Ya + j + u, 0, H - 1)) + xc);
#pragma unroll
        for (int u = 0; u < 16; ++u) h[v[u]] += 1;
    }
    for (; j <= r; ++j) h[__ldg(src_row(p, src, clampi(Ya + j, 0, H - 1)) + xc)] += 1;
    int y = Ya;
    for (int ty = ty0; ty < ty1; ++ty) {
        const int Y0 = p.row_begin + ty * th;
        for (; y + 8 <= Y0; y += 8) {  // slide the span down to rows Y0-r .. Y0+r
            unsigned vo[8], vi[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                vo[u] = __ldg(src_row(p, src, clampi(y + u - r, 0, H - 1)) + xc);
                vi[u] = __ldg(src_row(p, src, clampi(y + u + r + 1, 0, H - 1)) + xc);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                h[vo[u]] -= 1;
                h[vi[u]] += 1;
            }
        }
        for (; y < Y0; ++y) {
            const unsigned vo = __ldg(src_row(p, src, clampi(y - r, 0, H - 1)) + xc);
            const unsigned vi = __ldg(src_row(p, src, clampi(y + r + 1, 0, H - 1)) + xc);
            h[vo] -= 1;
            h[vi] += 1;
        }
        uint32_t acc = 0, cw[4] = {0, 0, 0, 0};
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const uint4 c = h4[q];
            cw[q >> 2] |= acc << (8 * (q & 3));
            acc += __vsadu4(c.x, 0) + __vsadu4(c.y, 0) + __vsadu4(c.z, 0) + __vsadu4(c.w, 0);
        }
        if (x < W) {
            uint4 *o = pre + (size_t)(blockIdx.z * tiles_y + ty) * 17 * W + x;
            o[0] = make_uint4(cw[0], cw[1], cw[2], cw[3]);
            // empty chunks are not written: a tile loads chunk b only when the
            // cumulative counts show coarse bin b present in the column
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const uint4 c = h4[q];
                if (c.x | c.y | c.z | c.w) o[(size_t)(1 + q) * W] = c;
            }
        }
    }
}

// PRE: initialised from k_ctmf_pre_u8's snapshots only (`pre` required):
// no staged init batches, so the stage holds the two rows of a row update
// and four CTAs fit per SM.  CTB: CTAs per SM the registers are budgeted
// for (4: 16 warps at 128 registers, with spills -- pays from r ~ 80; 3:
// 12 warps at 168).
template <int S, int MF = -1, bool PRE = false, int CTB = 3>
__global__ void __launch_bounds__(CT_WARPS * 32, CTB) k_ctmf_u8(SlabParams p, int tiles_x, int tiles_y,
                                                        uint8_t *__restrict__ snap, int snap_two_scans,
                                                        const uint4 *__restrict__ pre) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    // persistent warps: tiles are dealt round-robin to the resident warps
    // (no partial last wave); warp-uniform control, no block barriers
    const int first_tile = blockIdx.x * CT_WARPS + warp;
    if (first_tile >= tiles_x * tiles_y) return;
    const int r = p.radius;
    const CtmfGeom g = ctmf_geom(S, r, PRE ? 2 : CT_STAGE_ROWS);
    unsigned char *base = smem_raw + (size_t)warp * g.warp_bytes;
    uint4 *colA = reinterpret_cast<uint4 *>(base);               // bins 0-7
    uint4 *colB = colA + g.NCP;                                  // bins 8-15
    uint16_t *below = reinterpret_cast<uint16_t *>(base + g.colh_bytes);
    uint8_t *stage = base + g.colh_bytes + ((g.below_bytes + 15) & ~15);

    StageBar sbar = ct_stage_init(lane);
    for (int tile = first_tile; tile < tiles_x * tiles_y; tile += gridDim.x * CT_WARPS) {
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int W = p.W, H = p.H;
    const int X0 = tx * g.TW;
    const int Y0 = p.row_begin + ty * p.rows_per_cta;
    const int Y1 = min(Y0 + p.rows_per_cta, p.row_end);
    const uint8_t *src = static_cast<const uint8_t *>(p.src) + blockIdx.z * p.src_img_stride;
    uint8_t *dst = static_cast<uint8_t *>(p.dst) + blockIdx.z * p.dst_img_stride;
    const uint8_t *lut = static_cast<const uint8_t *>(p.lut);
    const int xt = X0 + lane * S;        // first output column of this lane
    const int ct = lane * S;             // column index of its window's left edge
    const uint32_t rank = p.rank;
    // staged column span [A, sx1): covers clamp(X0-r .. X0+TW+r-1)
    const int sx0 = max(0, X0 - r);
    const int sx1 = min(W, X0 + g.TW + r);
    const int A = ct_span_base(sx0);
    const bool aligned = ct_rows_aligned16(src, p.src_pitch);
    const int SPB = g.SPB;
    if (p.in_rows) {  // streaming: this tile's source rows have arrived
        if (lane == 0) stream_wait_rows_1(p, Y1 + r);
    }
    __syncwarp();

    // ---- per-tile snapshot of every column's initial span (rows clamp(Y0-r ..
    // Y0+r)) in a global workspace; every pass then initialises its column
    // histograms from it in O(columns) instead of rescanning n rows.
    // Layout per resident warp (reused for each of its tiles): cu[NCP] (16 B:
    // count below 16*b, bytes), off[NCP] (u16), then a heap of 16-B fine
    // chunks.  Two scans of the spans: before the coarse pass only cu; after
    // it, the fine chunks of the bins the fine passes will need (coarse bins
    // of the tile's outputs that are present in the column), packed per
    // column from chunk off[c] -- a live set small enough to stay in L2.
    const size_t heap_off = ((size_t)g.NCP * 18 + 15) & ~(size_t)15;
    const size_t snap_stride = heap_off + (size_t)g.NCP * 256;
    uint4 *snap_cu = nullptr, *snap_heap = nullptr;
    uint16_t *snap_off = nullptr;
    uint32_t needb[4] = {0, 0, 0, 0};  // byte masks of the needed bins
    auto snap_scan = [&](bool cu_too, bool chunks, uint32_t need) {
        uint8_t *scr = reinterpret_cast<uint8_t *>(colA) + lane * 260;  // lane-private column
        int heap_top = 0;
        for (int g0 = 0; g0 < g.NC; g0 += 32) {
            const int c = g0 + lane;
            const int gx = clampi(X0 - r + min(c, g.NC - 1), 0, W - 1);
            for (int i = 0; i < 65; ++i) reinterpret_cast<uint32_t *>(scr)[i] = 0;
            // 16 loads in flight per lane: the spans come from L2 and this
            // scan is latency-bound otherwise
            int j = -r;
            for (; j + 15 <= r; j += 16) {
                unsigned v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) v[u] = __ldg(src_row(p, src, clampi(Y0 + j + u, 0, H - 1)) + gx);
#pragma unroll
                for (int u = 0; u < 16; ++u) scr[v[u]] += 1;
            }
            for (; j + 3 <= r; j += 4) {
                unsigned v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = __ldg(src_row(p, src, clampi(Y0 + j + u, 0, H - 1)) + gx);
#pragma unroll
                for (int u = 0; u < 4; ++u) scr[v[u]] += 1;
            }
            for (; j <= r; ++j) scr[__ldg(src_row(p, src, clampi(Y0 + j, 0, H - 1)) + gx)] += 1;
            const uint32_t *w = reinterpret_cast<const uint32_t *>(scr);
            if (cu_too) {
                uint32_t acc = 0, cw[4] = {0, 0, 0, 0};
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    cw[q >> 2] |= acc << (8 * (q & 3));
                    acc += __vsadu4(w[4 * q], 0) + __vsadu4(w[4 * q + 1], 0) + __vsadu4(w[4 * q + 2], 0) +
                           __vsadu4(w[4 * q + 3], 0);
                }
                if (c < g.NC) snap_cu[c] = make_uint4(cw[0], cw[1], cw[2], cw[3]);
                if (!chunks) continue;
            }
            uint32_t pres = 0;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const uint32_t cb = w[4 * q] | w[4 * q + 1] | w[4 * q + 2] | w[4 * q + 3];
                pres |= (cb ? 1u : 0u) << q;
            }
            pres &= need;
            // warp exclusive scan of the chunk counts -> heap positions
            const int K = c < g.NC ? __popc(pres) : 0;
            int incl = K;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const int off = heap_top + incl - K;
            heap_top += __shfl_sync(0xffffffffu, incl, 31);
            if (c < g.NC) {
                snap_off[c] = (uint16_t)off;
                int k = off;
                for (uint32_t m = pres; m; m &= m - 1) {
                    const int q = __ffs(m) - 1;
                    snap_heap[k++] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
                }
            }
        }
        __syncwarp();
    };
    // precomputed snapshots (k_ctmf_pre_u8): cu at pre_t[gx], chunk b at pre_t[(1 + b) W + gx]
    const uint4 *pre_t = pre ? pre + (size_t)(blockIdx.z * tiles_y + ty) * 17 * W : nullptr;
    if (!PRE && snap && !pre) {
        const size_t slot = ((size_t)blockIdx.z * gridDim.x + blockIdx.x) * CT_WARPS + warp;
        uint8_t *rec = snap + slot * snap_stride;
        snap_cu = reinterpret_cast<uint4 *>(rec);
        snap_off = reinterpret_cast<uint16_t *>(rec + (size_t)g.NCP * 16);
        snap_heap = reinterpret_cast<uint4 *>(rec + heap_off);
        // snap_two_scans: cu first, chunks of the needed bins after the coarse
        // pass (small live set); else one scan storing every present bin
        snap_scan(true, !snap_two_scans, 0xffffu);
        if (!snap_two_scans) {
#pragma unroll
            for (int i = 0; i < 4; ++i) needb[i] = 0xffffffffu;
        }
    }
    const uint32_t nspan = (uint32_t)(2 * r + 1);

    // pass 0 = coarse; pass 1 = fine for coarse bin `beta`
    uint32_t tile_mask = 0;
    int beta = -1;
    // rows of the tile (relative to Y0) where coarse bin b = lane occurs,
    // recorded by the coarse pass; fine pass b sweeps only up to rlast and
    // resolves only from rfirst (before it, only the column histograms move)
    int rfirst = 1 << 30, rlast = -1;
    int yfirst = Y0, ylast = Y1 - 1;
    for (int pass = 0;; ++pass) {
        if (pass > 0) {
            if (tile_mask == 0) break;
            if (!PRE && pass == 1 && snap && !pre && snap_two_scans) {
                __syncwarp();
                snap_scan(false, true, tile_mask);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t nb = (tile_mask >> (4 * i)) & 15u;
                    needb[i] = ((nb & 1u) ? 0xffu : 0u) | ((nb & 2u) ? 0xff00u : 0u) |
                               ((nb & 4u) ? 0xff0000u : 0u) | ((nb & 8u) ? 0xff000000u : 0u);
                }
            }
            // descending: a pixel finalised by pass beta holds a value >= 16*beta,
            // which can never be mistaken for a lower coarse bin still pending
            beta = 31 - __clz(tile_mask);
            tile_mask &= ~(1u << beta);
        }
        const bool fine = pass > 0;
        if (fine) {
            yfirst = Y0 + __shfl_sync(0xffffffffu, rfirst, beta);
            ylast = Y0 + __shfl_sync(0xffffffffu, rlast, beta);
        }
        // bin of value v in this pass: 0..15, 16 = "below" (fine only), -1 = ignored
        auto bin_of = [&](unsigned v) -> int {
            if (!fine) return (int)(v >> 4);
            const int hb = (int)(v >> 4);
            return hb == beta ? (int)(v & 15) : (hb < beta ? 16 : -1);
        };
        auto bump = [&](int c, int b, int d) {
            if (b < 0) return;
            if (b == 16) {
                below[c] += d;
            } else {
                const int sl = ct_slot<S>(c);
                reinterpret_cast<uint16_t *>((b & 8) ? colB + sl : colA + sl)[b & 7] += d;
            }
        };
        // --- column histograms for row Y0: rows clamp(Y0-r .. Y0+r)
        __syncwarp();
        if (PRE || snap || pre) {
            for (int c = lane; c < g.NCP; c += 32) {
                uint32_t cnt[4] = {0, 0, 0, 0};
                uint32_t bl = 0;
                if (c < g.NC) {
                    const int gxc = clampi(X0 - r + c, 0, W - 1);
                    const uint4 cu = pre ? __ldcg(pre_t + gxc) : __ldcg(snap_cu + c);
                    // coarse counts = next cumulative - cumulative (bytewise, no borrow)
                    const uint32_t cwv[4] = {cu.x, cu.y, cu.z, cu.w};
                    const uint32_t nxt[4] = {__funnelshift_r(cwv[0], cwv[1], 8), __funnelshift_r(cwv[1], cwv[2], 8),
                                             __funnelshift_r(cwv[2], cwv[3], 8), __funnelshift_r(cwv[3], nspan, 8)};
                    uint32_t d[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) d[i] = nxt[i] - cwv[i];
                    if (!fine) {
#pragma unroll
                        for (int i = 0; i < 4; ++i) cnt[i] = d[i];
                    } else {
                        const uint32_t wsel = beta < 8 ? (beta < 4 ? cu.x : cu.y) : (beta < 12 ? cu.z : cu.w);
                        bl = (wsel >> (8 * (beta & 3))) & 0xffu;
                        const uint32_t dsel = beta < 8 ? (beta < 4 ? d[0] : d[1]) : (beta < 12 ? d[2] : d[3]);
                        if ((dsel >> (8 * (beta & 3))) & 0xffu) {
                            uint4 f;
                            if (pre) {
                                f = __ldcg(pre_t + (size_t)(1 + beta) * W + gxc);
                            } else {
                            // chunk index = off + number of present bins below beta
                            int k = __ldcg(snap_off + c);
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const int nb = min(max(beta - 4 * i, 0), 4);
                                const uint32_t sel = nb >= 4 ? 0xffffffffu : ((1u << (8 * nb)) - 1u);
                                k += __popc(__vcmpne4(d[i], 0) & sel & needb[i]) >> 3;
                            }
                            f = __ldcg(snap_heap + k);
                            }
                            cnt[0] = f.x; cnt[1] = f.y; cnt[2] = f.z; cnt[3] = f.w;
                        }
                    }
                }
                const int sl = c < g.NC ? ct_slot<S>(c) : c;
                colA[sl] = make_uint4(__byte_perm(cnt[0], 0, 0x4140), __byte_perm(cnt[0], 0, 0x4342),
                                      __byte_perm(cnt[1], 0, 0x4140), __byte_perm(cnt[1], 0, 0x4342));
                colB[sl] = make_uint4(__byte_perm(cnt[2], 0, 0x4140), __byte_perm(cnt[2], 0, 0x4342),
                                      __byte_perm(cnt[3], 0, 0x4140), __byte_perm(cnt[3], 0, 0x4342));
                below[c] = (uint16_t)bl;
            }
        } else {
        for (int c = lane; c < g.NCP; c += 32) {
            colA[c] = make_uint4(0, 0, 0, 0);
            colB[c] = make_uint4(0, 0, 0, 0);
            below[c] = 0;
        }
        for (int j0 = -r; j0 <= r; j0 += CT_STAGE_ROWS) {
            const int nr = min(CT_STAGE_ROWS, r - j0 + 1);
            int gr[CT_STAGE_ROWS];
#pragma unroll
            for (int k = 0; k < CT_STAGE_ROWS; ++k) gr[k] = clampi(Y0 + j0 + k, 0, H - 1);
            __syncwarp();
            ct_stage(p, src, stage, SPB, gr, nr, A, sx1, aligned, lane, &sbar);
            __syncwarp();
            // per column: count the batch's bins in 4-bit lanes of two words
            // (no shared-memory read-modify-write chain), then add the
            // expanded counts to the column record with two 16-B RMWs.
            for (int c = lane; c < g.NC; c += 32) {
                const int si = clampi(X0 - r + c, 0, W - 1) - A;
                uint64_t nib = 0;  // 16 four-bit counts (batch <= 8 rows)
                uint32_t nb = 0;   // below (fine passes)
                for (int k = 0; k < nr; ++k) {
                    const unsigned v = stage[k * SPB + si];
                    if (!fine) {
                        nib += 1ull << (4 * (v >> 4));
                    } else {
                        const int hb = (int)(v >> 4);
                        nib += (hb == beta) ? (1ull << (4 * (v & 15))) : 0ull;
                        nb += (hb < beta) ? 1u : 0u;
                    }
                }
                const uint32_t n0 = (uint32_t)nib, n1 = (uint32_t)(nib >> 32);
                const int sl = ct_slot<S>(c);
                if (n0) {
                    const uint32_t t = n0 >> 4;
                    uint4 h = colA[sl];
                    h.x += __byte_perm(n0, t, 0x7470) & 0x000f000fu;
                    h.y += __byte_perm(n0, t, 0x7571) & 0x000f000fu;
                    h.z += __byte_perm(n0, t, 0x7672) & 0x000f000fu;
                    h.w += __byte_perm(n0, t, 0x7773) & 0x000f000fu;
                    colA[sl] = h;
                }
                if (n1) {
                    const uint32_t t = n1 >> 4;
                    uint4 h = colB[sl];
                    h.x += __byte_perm(n1, t, 0x7470) & 0x000f000fu;
                    h.y += __byte_perm(n1, t, 0x7571) & 0x000f000fu;
                    h.z += __byte_perm(n1, t, 0x7672) & 0x000f000fu;
                    h.w += __byte_perm(n1, t, 0x7773) & 0x000f000fu;
                    colB[sl] = h;
                }
                if (nb) below[c] += nb;
            }
        }
        }
        __syncwarp();
        // --- lane window at x_t, row Y0
        uint32_t ws[8], wb;
        ct_window<S, MF>(colA, colB, below, fine, lane, r, g.NC, ws, wb);
        const int yend = fine ? ylast + 1 : Y1;
        for (int y = Y0; y < yend; ++y) {
            if (y > Y0) {
                // --- advance column histograms one row
                int gr[CT_STAGE_ROWS];
                gr[0] = clampi(y - r - 1, 0, H - 1);
                gr[1] = clampi(y + r, 0, H - 1);
                if (gr[0] != gr[1]) {
                    __syncwarp();
                    ct_stage(p, src, stage, SPB, gr, 2, A, sx1, aligned, lane, &sbar);
                    __syncwarp();
                    // two counter updates per column; U columns per batch with all
                    // loads issued before any store (addresses are distinct;
                    // ignored values hit a dummy counter)
                    constexpr int U = 4;
                    uint16_t *h16 = reinterpret_cast<uint16_t *>(colA);  // colA | colB | below | dummy
                    const int offB = g.NCP * 8, offBelow = 2 * g.NCP * 8, dummy = offBelow + g.NCP;
                    auto idx_of = [&](int c, int sl, unsigned v) -> int {
                        if (!fine) return ((v & 0x80) ? offB : 0) + sl * 8 + (int)((v >> 4) & 7);
                        const int hb = (int)(v >> 4);
                        const int in = ((v & 8) ? offB : 0) + sl * 8 + (int)(v & 7);
                        return hb == beta ? in : (hb < beta ? offBelow + c : dummy);
                    };
                    for (int c0 = lane; c0 < g.NC; c0 += 32 * U) {
                        int io[U], ii[U];
                        uint16_t vo[U], vi[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int c = min(c0 + 32 * u, g.NC - 1);
                            const int si = clampi(X0 - r + c, 0, W - 1) - A;
                            const int sl = ct_slot<S>(c);
                            const unsigned a = stage[si], b = stage[SPB + si];
                            io[u] = idx_of(c, sl, a);
                            ii[u] = idx_of(c, sl, b);
                            if (c0 + 32 * u >= g.NC || io[u] == ii[u]) io[u] = ii[u] = dummy;
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            vo[u] = h16[io[u]];
                            vi[u] = h16[ii[u]];
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            if (io[u] != dummy) h16[io[u]] = vo[u] - 1;
                            if (ii[u] != dummy) h16[ii[u]] = vi[u] + 1;
                        }
                    }
                }
                __syncwarp();
                if (y < yfirst) continue;  // no output of this row needs this pass
                // --- lane window at x_t for the new row, from the column histograms
                ct_window<S, MF>(colA, colB, below, fine, lane, r, g.NC, ws, wb);
            } else if (y < yfirst) {
                continue;
            }
            // --- slide right over the lane's S outputs
            uint32_t w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = ws[i];
            uint32_t wbl = wb;
            uint8_t *drow = dst + (int64_t)(y - p.row_begin) * p.dst_pitch;
            uint32_t outw[S / 4];
            uint32_t row_mask = 0;  // coarse pass: bins of this row's outputs
            const bool full = (xt + S <= W) && ((reinterpret_cast<uintptr_t>(drow + xt) & 3) == 0);
            if (fine) {
                if (full) {
#pragma unroll
                    for (int q = 0; q < S / 4; ++q) outw[q] = *reinterpret_cast<const uint32_t *>(drow + xt + 4 * q);
                } else {
#pragma unroll
                    for (int q = 0; q < S / 4; ++q) outw[q] = 0;
                    for (int s = 0; s < S; ++s)
                        if (xt + s < W) outw[s >> 2] |= (uint32_t)drow[xt + s] << (8 * (s & 3));
                }
            }
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (s > 0) {
                    const int cin = ct + s + 2 * r, cout = ct + s - 1;
                    const int si = ct_slot<S>(cin), so = ct_slot<S>(cout);
                    const uint4 ia = colA[si], ib = colB[si], oa = colA[so], ob = colB[so];
                    w[0] = w[0] + ia.x - oa.x; w[1] = w[1] + ia.y - oa.y;
                    w[2] = w[2] + ia.z - oa.z; w[3] = w[3] + ia.w - oa.w;
                    w[4] = w[4] + ib.x - ob.x; w[5] = w[5] + ib.y - ob.y;
                    w[6] = w[6] + ib.z - ob.z; w[7] = w[7] + ib.w - ob.w;
                    if (fine) wbl = wbl + below[cin] - below[cout];
                }
                const uint32_t cur = (outw[s >> 2] >> (8 * (s & 3))) & 0xffu;
                if (!fine) {
                    uint32_t k = rank;
                    const int b = ct_descend(w, k);
                    row_mask |= (xt + s < W) ? (1u << b) : 0u;
                    outw[s >> 2] = (s & 3) ? (outw[s >> 2] | ((uint32_t)b << (8 * (s & 3)))) : (uint32_t)b;
                } else if ((int)cur == beta) {
                    uint32_t k = rank - wbl;
                    const int b = ct_descend(w, k);
                    uint32_t v = (uint32_t)(beta << 4) | (uint32_t)b;
                    if (lut) v = __ldg(lut + v);
                    outw[s >> 2] = (outw[s >> 2] & ~(0xffu << (8 * (s & 3)))) | (v << (8 * (s & 3)));
                }
            }
            if (!fine) {
                const uint32_t rm = __reduce_or_sync(0xffffffffu, row_mask);
                tile_mask |= rm;
                if (lane < 16 && ((rm >> lane) & 1u)) {
                    if (rlast < 0) rfirst = y - Y0;
                    rlast = y - Y0;
                }
            }
            if (full) {
#pragma unroll
                for (int q = 0; q < S / 4; ++q) *reinterpret_cast<uint32_t *>(drow + xt + 4 * q) = outw[q];
            } else {
                for (int s = 0; s < S; ++s)
                    if (xt + s < W) drow[xt + s] = (uint8_t)(outw[s >> 2] >> (8 * (s & 3)));
            }
            __syncwarp();
        }
        __syncwarp();
    }
    __syncwarp();
    if (p.out_px && lane == 0) stream_signal_1(p, Y0, Y1, X0, X0 + g.TW);
    }  // tiles
}

}  // namespace mtb
