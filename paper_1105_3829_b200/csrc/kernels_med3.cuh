// kernels_med3.cuh -- 3x3 median (r = 1) of 8-bit frames, register-resident.
//
// The r = 1 filter is bound by moving the frame, not by selection: 12
// min/max per pair of outputs.  So the data path is what this kernel is
// about (k_sortnet<3> staged byte-wise through shared memory and wrote
// single bytes: 10% of the HBM roofline).
//
//   * Lane t of a warp owns 8 adjacent output columns x0 = X + 8t and walks
//     DOWN a band of RT rows.  Each input row is one coalesced 64-bit load
//     per lane (256 B per warp); the left / right neighbour columns come
//     from lanes t-1 / t+1 by shuffle (lanes 0 and 31 load one byte).
//     Rows are prefetched two iterations (4 rows) ahead.
//   * The 10 bytes are widened into 9 packed columns Q_m = (col x0-1+m,
//     col x0+m) as u16 pairs: output pair (x0+2k, x0+2k+1) has window
//     columns Q_2k, Q_2k+1, Q_2k+2, and VIMNMX.U16x2 serves both outputs.
//   * Two output rows per step share the sorted core (rows y, y+1) of every
//     packed column; each adds its own third row (y-1 or y+2) as a 3-sort
//     (min, med, max).  The median of 3 sorted columns is
//         med3( max(mins), med3(meds), min(maxes) )
//     (the classic 3x3 selection, exact).
//   * Outputs are packed to 8 bytes and written with one 64-bit store.
//
// Replicate borders: columns clamp in the loads (partial lanes at the right
// edge load byte-wise), rows clamp to [0, H-1].  Median rank only.
#pragma once
#include "common.cuh"

namespace mtb {

struct Med3Raw {
    uint32_t lo, hi, e;  // cols x0..x0+3, x0+4..x0+7; e: lane 0 col x0-1, lane 31 col x0+8
};

__device__ __forceinline__ uint32_t med3u2(uint32_t a, uint32_t b, uint32_t c) {
    return __vmaxu2(__vminu2(a, b), __vminu2(__vmaxu2(a, b), c));
}

// one warp: output columns [x0 .. x0+8) of lane t, rows [Y0, Y1).
// FULL: every lane's 8 columns lie inside the image and the rows are
// 8-byte aligned (one 64-bit load / store per lane and row).
template <bool FULL>
__device__ __forceinline__ void med3_band(const SlabParams &p, const uint8_t *src, uint8_t *dst, int x0,
                                          int Y0, int Y1) {
    const int lane = threadIdx.x & 31;
    const int W = p.W, H = p.H;
    const uint8_t *lut = static_cast<const uint8_t *>(p.lut);
    // rows Y0-1 .. Y1 are the ones this band reads (clamped to the image)
    const int ylo = max(Y0 - 1, 0), yhi = min(Y1, H - 1);
    const bool edge = lane == 0 || lane == 31;
    const int xe = clampi(lane == 0 ? x0 - 1 : x0 + 8, 0, W - 1);  // lane 0 / 31: outer neighbour

    // 32-bit row offsets (the host checks src_rows * src_pitch < 2^31)
    const int pitch = (int)p.src_pitch, row0 = p.src_row0;
    auto load = [&](int y) {
        const uint8_t *row = src + (clampi(y, ylo, yhi) - row0) * pitch;
        Med3Raw v;
        if (FULL) {
            const uint2 w = __ldg(reinterpret_cast<const uint2 *>(row + x0));
            v.lo = w.x;
            v.hi = w.y;
        } else {
            uint32_t b[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) b[i] = __ldg(row + clampi(x0 + i, 0, W - 1));
            v.lo = b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24);
            v.hi = b[4] | (b[5] << 8) | (b[6] << 16) | (b[7] << 24);
        }
        v.e = edge ? __ldg(row + xe) : 0u;
        return v;
    };
    // 9 packed columns Q_m = (col x0-1+m, col x0+m)
    auto pack = [&](const Med3Raw &v, uint32_t (&q)[9]) {
        const uint32_t up = __shfl_up_sync(0xffffffffu, v.hi, 1) >> 24;     // col x0-1 from lane-1
        const uint32_t dn = __shfl_down_sync(0xffffffffu, v.lo, 1) & 0xffu;  // col x0+8 from lane+1
        const uint32_t L = lane == 0 ? v.e : up;
        const uint32_t R = lane == 31 ? v.e : dn;
        const uint32_t mid = __byte_perm(v.lo, v.hi, 0x5432);  // cols x0+2 .. x0+5
        q[0] = __byte_perm(v.lo, L, 0x5054);   // (x0-1, x0)
        q[1] = __byte_perm(v.lo, 0, 0x4140);   // (x0, x0+1)
        q[2] = __byte_perm(v.lo, 0, 0x4241);   // (x0+1, x0+2)
        q[3] = __byte_perm(v.lo, 0, 0x4342);   // (x0+2, x0+3)
        q[4] = __byte_perm(mid, 0, 0x4241);    // (x0+3, x0+4)
        q[5] = __byte_perm(v.hi, 0, 0x4140);   // (x0+4, x0+5)
        q[6] = __byte_perm(v.hi, 0, 0x4241);   // (x0+5, x0+6)
        q[7] = __byte_perm(v.hi, 0, 0x4342);   // (x0+6, x0+7)
        q[8] = __byte_perm(v.hi, R, 0x5453);   // (x0+7, x0+8)
    };
    auto store = [&](int y, const uint32_t (&mn)[9], const uint32_t (&md)[9], const uint32_t (&mx)[9]) {
        uint32_t o[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t a = __vmaxu2(__vmaxu2(mn[2 * k], mn[2 * k + 1]), mn[2 * k + 2]);
            const uint32_t c = __vminu2(__vminu2(mx[2 * k], mx[2 * k + 1]), mx[2 * k + 2]);
            const uint32_t b = med3u2(md[2 * k], md[2 * k + 1], md[2 * k + 2]);
            o[k] = med3u2(a, b, c);  // (med3 via min/max: 4 ops, as the sum form)
        }
        uint32_t w0 = __byte_perm(o[0], o[1], 0x6420), w1 = __byte_perm(o[2], o[3], 0x6420);
        uint8_t *d = dst + (int64_t)(y - p.row_begin) * p.dst_pitch + x0;
        if (lut) {
            uint32_t b[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                b[i] = __ldg(lut + ((w0 >> (8 * i)) & 0xffu));
                b[4 + i] = __ldg(lut + ((w1 >> (8 * i)) & 0xffu));
            }
            w0 = b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24);
            w1 = b[4] | (b[5] << 8) | (b[6] << 16) | (b[7] << 24);
        }
        if (FULL) {
            *reinterpret_cast<uint2 *>(d) = make_uint2(w0, w1);
        } else if (x0 < W) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (x0 + i < W) d[i] = (uint8_t)((i < 4 ? w0 : w1) >> (8 * (i & 3)));
        }
    };

    // packed rows y-1 (qa) and y (qb); raw rows y+1, y+2 (ready) and y+3, y+4 (in flight)
    uint32_t qa[9], qb[9];
    {
        const Med3Raw r0 = load(Y0 - 1), r1 = load(Y0);
        pack(r0, qa);
        pack(r1, qb);
    }
    Med3Raw n1 = load(Y0 + 1), n2 = load(Y0 + 2);
    Med3Raw f1 = load(Y0 + 3), f2 = load(Y0 + 4);
#pragma unroll 2
    for (int y = Y0; y < Y1; y += 2) {
        uint32_t qc[9], qd[9];
        pack(n1, qc);
        pack(n2, qd);
        n1 = f1;
        n2 = f2;
        f1 = load(y + 5);
        f2 = load(y + 6);
        uint32_t mn[9], md[9], mx[9];
        // 3-sort of every packed column: min3, max3 (VIMNMX3) and the sum
        // minus both (lanes <= 765: no carry / borrow across lanes)
#pragma unroll
        for (int m = 0; m < 9; ++m) {
            mn[m] = __vminu2(__vminu2(qa[m], qb[m]), qc[m]);  // row y: rows y-1, y, y+1
            mx[m] = __vmaxu2(__vmaxu2(qa[m], qb[m]), qc[m]);
            md[m] = qa[m] + qb[m] + qc[m] - mn[m] - mx[m];
        }
        store(y, mn, md, mx);
        if (y + 1 < Y1) {
#pragma unroll
            for (int m = 0; m < 9; ++m) {
                mn[m] = __vminu2(__vminu2(qb[m], qc[m]), qd[m]);  // row y+1: rows y, y+1, y+2
                mx[m] = __vmaxu2(__vmaxu2(qb[m], qc[m]), qd[m]);
                md[m] = qb[m] + qc[m] + qd[m] - mn[m] - mx[m];
            }
            store(y + 1, mn, md, mx);
        }
#pragma unroll
        for (int m = 0; m < 9; ++m) {
            qa[m] = qc[m];
            qb[m] = qd[m];
        }
    }
}

// CTA = 4 warps side by side (1024 columns) x p.rows_per_cta rows; the
// host sizes the row bands so the grid is one wave.
__global__ void __launch_bounds__(128) k_med3_u8(SlabParams p) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int X = (blockIdx.x * 4 + warp) * 256;
    const int x0 = X + lane * 8;
    const int Y0 = p.row_begin + blockIdx.y * p.rows_per_cta;
    const int Y1 = min(Y0 + p.rows_per_cta, p.row_end);
    const uint8_t *src = static_cast<const uint8_t *>(p.src) + blockIdx.z * p.src_img_stride;
    uint8_t *dst = static_cast<uint8_t *>(p.dst) + blockIdx.z * p.dst_img_stride;
    stream_wait_rows(p, Y1 + 1);
    // vector path: the whole warp inside the image, rows 8-byte aligned
    const bool aligned = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) |
                           (uintptr_t)p.src_pitch | (uintptr_t)p.dst_pitch) & 7) == 0;
    if (X < p.W && Y0 < Y1) {
        if (aligned && X + 256 <= p.W)
            med3_band<true>(p, src, dst, x0, Y0, Y1);
        else
            med3_band<false>(p, src, dst, x0, Y0, Y1);
    }
    stream_signal(p, Y0, Y1, blockIdx.x * 1024, blockIdx.x * 1024 + 1024);
}

// ---------------------------------------------------------------------------
// k_med3t_u8: the same selection with the band's rows staged by TMA bulk
// copies.  The register kernel above keeps only ~4 rows per warp in flight,
// so on a one-wave grid it is latency-bound (Little's law).  Here thread 0
// of each CTA issues, at launch, one cp.async.bulk per source row of the
// CTA's whole band (RT + 2 rows x 1056 B, each completing on its own
// mbarrier): the entire frame is requested in the first microsecond, and
// threads walk down their 8 columns as rows land.
//
// CTA = 128 threads x 8 columns = 1024 output columns; staged row segment
// = columns [X-16, X+1040) (16-byte aligned, clipped to the image).
// Per output row and thread: one LDS.64 (own 8 columns) + two byte loads
// (left / right neighbours, clamped to the image); 9 packed columns, each
// 3-sorted from (min3, max3, sum - min3 - max3) with 3-input VIMNMX3.U16x2;
// four pair medians med3(max3(mins), med3(meds), min3(maxes)).
// Requires W % 16 == 0 and 16-byte aligned rows (host-checked).
constexpr int M3T_SEG = 1056;

__device__ __forceinline__ uint32_t m3t_smem(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t min3u2(uint32_t a, uint32_t b, uint32_t c) { return __vminu2(__vminu2(a, b), c); }
__device__ __forceinline__ uint32_t max3u2(uint32_t a, uint32_t b, uint32_t c) { return __vmaxu2(__vmaxu2(a, b), c); }

// median of three packed u16 pairs: a + b + c - min3 - max3 (lanes <= 765,
// no carry or borrow crosses a lane)
__device__ __forceinline__ uint32_t med3s(uint32_t a, uint32_t b, uint32_t c) {
    return a + b + c - min3u2(a, b, c) - max3u2(a, b, c);
}

__global__ void __launch_bounds__(128) k_med3t_u8(SlabParams p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    const int W = p.W, H = p.H;
    const int X = blockIdx.x * 1024;
    const int Y0 = p.row_begin + blockIdx.y * p.rows_per_cta;
    const int Y1 = min(Y0 + p.rows_per_cta, p.row_end);
    const int NR = Y1 - Y0 + 2;  // staged rows Y0-1 .. Y1
    const uint8_t *src = static_cast<const uint8_t *>(p.src) + blockIdx.z * p.src_img_stride;
    uint8_t *dst = static_cast<uint8_t *>(p.dst) + blockIdx.z * p.dst_img_stride;
    const uint8_t *lut = static_cast<const uint8_t *>(p.lut);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);  // [NR]
    uint8_t *rows = smem_raw + ((NR * 8 + 127) & ~127);      // [NR][M3T_SEG]
    stream_wait_rows(p, Y1 + 1);
    // staged column span [gx0, gx1): multiples of 16 (W % 16 == 0)
    const int gx0 = max(X - 16, 0), gx1 = min(X + 1040, W);
    const int off = gx0 - (X - 16);  // 16 at the left image edge, else 0
    const uint32_t bytes = (uint32_t)(gx1 - gx0);
    if (tid == 0) {
        for (int i = 0; i < NR; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(m3t_smem(bar + i)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < NR; ++i) {
            const int gy = clampi(Y0 - 1 + i, 0, H - 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m3t_smem(bar + i)),
                         "r"(bytes) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    m3t_smem(rows + i * M3T_SEG + off)),
                "l"(src_row(p, src, gy) + gx0), "r"(bytes), "r"(m3t_smem(bar + i))
                : "memory");
        }
    }
    __syncthreads();  // barriers initialised before anyone waits
    const int x0 = X + 8 * tid;
    const bool act = x0 < W;  // W % 16 == 0: an active thread's 8 columns are all inside
    // smem offsets of this thread's 8 columns and its clamped neighbours
    const int ow = 16 + 8 * tid;
    const int ol = act ? 16 + clampi(x0 - 1, 0, W - 1) - X : 16;
    const int orr = act ? 16 + min(x0 + 8, W - 1) - X : 16;
    auto wait_row = [&](int i) {
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n .reg .pred P;\n"
                " mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n"
                " selp.b32 %0, 1, 0, P;\n}\n"
                : "=r"(done)
                : "r"(m3t_smem(bar + i)), "r"(0u)
                : "memory");
        }
    };
    // packed columns Q_m = (col x0-1+m, col x0+m), m = 0..8, of staged row i
    auto pack = [&](int i, uint32_t (&q)[9]) {
        wait_row(i);
        const uint8_t *rb = rows + i * M3T_SEG;
        const uint2 v = *reinterpret_cast<const uint2 *>(rb + ow);
        const uint32_t L = rb[ol], R = rb[orr];
        const uint32_t mid = __byte_perm(v.x, v.y, 0x5432);  // cols x0+2 .. x0+5
        q[0] = __byte_perm(v.x, L, 0x5054);
        q[1] = __byte_perm(v.x, 0, 0x4140);
        q[2] = __byte_perm(v.x, 0, 0x4241);
        q[3] = __byte_perm(v.x, 0, 0x4342);
        q[4] = __byte_perm(mid, 0, 0x4241);
        q[5] = __byte_perm(v.y, 0, 0x4140);
        q[6] = __byte_perm(v.y, 0, 0x4241);
        q[7] = __byte_perm(v.y, 0, 0x4342);
        q[8] = __byte_perm(v.y, R, 0x5453);
    };
    // one output row from its three packed input rows
    auto row_out = [&](const uint32_t (&qa)[9], const uint32_t (&qb)[9], const uint32_t (&qc)[9], uint8_t *d) {
        uint32_t mn[9], md[9], mx[9];
#pragma unroll
        for (int m = 0; m < 9; ++m) {
            mn[m] = min3u2(qa[m], qb[m], qc[m]);
            mx[m] = max3u2(qa[m], qb[m], qc[m]);
            md[m] = qa[m] + qb[m] + qc[m] - mn[m] - mx[m];
        }
        uint32_t o[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            o[k] = med3s(max3u2(mn[2 * k], mn[2 * k + 1], mn[2 * k + 2]), med3s(md[2 * k], md[2 * k + 1], md[2 * k + 2]),
                         min3u2(mx[2 * k], mx[2 * k + 1], mx[2 * k + 2]));
        uint32_t w0 = __byte_perm(o[0], o[1], 0x6420), w1 = __byte_perm(o[2], o[3], 0x6420);
        if (lut) {
            uint32_t b[8];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                b[j] = __ldg(lut + ((w0 >> (8 * j)) & 0xffu));
                b[4 + j] = __ldg(lut + ((w1 >> (8 * j)) & 0xffu));
            }
            w0 = b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24);
            w1 = b[4] | (b[5] << 8) | (b[6] << 16) | (b[7] << 24);
        }
        if (act) *reinterpret_cast<uint2 *>(d) = make_uint2(w0, w1);
    };
    // two output rows per step (two independent selection chains per
    // thread); staged rows i-2 .. i+1
    uint32_t qa[9], qb[9];
    pack(0, qa);
    pack(1, qb);
    uint8_t *d = dst + (int64_t)(Y0 - p.row_begin) * p.dst_pitch + x0;
    int i = 2;
#pragma unroll 1
    for (; i + 1 < NR; i += 2) {
        uint32_t qc[9], qd[9];
        pack(i, qc);
        pack(i + 1, qd);
        row_out(qa, qb, qc, d);
        row_out(qb, qc, qd, d + p.dst_pitch);
        d += 2 * p.dst_pitch;
#pragma unroll
        for (int m = 0; m < 9; ++m) {
            qa[m] = qc[m];
            qb[m] = qd[m];
        }
    }
    if (i < NR) {
        uint32_t qc[9];
        pack(i, qc);
        row_out(qa, qb, qc, d);
    }
    stream_signal(p, Y0, Y1, X, X + 1024);
}

}  // namespace mtb
