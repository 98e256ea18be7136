// kernels_bandtc.cuh -- 8-bit rank filter: window histograms as band-matrix
// products on the 5th-generation tensor cores (tcgen05.mma kind::i8, operands
// in shared memory / tensor memory, accumulators in tensor memory).
//
// Same decomposition as kernels_bandmma.cuh (the reference's per-column trees
// + window merge, _kernels.py:115-194, and extract_u, :229-253): the CTA
// keeps, for every column c of its halo'd stripe, the 256-bin histogram of the
// column's vertical span as byte planes fine[v][c] plus 16 cumulative coarse
// planes cum[j][c] (pixels below 16 j), moved down one row with shared-memory
// atomics.  The window count of pixel x for a plane P is
//     sum_c Band[x][c] * P[c],     Band[x][c] = 1 iff x <= c <= x + 2r.
//
// Here one tcgen05.mma computes it for 128 adjacent pixels (M = 128) x N
// planes x 32 columns:
//   * A = the band tile (128 x 32 zeros / ones).  It only depends on the
//     k-step, so all NKA = ceil((128 + 2r) / 32) tiles live in TENSOR MEMORY
//     for the whole launch (8 columns each, written once with tcgen05.st).
//   * B = the plane bytes, read by the tensor core straight from shared
//     memory through a matrix descriptor: no B-fragment loads into registers
//     (the mma.sync kernel re-read the planes 6.7 times per row that way).
//     For that the planes use the canonical K-major no-swizzle layout: groups
//     of 8 planes, 16-byte column chunks, address(p, c) = (p >> 3) GSZ +
//     (c >> 4) 128 + (p & 7) 16 + (c & 15).
//   * D = s32 accumulators in tensor memory; each thread reads ITS pixel's
//     counts with tcgen05.ld (lane = pixel, registers = bins): no transpose
//     through shared memory, one thread descends one pixel.
// Per row and 128-pixel tile: one N = 16 product over the cumulative planes
// (every pixel's exact coarse bin and the count below it) and one N = NF
// product over the value planes of NF / 16 coarse bins from a base predicted
// one row up.  A pixel whose coarse bin lies outside that window is a miss: the
// tile repeats the value product from the lowest missed bin (its planes are
// still those of this row) -- exact for any image.
//
// All arithmetic is exact integer counting (r <= 127: u8 column counts).
#pragma once
#include "common.cuh"

namespace mtb {

constexpr int BT_M = 128;          // pixels per product (tensor-memory lanes)
constexpr int BT_MAXTILES = 4;     // 128-pixel tiles per CTA (512 threads)
constexpr int BT_TMEM_COLS = 512;  // the whole tensor memory (one CTA per SM)
constexpr int BT_ACOL0 = 416;      // band tiles: columns 416 .. 416 + 8 NKA (NKA <= 12)
constexpr int BT_CUMG = 0, BT_FINEG = 2;  // plane groups: cum[0..15] = groups 0, 1; fine[v] = group 2 + v / 8

__host__ __device__ constexpr int bt_nka(int r) { return (BT_M + 2 * r + 31) / 32; }
__host__ __device__ constexpr int bt_ncols(int TW, int r) { return TW - BT_M + 32 * bt_nka(r); }
__host__ __device__ constexpr int bt_groups(int NF) { return 32 + NF / 8 + 2; }  // cum, fine, zero tail of a window from bin 15
__host__ __device__ constexpr size_t bt_smem(int TW, int r, int NF) {
    const size_t planes = (size_t)bt_groups(NF) * (bt_ncols(TW, r) / 16) * 128;
    return planes > 120 * 1024 ? planes : 120 * 1024;  // (at least 120 KB: one CTA per SM, it owns all of tensor memory)
}

__device__ __forceinline__ uint32_t bt_smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: 8 rows x 16 B core matrices; lbo = stride of the second
// 16-byte K chunk, sbo = stride between groups of 8 rows; version 1 (Blackwell)
__device__ __forceinline__ uint64_t bt_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr & 0x3ffffu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3fffu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fffu) << 32) | ((uint64_t)1 << 46);
}
// D[tmem_d] (+)= A[tmem_a] x B[desc]: u8 x u8 -> s32
// (called by a whole converged warp with warp-uniform operands: one elected lane issues)
__device__ __forceinline__ void bt_mma(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p, q;\n elect.sync _|q, 0xffffffff;\n setp.ne.b32 p, %4, 0;\n"
        " @q tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n}\n"
        ::"r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc), "r"(0u) : "memory");
}
__device__ __forceinline__ void bt_commit(uint32_t bar) {
    asm volatile(
        "{\n .reg .pred q;\n elect.sync _|q, 0xffffffff;\n"
        " @q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bt_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.b32 %0, 1, 0, P;\n}\n"
                     : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void bt_ld16(uint32_t taddr, int (&v)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(taddr) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// smallest j with f[0] + .. + f[j] >= k (1 <= k <= sum of the 16 counts)
__device__ __forceinline__ int bt_descend16(const int (&f)[16], int k) {
    const int s8 = f[0] + f[1] + f[2] + f[3] + f[4] + f[5] + f[6] + f[7];
    const bool p8 = s8 < k;
    k -= p8 ? s8 : 0;
    int g[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) g[i] = p8 ? f[8 + i] : f[i];
    const int s4 = g[0] + g[1] + g[2] + g[3];
    const bool p4 = s4 < k;
    k -= p4 ? s4 : 0;
    const int h0 = p4 ? g[4] : g[0], h1 = p4 ? g[5] : g[1], h2 = p4 ? g[6] : g[2];
    const int s2 = h0 + h1;
    const bool p2 = s2 < k;
    k -= p2 ? s2 : 0;
    const int e0 = p2 ? h2 : h0;
    const bool p1 = e0 < k;
    return (p8 ? 8 : 0) + (p4 ? 4 : 0) + (p2 ? 2 : 0) + (p1 ? 1 : 0);
}

// NF: value planes of the keyed product (32: two coarse bins, 64: four).
// Block = TW threads (TW = 128 MT output columns, thread = pixel); grid =
// (stripes, row slabs, images).
template <int NF, bool STREAM>
__global__ void __launch_bounds__(BT_M * BT_MAXTILES, 1) k_bandtc_u8(SlabParams p, int TW) {
    static_assert(NF == 32 || NF == 64, "two or four coarse bins per keyed window");
    constexpr int NB = NF / 16;             // coarse bins of the keyed window
    constexpr int DST = NF + 32;            // tensor-memory columns per tile: NF value bins | 16 cumulative | pad
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t s_bar[BT_MAXTILES];
    __shared__ uint32_t s_tmem;
    __shared__ int s_lo[2][BT_MAXTILES], s_hi[2][BT_MAXTILES], s_minv[2][BT_MAXTILES], s_retry[BT_MAXTILES];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NTH = blockDim.x;
    const int tile = tid >> 7, m = tid & 127;  // the thread's tile and its pixel = tensor-memory lane
    const int r = p.radius, r2 = 2 * r, H = p.H, W = p.W;
    const int NKA = bt_nka(r), NCOLS = bt_ncols(TW, r), NC = TW + r2, NPC = NCOLS >> 4, GSZ = NPC * 128;
    uint32_t *planew = reinterpret_cast<uint32_t *>(smem_raw);
    const int X0 = blockIdx.x * TW;
    const int y0 = p.row_begin + blockIdx.y * p.rows_per_cta;
    if (y0 >= p.row_end) return;  // CTA-uniform (barriers below)
    const int y1 = min(y0 + p.rows_per_cta, p.row_end);
    if (STREAM) stream_wait_rows(p, y1 + r);
    const uint8_t *src = static_cast<const uint8_t *>(p.src) + blockIdx.z * p.src_img_stride;
    uint8_t *dst = static_cast<uint8_t *>(p.dst) + blockIdx.z * p.dst_img_stride;
    const uint8_t *lut = static_cast<const uint8_t *>(p.lut);

    // ---- tensor memory, barriers, planes of row y0
    if (tid < BT_MAXTILES) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bt_smem_u32(&s_bar[tid])) : "memory");
        s_lo[0][tid] = s_lo[1][tid] = 255;
        s_hi[0][tid] = s_hi[1][tid] = -1;
        s_minv[0][tid] = s_minv[1][tid] = 255;
        s_retry[tid] = 255;
    }
    if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(bt_smem_u32(&s_tmem)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    const int nplw = bt_groups(NF) * GSZ / 4;
    for (int i = tid; i < nplw; i += NTH) planew[i] = 0;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = s_tmem;
    // band tiles into tensor memory: lane = pixel m, k-step s at columns ACOL0 + 8 s, byte k = column 32 s + k
    if (tile == 0) {
        for (int s = 0; s < NKA; ++s) {
            uint32_t w[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                w[j] = 0;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int c = 32 * s + 4 * j + b;
                    w[j] |= ((c >= m && c <= m + r2) ? 1u : 0u) << (8 * b);
                }
            }
            const uint32_t ta = tm + ((uint32_t)(32 * warp) << 16) + BT_ACOL0 + 8 * s;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                         ::"r"(ta), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]) : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    // word of (plane pl, word column wc = c >> 2) in the blocked layout
    auto pword = [&](int pl, int wc) { return ((pl >> 3) * GSZ + (wc >> 2) * 128 + (pl & 7) * 16 + (wc & 3) * 4) >> 2; };
    // Slot s = (byte lane, word column): the lanes of a warp hit distinct words.
    const int nwords = (NC + 3) >> 2, nslots = 4 * nwords;
    for (int s = tid; s < nslots; s += NTH) {
        const int bl = s / nwords, wc = s - bl * nwords, c = 4 * wc + bl;
        if (c >= NC) continue;
        const int gx = clampi(X0 - r + c, 0, W - 1);
        const uint32_t one = 1u << (8 * bl);
        int j = -r;
        for (; j + 7 <= r; j += 8) {  // 8 loads in flight (the rows come from L2)
            unsigned v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(src_row(p, src, clampi(y0 + j + u, 0, H - 1)) + gx);
#pragma unroll
            for (int u = 0; u < 8; ++u) atomicAdd(planew + pword(16 + (int)v[u], wc), one);
        }
        for (; j <= r; ++j)
            atomicAdd(planew + pword(16 + (int)__ldg(src_row(p, src, clampi(y0 + j, 0, H - 1)) + gx), wc), one);
    }
    __syncthreads();
    // cumulative planes from the value planes (bytewise; a column's total is n <= 255)
    for (int wc = tid; wc < nwords; wc += NTH) {
        uint32_t run = 0;
        for (int j = 0; j < 16; ++j) {
            planew[pword(j, wc)] = run;
#pragma unroll
            for (int v = 0; v < 16; ++v) run += planew[pword(16 + 16 * j + v, wc)];
        }
    }

    // ---- row updates: one slot per thread (more: a loop), pixels a row ahead
    int pwc = -1;  // the slot's word column (-1: no slot)
    uint32_t pone = 0;
    const uint8_t *pin = src;
    {
        const int bl = tid / nwords, wc = tid - bl * nwords, c = 4 * wc + bl;
        if (tid < nslots && c < NC) pwc = wc;
        pin = src_row(p, src, p.src_row0) + clampi(X0 - r + min(c, NC - 1), 0, W - 1);
        pone = 1u << (8 * (bl & 3));
    }
    unsigned pvo = 0, pvi = 0;
    const uint8_t *pout = pin + (int64_t)(clampi(y0 - r, 0, H - 1) - p.src_row0) * p.src_pitch;
    const uint8_t *pent = pin + (int64_t)(clampi(y0 + 1 + r, 0, H - 1) - p.src_row0) * p.src_pitch;
    auto prefetch = [&](int yn) {  // update yn-1 -> yn: leaving row yn-r-1, entering row yn+r
        if (pwc >= 0) {
            pvo = __ldg(pout);
            pvi = __ldg(pent);
        }
        if (yn - r > 0 && yn - r <= H - 1) pout += p.src_pitch;
        if (yn + 1 + r <= H - 1) pent += p.src_pitch;
    };
    auto move = [&](int wc, uint32_t one, unsigned vo, unsigned vi) {
        atomicAdd(planew + pword(16 + (int)vo, wc), 0u - one);
        atomicAdd(planew + pword(16 + (int)vi, wc), one);
        // cum[j] counts the pixels below 16 j
        const int a = (int)(vo >> 4), b = (int)(vi >> 4);
        const uint32_t d = b > a ? 0u - one : one;
        for (int j = min(a, b) + 1; j <= max(a, b); ++j) atomicAdd(planew + pword(j, wc), d);
    };

    // ---- products: thread 0 of every tile issues; all 128 threads of the tile read
    const bool issuer = m == 0;                     // the tile's bookkeeping thread
    const bool issue_warp = (warp & 3) == 0;        // the tile's first warp issues its products (one elected lane)
    const uint32_t bar = bt_smem_u32(&s_bar[tile]);
    uint32_t parity = 0;
    const uint32_t dcol = (uint32_t)tile * DST;                       // the tile's accumulator columns
    const uint32_t tlane = tm + ((uint32_t)(32 * (warp & 3)) << 16);  // this warp's lane quadrant
    const uint32_t idesc_f = (2u << 4) | ((uint32_t)(NF >> 3) << 17) | ((uint32_t)(BT_M >> 4) << 24);
    const uint32_t idesc_c = (2u << 4) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(BT_M >> 4) << 24);
    const uint32_t utile = (uint32_t)__shfl_sync(0xffffffffu, tile, 0);  // (warp-uniform for the compiler)
    const uint32_t sbase = bt_smem_u32(smem_raw) + utile * 8 * 128;  // the tile's first column chunk
    const uint32_t udcol = utile * DST;
    auto issue = [&](int B, bool with_cum) {
        // generic-proxy plane writes (atomics) of all threads are ordered by the barrier; make them
        // visible to the tensor core's async-proxy reads
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t uB = (uint32_t)__shfl_sync(0xffffffffu, B, 0);
        const uint64_t df = bt_desc(sbase + (BT_FINEG + 2 * uB) * (uint32_t)GSZ, 128, GSZ);
        const uint64_t dc = bt_desc(sbase + (uint32_t)BT_CUMG * GSZ, 128, GSZ);
#pragma unroll 4
        for (int s = 0; s < NKA; ++s) {
            const uint32_t ta = tm + BT_ACOL0 + 8 * s;
            bt_mma(tm + udcol, ta, df + (uint64_t)(16 * s), idesc_f, s > 0);             // + 256 bytes per k-step
            if (with_cum) bt_mma(tm + udcol + NF, ta, dc + (uint64_t)(16 * s), idesc_c, s > 0);
        }
        bt_commit(bt_smem_u32(&s_bar[utile]));
    };

    const int xl = tile * BT_M + m;
    const bool valid = X0 + xl < W;
    uint8_t *dpx = dst + (int64_t)(y0 - p.row_begin) * p.dst_pitch + X0 + xl;
    const int rank = (int)p.rank;
    // value chunks of the pixels whose coarse bin lies in [B, B + NB): the chunk's 16 counts, then the descent
    auto resolve = [&](int B, int cb, int kf, bool want, int &val, bool &miss) {
        const int d = cb - B;
        const bool inwin = want && d >= 0 && d < NB;
#pragma unroll
        for (int dd = 0; dd < NB; ++dd) {
            if (__any_sync(0xffffffffu, inwin && d == dd)) {  // (the load's address is warp-uniform)
                int f[16];
                bt_ld16(tlane + dcol + 16 * dd, f);
                if (inwin && d == dd) {
                    val = 16 * cb + bt_descend16(f, kf);
                    miss = false;
                }
            }
        }
    };

    if (y0 + 1 < y1) prefetch(y0 + 1);
    for (int y = y0; y < y1; ++y, dpx += p.dst_pitch) {
        const int cur = (y - y0) & 1;  // statistics of this row; the row above left its own in cur ^ 1
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();  // the planes are those of row y; last row's accumulators have been read
        // the tile's window base from the coarse bins of the row above (every thread of the tile
        // computes the same): the bins the tile used, centred in the window
        int Bt = 0;
        if (y > y0) {
            const int lo = s_lo[cur ^ 1][tile], hi = s_hi[cur ^ 1][tile], nib = s_minv[cur ^ 1][tile] & 15;
            if (lo <= hi) {
                const int slack = NB - (hi - lo + 1);
                const int under = slack <= 0 ? 0 : slack / 2 + (((slack & 1) && nib < 8) ? 1 : 0);
                Bt = max(lo - under, 0);
            }
        }
        if (issue_warp) issue(Bt, true);
        bt_wait(bar, parity);
        parity ^= 1;
        // every pixel's coarse bin and the count below it from the 16 cumulative counts
        int c[16];
        bt_ld16(tlane + dcol + NF, c);
        const bool p8 = c[8] < rank;
        const int a4 = p8 ? c[12] : c[4];
        int cb = p8 ? 8 : 0, below = p8 ? c[8] : 0;
        const bool p4 = a4 < rank;
        cb += p4 ? 4 : 0;
        below = p4 ? a4 : below;
        const int a2 = p8 ? (p4 ? c[14] : c[10]) : (p4 ? c[6] : c[2]);
        const bool p2 = a2 < rank;
        cb += p2 ? 2 : 0;
        below = p2 ? a2 : below;
        const int q0 = p2 ? c[3] : c[1], q1 = p2 ? c[7] : c[5], q2 = p2 ? c[11] : c[9], q3 = p2 ? c[15] : c[13];
        const int a1 = p8 ? (p4 ? q3 : q2) : (p4 ? q1 : q0);
        const bool p1 = a1 < rank;
        cb += p1 ? 1 : 0;
        below = p1 ? a1 : below;
        const int kf = rank - below;  // rank within coarse bin cb
        bool miss = cb < Bt || cb >= Bt + NB;
        // every product of this row is done once all threads are here; any pixel outside its window?
        int anymiss = __syncthreads_or(miss && valid);
        if (issuer && y > y0) {  // the row above's statistics have been read by the whole tile
            s_lo[cur ^ 1][tile] = 255;
            s_hi[cur ^ 1][tile] = -1;
            s_minv[cur ^ 1][tile] = 255;
        }
        int val = 0;
        miss = true;
        resolve(Bt, cb, kf, true, val, miss);
        while (anymiss) {
            // the tile repeats the value product from its lowest missed coarse bin (the planes are
            // still those of this row: no thread has left the loop)
            if (miss && valid) atomicMin(&s_retry[tile], cb);
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncthreads();  // (also: every value chunk of the last product has been read)
            const int nb = s_retry[tile];
            if (nb != 255) {
                if (issue_warp) issue(nb, false);
                bt_wait(bar, parity);
                parity ^= 1;
                resolve(nb, cb, kf, miss, val, miss);
            }
            __syncthreads();
            if (issuer) s_retry[tile] = 255;
            anymiss = __syncthreads_or(miss && valid);
        }
        // coarse bins and lowest value of this row's pixels: the next row's base
        {
            const int wlo = __reduce_min_sync(0xffffffffu, valid ? cb : 255);
            const int whi = __reduce_max_sync(0xffffffffu, valid ? cb : -1);
            const int wmv = __reduce_min_sync(0xffffffffu, valid ? val : 255);
            if (lane == 0) {
                atomicMin(&s_lo[cur][tile], wlo);
                atomicMax(&s_hi[cur][tile], whi);
                atomicMin(&s_minv[cur][tile], wmv);
            }
        }
        if (valid) *dpx = lut ? __ldg(lut + val) : (uint8_t)val;
        // the planes move on to row y+1 (other warps may still be descending: they read tensor memory only)
        if (y + 1 < y1) {
            if (pwc >= 0) move(pwc, pone, pvo, pvi);
            if (nslots > NTH) {
                const uint8_t *ro = src_row(p, src, clampi(y - r, 0, H - 1));
                const uint8_t *ri = src_row(p, src, clampi(y + 1 + r, 0, H - 1));
                for (int s = tid + NTH; s < nslots; s += NTH) {
                    const int bl = s / nwords, wc = s - bl * nwords, cc = 4 * wc + bl;
                    if (cc >= NC) continue;
                    const int gx = clampi(X0 - r + cc, 0, W - 1);
                    move(wc, 1u << (8 * bl), __ldg(ro + gx), __ldg(ri + gx));
                }
            }
            if (y + 2 < y1) prefetch(y + 2);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
    if (STREAM) stream_signal(p, y0, y1, X0, X0 + TW);
}

}  // namespace mtb
