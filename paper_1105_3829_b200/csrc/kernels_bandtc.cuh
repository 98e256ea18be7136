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
// Bins of 15 values: bin j = values 15j .. 15j+14 owns 16 consecutive planes
// (two groups): the cumulative plane "pixels below 15j", then its 15 value
// planes -- so the planes of NB consecutive bins are ONE contiguous B operand
// and a row costs one product (N = 16 NB) per k-step and 128-pixel tile; its
// result holds, per bin, the count below the bin and the bin's 15 counts.  The
// window base is predicted from the bins the tile used one row up.  A pixel
// whose rank lies below or above the window is a miss: the tile repeats the
// product from a window on that side (its planes are still those of this row)
// until every pixel is resolved -- exact for any image.
//
// All arithmetic is exact integer counting (r <= 127: u8 column counts).
#pragma once
#include "common.cuh"

namespace mtb {

constexpr int BT_M = 128;          // pixels per product (tensor-memory lanes)
constexpr int BT_MAXTILES = 4;     // 128-pixel tiles per CTA (512 threads)
constexpr int BT_TMEM_COLS = 512;  // the whole tensor memory (one CTA per SM)
constexpr int BT_ACOL0 = 416;      // band tiles: columns 416 .. 416 + 8 NKA (NKA <= 12)
constexpr int BT_BINS = 18;         // bins of 15 values (18 x 15 >= 256), 16 planes = 2 groups each

__host__ __device__ constexpr int bt_nka(int r) { return (BT_M + 2 * r + 31) / 32; }
__host__ __device__ constexpr int bt_ncols(int TW, int r) { return TW - BT_M + 32 * bt_nka(r); }
__host__ __device__ constexpr int bt_groups(int) { return 2 * BT_BINS; }
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

// NF: planes of the keyed product (32: two bins of 15 values, 64: four).
// Block = 2 TW threads: thread t < TW = pixel t of the stripe (TW = 128 MT
// output columns); the others only help with the row updates.  Grid =
// (stripes, row slabs, images).
template <int NF, bool STREAM>
__global__ void __launch_bounds__(2 * BT_M * BT_MAXTILES, 1) k_bandtc_u8(SlabParams p, int TW) {
    static_assert(NF == 32 || NF == 64, "two or four bins per keyed window");
    constexpr int NB = NF / 16;  // bins of the keyed window
    constexpr int DST = NF;      // tensor-memory columns per tile
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
        s_minv[0][tid] = s_minv[1][tid] = 4096;
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
    // plane of value v: bin v / 15 (exact for v < 256), plane 1 + v % 15 of the bin's 16
    auto vplane = [](unsigned v) { const unsigned j = (v * 137u) >> 11; return (int)(v + j + 1u); };  // 16 j + 1 + (v - 15 j)
    auto vbin = [](unsigned v) { return (int)((v * 137u) >> 11); };
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
            for (int u = 0; u < 8; ++u) atomicAdd(planew + pword(vplane(v[u]), wc), one);
        }
        for (; j <= r; ++j)
            atomicAdd(planew + pword(vplane(__ldg(src_row(p, src, clampi(y0 + j, 0, H - 1)) + gx)), wc), one);
    }
    __syncthreads();
    // cumulative planes (plane 16 j: pixels below 15 j) from the value planes (bytewise; a
    // column's total is n <= 255)
    for (int wc = tid; wc < nwords; wc += NTH) {
        uint32_t run = 0;
        for (int j = 0; j < BT_BINS; ++j) {
            planew[pword(16 * j, wc)] = run;
#pragma unroll
            for (int v = 1; v < 16; ++v) run += planew[pword(16 * j + v, wc)];
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
        atomicAdd(planew + pword(vplane(vo), wc), 0u - one);
        atomicAdd(planew + pword(vplane(vi), wc), one);
        // plane 16 j counts the pixels below 15 j
        const int a = vbin(vo), b = vbin(vi);
        const uint32_t d = b > a ? 0u - one : one;
        for (int j = min(a, b) + 1; j <= max(a, b); ++j) atomicAdd(planew + pword(16 * j, wc), d);
    };

    // ---- products: the first warp of every tile issues (one elected lane); the tile's 128
    // threads read their pixels' counts
    const bool worker = tid < TW;                    // a pixel thread (the others only move the planes)
    const bool issuer = worker && m == 0;            // the tile's bookkeeping thread
    const bool issue_warp = worker && (warp & 3) == 0;
    const uint32_t utile = (uint32_t)__shfl_sync(0xffffffffu, tile, 0);  // (warp-uniform for the compiler)
    const uint32_t bar = bt_smem_u32(&s_bar[worker ? tile : 0]);
    uint32_t parity = 0;
    const uint32_t dcol = (uint32_t)tile * DST;                       // the tile's accumulator columns
    const uint32_t udcol = utile * DST;
    const uint32_t tlane = tm + ((uint32_t)(32 * (warp & 3)) << 16);  // this warp's lane quadrant
    const uint32_t idesc = (2u << 4) | ((uint32_t)(NF >> 3) << 17) | ((uint32_t)(BT_M >> 4) << 24);
    const uint32_t sbase = bt_smem_u32(smem_raw) + utile * 8 * 128;   // the tile's first column chunk
    auto issue = [&](int B) {
        // generic-proxy plane writes (atomics) of all threads are ordered by the barrier; make them
        // visible to the tensor core's async-proxy reads
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t uB = (uint32_t)__shfl_sync(0xffffffffu, B, 0);
        const uint64_t db = bt_desc(sbase + 2 * uB * (uint32_t)GSZ, 128, GSZ);
#pragma unroll 4
        for (int s = 0; s < NKA; ++s) bt_mma(tm + udcol, tm + BT_ACOL0 + 8 * s, db + (uint64_t)(16 * s), idesc, s > 0);  // + 256 bytes per k-step
        bt_commit(bt_smem_u32(&s_bar[utile]));
    };

    const int xl = tile * BT_M + m;
    const bool valid = worker && X0 + xl < W;
    uint8_t *dpx = dst + (int64_t)(y0 - p.row_begin) * p.dst_pitch + X0 + xl;
    const int rank = (int)p.rank;
    // After a product from base B: the pixel's bin if the window holds its rank value.  lob / hib
    // bound the bin from what the misses told (below the window / above it).
    auto resolve = [&](int B, bool want, int &val, int &bin, bool &miss, int &lob, int &hib) {
        int bl[NB];  // counts below each bin of the window
#pragma unroll
        for (int i = 0; i < NB; ++i)
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(bl[i]) : "r"(tlane + dcol + 16 * i) : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        int ci = 0;
#pragma unroll
        for (int i = 1; i < NB; ++i) ci += bl[i] < rank ? 1 : 0;
        const bool low = rank <= bl[0];  // the rank value lies below the window
        if (want && low) hib = min(hib, B - 1);
        const bool look = want && !low;
#pragma unroll
        for (int dd = 0; dd < NB; ++dd) {
            if (__any_sync(0xffffffffu, look && ci == dd)) {  // (the load's address is warp-uniform)
                int f[16];
                bt_ld16(tlane + dcol + 16 * dd, f);
                if (look && ci == dd) {
                    const int k = rank - f[0];
                    f[0] = 0;
                    int tot = 0;
#pragma unroll
                    for (int i = 1; i < 16; ++i) tot += f[i];
                    if (k <= tot) {
                        bin = B + dd;
                        val = 15 * bin + bt_descend16(f, k) - 1;
                        miss = false;
                    } else {
                        lob = max(lob, B + NB);  // above the window (only its last bin can say so)
                    }
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
        int val = 0, bin = 0, lob = 0, hib = BT_BINS - 1;
        bool miss = worker;
        int Bt = (BT_BINS - NB) / 2;
        if (worker) {
            // the tile's window base from the bins of the row above (every thread of the tile
            // computes the same): the bins the tile used, centred in the window
            if (y > y0) {
                const int lo = s_lo[cur ^ 1][tile], hi = s_hi[cur ^ 1][tile], pos = s_minv[cur ^ 1][tile];
                if (lo <= hi) {
                    const int slack = NB - (hi - lo + 1);
                    const int under = slack <= 0 ? 0 : slack / 2 + (((slack & 1) && pos - 15 * lo < 7) ? 1 : 0);
                    Bt = min(max(lo - under, 0), BT_BINS - NB);
                }
            }
            if (issue_warp) issue(Bt);
            bt_wait(bar, parity);
            parity ^= 1;
            resolve(Bt, true, val, bin, miss, lob, hib);
        }
        // every product of this row is done once all threads are here; any pixel outside its window?
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        int anymiss = __syncthreads_or(miss && valid);
        if (issuer && y > y0) {  // the row above's statistics have been read by the whole tile
            s_lo[cur ^ 1][tile] = 255;
            s_hi[cur ^ 1][tile] = -1;
            s_minv[cur ^ 1][tile] = 4096;
        }
        while (anymiss) {
            // the tile repeats the product from a window on the side its lowest missed pixel asked
            // for (the planes are still those of this row: no thread has left the loop)
            if (miss && valid) atomicMin(&s_retry[tile], hib < BT_BINS - 1 ? max(hib - NB + 1, 0) : min(lob, BT_BINS - NB));
            __syncthreads();
            if (worker) {
                const int nb = s_retry[tile];
                if (nb != 255) {
                    if (issue_warp) issue(nb);
                    bt_wait(bar, parity);
                    parity ^= 1;
                    resolve(nb, miss, val, bin, miss, lob, hib);
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncthreads();
            if (issuer) s_retry[tile] = 255;
            anymiss = __syncthreads_or(miss && valid);
        }
        if (worker) {
            // bins and lowest value of this row's pixels: the next row's base
            const int wlo = __reduce_min_sync(0xffffffffu, valid ? bin : 255);
            const int whi = __reduce_max_sync(0xffffffffu, valid ? bin : -1);
            const int wmv = __reduce_min_sync(0xffffffffu, valid ? val : 4096);
            if (lane == 0) {
                atomicMin(&s_lo[cur][tile], wlo);
                atomicMax(&s_hi[cur][tile], whi);
                atomicMin(&s_minv[cur][tile], wmv);
            }
            if (valid) *dpx = lut ? __ldg(lut + val) : (uint8_t)val;
        }
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
