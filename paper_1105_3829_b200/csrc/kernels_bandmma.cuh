// kernels_bandmma.cuh -- 8-bit rank filter: per-column histograms in shared
// memory as byte planes, window histograms as band-matrix products on the
// tensor cores (mma.sync m16n8k32, u8 x u8 -> s32).
//
// The reference keeps one histogram tree per image column and merges the
// window's columns (_kernels.py:115-194 sync_node, :229-253 extract_u).  Here
// the CTA keeps, for every column c of its halo'd stripe [X0-r, X0+TW+r), the
// 256-bin histogram of the column's vertical span (rows y-r .. y+r) as 256
// byte PLANES fine[v][c] (u8 counts: a column holds n <= 255 pixels), plus 16
// cumulative coarse planes cum[j][c] = number of the column's pixels below
// 16 j.  Moving down one row is one -1 and one +1 on the fine planes and
// +-1 on the cumulative planes between the two coarse bins.
//
// The window count of output pixel x for any plane P is
//     sum_c Band[x][c] * P[c],      Band[x][c] = 1 iff x <= c <= x + 2r
// -- a product of a 0/1 band matrix with the plane bytes.  One warp computes
// it for 16 adjacent pixels x 8 planes per mma.sync, walking the 16+2r
// columns the 16 windows touch in k-tiles of 32 columns (NK = ceil((16+2r)/32)).
// The band fragments are per-lane constants (all ones for interior k-tiles);
// the plane bytes are the B fragments, one 8-byte shared-memory load per lane
// and k-tile.  No O(n) gathers per pixel on the CUDA cores, no prefix scans,
// no sliding windows: the gather is the tensor core's k-loop.
//
// Keyed windows.  A warp resolves 32 output pixels (two groups of 16, 32
// columns apart so that they share k-tiles) with ONE product over 8*NT planes:
// the cumulative plane cum[B] ("below 16 B") and the 8*NT-1 value planes
// 16B .. 16B+8NT-2.  B is predicted from the same pixels' results one row up
// (the median of a large window moves slowly: on the benchmark frame the
// prediction misses 0.05% of the time at r = 63 with NT = 4 and 0.5% at
// r = 31 with NT = 6).  A pixel whose rank falls outside the keyed window
// is a miss: the warp then takes the coarse bin of every unresolved pixel from
// the 16 cumulative planes (one product) and repeats the keyed product from
// the lowest one, until every pixel is resolved -- exact for any image, the
// prediction only decides the speed.  The accumulator fragments are
// transposed through a per-warp buffer so that each lane descends one pixel's
// packed u16 counts (the reference's extract_u, 16-ary).
//
// All arithmetic is exact integer counting; window counts fit u16 because
// n^2 <= 65535 is required (r <= 127).
#pragma once
#include "common.cuh"

namespace mtb {

constexpr int BM_PLANES = 272;  // 16 cumulative coarse planes, then one plane per value
constexpr int BM_MAXT = 512;    // threads per CTA (128 registers per thread)
constexpr int BM_TPITCH = 34;   // 16-byte units between the rows of a transpose buffer

// stripe geometry for a radius: TW output columns (multiple of 64), NP plane
// pitch in bytes (>= halo'd columns and the last k-tile a warp reads; NP mod
// 64 == 32 keeps the four plane rows of a half-warp's B-fragment load in
// distinct bank groups)
__host__ __device__ constexpr int bm_nk(int r) { return (16 + 2 * r + 31) / 32; }
__host__ __device__ constexpr int bm_pitch(int TW, int r) {
    const int a = TW + 2 * r, b = TW + 32 * bm_nk(r) - 16;
    const int need = a > b ? a : b;
    return ((need + 31) / 64) * 64 + 32;  // smallest value >= need with value mod 64 == 32
}
__host__ __device__ constexpr int bm_tbuf_bytes(int NT) { return NT * BM_TPITCH * 16; }
__host__ __device__ constexpr size_t bm_smem(int TW, int r, int warps, int NT) {
    // planes | per-warp transpose buffers
    return (size_t)BM_PLANES * bm_pitch(TW, r) + (size_t)warps * bm_tbuf_bytes(NT);
}

__device__ __forceinline__ void bm_mma(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// 0/1 bytes of window [m, m+2r] over the four columns col0 .. col0+3
__device__ __forceinline__ uint32_t bm_mask4(int col0, int m, int r2) {
    uint32_t v = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) v |= ((col0 + i >= m && col0 + i <= m + r2) ? 1u : 0u) << (8 * i);
    return v;
}

__device__ __forceinline__ uint32_t bm_hsum16(uint32_t w) { return (w * 0x10001u) >> 16; }

// smallest bin b with cumsum(bins[0..b]) >= k (16 u16 bins packed in w[0..7],
// bins 2i | 2i+1 << 16; the caller guarantees sum >= k); leaves in k the rank
// within bin b
__device__ __forceinline__ int bm_descend(const uint32_t (&w)[8], uint32_t &k) {
    uint32_t s = bm_hsum16(w[0] + w[1] + w[2] + w[3]);
    const bool r1 = s < k;
    k -= r1 ? s : 0u;
    const uint32_t a0 = r1 ? w[4] : w[0], a1 = r1 ? w[5] : w[1];
    const uint32_t a2 = r1 ? w[6] : w[2], a3 = r1 ? w[7] : w[3];
    s = bm_hsum16(a0 + a1);
    const bool r2 = s < k;
    k -= r2 ? s : 0u;
    const uint32_t b0 = r2 ? a2 : a0, b1 = r2 ? a3 : a1;
    s = bm_hsum16(b0);
    const bool r3 = s < k;
    k -= r3 ? s : 0u;
    const uint32_t c = r3 ? b1 : b0;
    s = c & 0xffffu;
    const bool r4 = s < k;
    k -= r4 ? s : 0u;
    return (r1 ? 8 : 0) | (r2 ? 4 : 0) | (r3 ? 2 : 0) | (r4 ? 1 : 0);
}

// One product: 8*NTL planes for the two groups of 16 pixels whose windows
// start at stripe columns xa and xa + 32.  Plane of bin i: row(i).  Results
// transposed through tb: lane l gets pixel (l >> 4) * 32 + (l & 15) of the
// pair as 8*NTL u16 counts packed in w[0 .. 4*NTL) (bins 2i | 2i+1 << 16).
template <int NK, int NTL, typename RowOf>
__device__ __forceinline__ void bm_product(const uint8_t *planes, int NP, int xa, int lane,
                                           const uint32_t (&af)[3][4], unsigned char *tb, RowOf row,
                                           uint32_t (&w)[4 * NTL], int dbg = 0) {
    const int g = lane >> 2, q = lane & 3;
    int acc[2][NTL][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int t = 0; t < NTL; ++t)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[a][t][i] = 0;
    const uint32_t ones[4] = {0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u};
#pragma unroll
    for (int t = 0; t < NTL; ++t) {
        // n-tile t holds bins 8t .. 8t+7, this lane's B-fragment column is bin
        // 8t + g: the four plane rows a half-warp reads are consecutive, so with
        // the pitch = 32 (mod 64) they sit in distinct bank groups
        const uint8_t *rp = planes + (size_t)row(8 * t + g) * NP + xa + 8 * q;
#pragma unroll
        for (int j = 0; j <= NK; ++j) {
            const uint2 b = *reinterpret_cast<const uint2 *>(rp + 32 * j);
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                const int kt = j - a;  // group a's k-tile held by this load
                if (kt < 0 || kt >= NK) continue;
                if (kt == 0)
                    bm_mma(acc[a][t], af[0], b.x, b.y);
                else if (kt == NK - 1)
                    bm_mma(acc[a][t], af[2], b.x, b.y);
                else if (kt == NK - 2)
                    bm_mma(acc[a][t], af[1], b.x, b.y);
                else
                    bm_mma(acc[a][t], ones, b.x, b.y);
            }
        }
    }
    // lane (g, q) holds, per n-tile t, bins 8t+2q and 8t+2q+1 of pixels g (regs
    // 0, 1) and g + 8 (regs 2, 3) of each group.  It writes its NTL packed words
    // as 8-byte half-units q NTL/2 .. of the pixel's record (record word
    // q NTL + t = bins 8t+2q | 8t+2q+1); half-unit h of pixel p lives at
    // ((h >> 1) * PITCH + p) * 16 + (h & 1) * 8
    __syncwarp();
#pragma unroll
    for (int a = 0; a < 2; ++a) {
#pragma unroll
        for (int hh = 0; hh < NTL / 2; ++hh) {
            const int h = q * (NTL / 2) + hh;
            unsigned char *dst = tb + ((h >> 1) * BM_TPITCH) * 16 + (h & 1) * 8;
            const uint2 lo = make_uint2(__byte_perm(acc[a][2 * hh][0], acc[a][2 * hh][1], 0x5410),
                                        __byte_perm(acc[a][2 * hh + 1][0], acc[a][2 * hh + 1][1], 0x5410));
            const uint2 hi = make_uint2(__byte_perm(acc[a][2 * hh][2], acc[a][2 * hh][3], 0x5410),
                                        __byte_perm(acc[a][2 * hh + 1][2], acc[a][2 * hh + 1][3], 0x5410));
            *reinterpret_cast<uint2 *>(dst + (16 * a + g) * 16) = lo;
            *reinterpret_cast<uint2 *>(dst + (16 * a + g + 8) * 16) = hi;
        }
    }
    __syncwarp();
    // record word qq NTL + t -> w[4t + qq] (bins 2i | 2i+1 << 16 in w[i])
    uint32_t rec[4 * NTL];
#pragma unroll
    for (int u = 0; u < NTL; ++u) {
        const uint4 v = *reinterpret_cast<const uint4 *>(tb + (u * BM_TPITCH + lane) * 16);
        rec[4 * u] = v.x; rec[4 * u + 1] = v.y; rec[4 * u + 2] = v.z; rec[4 * u + 3] = v.w;
    }
#pragma unroll
    for (int t = 0; t < NTL; ++t)
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) w[4 * t + qq] = rec[qq * NTL + t];
}

// NK: k-tiles per group of 16 pixels; NT: n-tiles of the keyed window (8 NT
// planes: cum[B] and 8 NT - 1 values).  Block = 32 * warps threads; grid =
// (stripes, row slabs, images).
template <int NK, int NT, bool STREAM>
__global__ void __launch_bounds__(BM_MAXT, 1) k_bandmma_u8(SlabParams p, int TW) {
    static_assert(NT == 4 || NT == 6, "keyed window of 32 or 48 planes");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NTH = blockDim.x;
    const int r = p.radius, r2 = 2 * r, H = p.H, W = p.W;
    const int NC = TW + r2, NP = bm_pitch(TW, r), NPW = NP >> 2;
    uint8_t *planes = smem_raw;
    uint32_t *planew = reinterpret_cast<uint32_t *>(smem_raw);
    unsigned char *tb = smem_raw + (size_t)BM_PLANES * NP + (size_t)warp * bm_tbuf_bytes(NT);
    const int X0 = blockIdx.x * TW;
    const int y0 = p.row_begin + blockIdx.y * p.rows_per_cta;
    if (y0 >= p.row_end) return;  // CTA-uniform (barriers below)
    const int y1 = min(y0 + p.rows_per_cta, p.row_end);
    if (STREAM) stream_wait_rows(p, y1 + r);
    const uint8_t *src = static_cast<const uint8_t *>(p.src) + blockIdx.z * p.src_img_stride;
    uint8_t *dst = static_cast<uint8_t *>(p.dst) + blockIdx.z * p.dst_img_stride;
    const uint8_t *lut = static_cast<const uint8_t *>(p.lut);

    // ---- column histograms of row y0: rows clamp(y0-r .. y0+r).  Slot s =
    // (byte lane, word): the lanes of a warp hit distinct words, so their
    // shared-memory atomics never collide inside the warp.
    for (int i = tid; i < BM_PLANES * NPW; i += NTH) planew[i] = 0;
    __syncthreads();
    const int nwords = (NC + 3) >> 2, nslots = 4 * nwords;
    for (int s = tid; s < nslots; s += NTH) {
        const int bl = s / nwords, wd = s - bl * nwords, c = 4 * wd + bl;
        if (c >= NC) continue;
        const int gx = clampi(X0 - r + c, 0, W - 1);
        const uint32_t one = 1u << (8 * bl);
        int j = -r;
        for (; j + 7 <= r; j += 8) {  // 8 loads in flight (the rows come from L2)
            unsigned v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(src_row(p, src, clampi(y0 + j + u, 0, H - 1)) + gx);
#pragma unroll
            for (int u = 0; u < 8; ++u) atomicAdd(planew + (16 + v[u]) * NPW + wd, one);
        }
        for (; j <= r; ++j)
            atomicAdd(planew + (16 + __ldg(src_row(p, src, clampi(y0 + j, 0, H - 1)) + gx)) * NPW + wd, one);
    }
    __syncthreads();
    // cumulative planes from the value planes: cum[j] = sum of planes below 16 j
    // (bytewise; a column's total is n <= 255, so no byte carries)
    for (int wd = tid; wd < nwords; wd += NTH) {
        uint32_t run = 0;
        for (int j = 0; j < 16; ++j) {
            planew[j * NPW + wd] = run;
#pragma unroll
            for (int v = 0; v < 16; ++v) run += planew[(16 + 16 * j + v) * NPW + wd];
        }
    }

    // ---- per-lane constants of the output phase
    const int g = lane >> 2, q = lane & 3;
    // band fragments of k-tiles 0, NK-2, NK-1 (the others are all ones):
    // [0]: pixel g, columns 8q..8q+3 of the tile; [1]: pixel g+8, same columns;
    // [2]: pixel g, columns 8q+4..8q+7; [3]: pixel g+8
    uint32_t af[3][4];
#pragma unroll
    for (int s = 0; s < 3; ++s) {
        const int kt = s == 0 ? 0 : (s == 1 ? NK - 2 : NK - 1);
        const int c0 = 32 * kt + 8 * q;
        af[s][0] = bm_mask4(c0, g, r2);
        af[s][1] = bm_mask4(c0, g + 8, r2);
        af[s][2] = bm_mask4(c0 + 4, g, r2);
        af[s][3] = bm_mask4(c0 + 4, g + 8, r2);
    }

    // ---- row updates: slot s = tid + u NTH, leaving / entering pixels a row
    // ahead; running row pointers (a clamped row index repeats the edge row)
    constexpr int PF = 2;
    uint32_t *pw[PF];       // plane word of the slot (row 0), nullptr: no slot
    uint32_t pone[PF];
    const uint8_t *pin[PF];  // the slot's column in source row 0 of this image
#pragma unroll
    for (int u = 0; u < PF; ++u) {
        const int s = tid + u * NTH;
        const int bl = s / nwords, wd = s - bl * nwords, c = 4 * wd + bl;
        pw[u] = (s < nslots && c < NC) ? planew + wd : nullptr;
        pin[u] = src_row(p, src, p.src_row0) + clampi(X0 - r + min(c, NC - 1), 0, W - 1);
        pone[u] = 1u << (8 * (bl & 3));
    }
    unsigned pvo[PF], pvi[PF];
    auto prefetch = [&](int yn) {
        const int64_t oo = (int64_t)(clampi(yn - r - 1, 0, H - 1) - p.src_row0) * p.src_pitch;
        const int64_t oi = (int64_t)(clampi(yn + r, 0, H - 1) - p.src_row0) * p.src_pitch;
#pragma unroll
        for (int u = 0; u < PF; ++u) {
            if (pw[u]) {
                pvo[u] = __ldg(pin[u] + oo);
                pvi[u] = __ldg(pin[u] + oi);
            }
        }
    };
    auto move = [&](uint32_t *wp, uint32_t one, unsigned vo, unsigned vi) {
        atomicAdd(wp + (16 + vo) * NPW, 0u - one);
        atomicAdd(wp + (16 + vi) * NPW, one);
        // cum[j] counts the pixels below 16 j: removing vo takes 1 from every
        // j > vo >> 4, adding vi gives 1 to every j > vi >> 4
        const int a = (int)(vo >> 4), b = (int)(vi >> 4);
        const uint32_t d = b > a ? 0u - one : one;
        for (int j = min(a, b) + 1; j <= max(a, b); ++j) atomicAdd(wp + j * NPW, d);
    };

    // ---- the warp's 32 output pixels (one pair of groups per warp: the
    // launcher starts TW / 32 warps)
    const int xa = 64 * (warp >> 1) + 16 * (warp & 1);    // first pixel of group 0; group 1 at xa + 32
    const int xl = xa + 32 * (lane >> 4) + (lane & 15);   // this lane's pixel (stripe-relative)
    const bool valid = X0 + xl < W;
    const bool live = X0 + xa < W;                         // (warp-uniform) something of the pair is in the image
    uint8_t *dpx = dst + (int64_t)(y0 - p.row_begin) * p.dst_pitch + X0 + xl;
    int Bp = 0xff;  // predicted window base (coarse bin); 0xff: none yet
    const uint32_t rank = p.rank;
    const int dbg = p.gate;

    for (int y = y0; y < y1; ++y, dpx += p.dst_pitch) {
        if (y > y0 && !(dbg & 2)) {
#pragma unroll
            for (int u = 0; u < PF; ++u)
                if (pw[u]) move(pw[u], pone[u], pvo[u], pvi[u]);
            if (nslots > PF * NTH) {
                const uint8_t *ro = src_row(p, src, clampi(y - r - 1, 0, H - 1));
                const uint8_t *ri = src_row(p, src, clampi(y + r, 0, H - 1));
                for (int s = tid + PF * NTH; s < nslots; s += NTH) {
                    const int bl = s / nwords, wd = s - bl * nwords, c = 4 * wd + bl;
                    if (c >= NC) continue;
                    const int gx = clampi(X0 - r + c, 0, W - 1);
                    move(planew + wd, 1u << (8 * bl), __ldg(ro + gx), __ldg(ri + gx));
                }
            }
        }
        if (y + 1 < y1) prefetch(y + 1);
        __syncthreads();
        if (live && !(dbg & 4)) {
            int B = Bp;
            uint32_t open = 0xffffffffu;  // lanes not yet resolved
            unsigned val = 0;
            for (int pass = 0;; ++pass) {
                if (pass > 0 || B == 0xff) {
                    // coarse bin of every open pixel from the 16 cumulative planes
                    uint32_t cw[8];
                    bm_product<NK, 2>(planes, NP, xa, lane, af, tb, [](int bin) { return bin; }, cw);
                    int cb = 0;  // number of j in 1..15 with cum[j] < rank = the coarse bin
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        cb += (i > 0 && (cw[i] & 0xffffu) < rank) ? 1 : 0;
                        cb += ((cw[i] >> 16) < rank) ? 1 : 0;
                    }
                    // lanes past the image edge and resolved lanes do not vote
                    B = __reduce_min_sync(0xffffffffu, (((open >> lane) & 1u) && valid) ? cb : 255);
                    if (B == 255) break;  // only lanes past the edge were open
                }
                uint32_t w[4 * NT];
                bm_product<NK, NT>(planes, NP, xa, lane, af, tb,
                                   [B](int bin) {
                                       const int v = 16 * B + bin - 1;  // value plane; bin 0: cum[B]
                                       return bin == 0 ? B : (v <= 255 ? 16 + v : 0);  // past 255: the zero plane
                                   },
                                   w, dbg);
                // chunk of 16 bins holding the rank, then the 16-ary descent;
                // a rank above the window's total ends in the last bin with
                // more left than the bin holds
                uint32_t k = rank;
                uint32_t c8[8];
                int base;
                const uint32_t s0 = bm_hsum16(w[0] + w[1] + w[2] + w[3] + w[4] + w[5] + w[6] + w[7]);
                const bool p1 = s0 < k;
                if constexpr (NT == 4) {
                    k -= p1 ? s0 : 0u;
                    base = p1 ? 16 : 0;
#pragma unroll
                    for (int i = 0; i < 8; ++i) c8[i] = p1 ? w[8 + i] : w[i];
                } else {
                    const uint32_t s1 = bm_hsum16(w[8] + w[9] + w[10] + w[11] + w[12] + w[13] + w[14] + w[15]);
                    const bool p2 = s0 + s1 < k;
                    k -= p2 ? s0 + s1 : (p1 ? s0 : 0u);
                    base = p2 ? 32 : (p1 ? 16 : 0);
#pragma unroll
                    for (int i = 0; i < 8; ++i) c8[i] = p2 ? w[(16 + i) % (4 * NT)] : (p1 ? w[8 + i] : w[i]);
                }
                int b16 = 1;
                if (!(dbg & 8)) b16 = bm_descend(c8, k); else k = 0;
                const uint32_t cl = c8[7] >> 16;  // count of a chunk's last bin
                const int bin = base + b16;
                // bin 0 is "below the window": a miss, like a rank above the window's total
                const bool hit = bin > 0 && !(b16 == 15 && k > cl);
                if (hit && ((open >> lane) & 1u)) val = (unsigned)(16 * B + bin - 1);
                open &= ~__ballot_sync(0xffffffffu, hit || !valid);
                if (!open) break;
            }
            // prediction for the next row: the lowest result of the pair, one below for drift
            const int lo = __reduce_min_sync(0xffffffffu, valid ? (int)val : 255);
            Bp = max(lo - 1, 0) >> 4;
            if (valid) *dpx = lut ? __ldg(lut + val) : (uint8_t)val;
        }
        __syncthreads();
    }
    if (STREAM) stream_signal(p, y0, y1, X0, X0 + TW);
}

}  // namespace mtb
