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
// Keyed windows.  A warp resolves 16 adjacent output pixels with ONE product
// over 32 planes: the cumulative plane cum[B] ("below 16 B") and the 31 value
// planes 16B .. 16B+30.  B is predicted from the same pixels' results one row
// up (the median of a large window moves slowly: on the benchmark frame the
// prediction misses 0.3% of the time at r = 31 and never at r = 63).  A pixel
// whose rank falls outside the keyed window is a miss: the warp then takes
// the coarse bin of every unresolved pixel from the 16 cumulative planes (one
// product) and repeats the keyed product from the lowest one, until every
// pixel is resolved -- exact for any image, the prediction only decides the
// speed.  The accumulator fragments are transposed through a per-warp buffer
// so that a pair of lanes descends one pixel's 32 packed u16 counts, 16 bins
// each (the reference's extract_u, 16-ary).
//
// All arithmetic is exact integer counting; window counts fit u16 because
// n^2 <= 65535 is required (r <= 127).
#pragma once
#include <cstdio>
#include <type_traits>
#include "common.cuh"

namespace mtb {

constexpr int BM_PLANES = 272;  // 16 cumulative coarse planes, then one plane per value
constexpr int BM_MAXT = 1024;   // threads per CTA: one warp per 16 output columns
constexpr int BM_REC = 80;      // bytes between pixel records of a transpose buffer (64 used)
constexpr int BM_TBUF = 16 * BM_REC;

// stripe geometry for a radius: TW output columns (multiple of 16), NP plane
// pitch in bytes (>= halo'd columns and the last k-tile a warp reads; NP mod
// 64 == 32 keeps the four plane rows of a half-warp's B-fragment load in
// distinct bank groups)
__host__ __device__ constexpr int bm_nk(int r) { return (16 + 2 * r + 31) / 32; }
__host__ __device__ constexpr int bm_pitch(int TW, int r) {
    const int a = TW + 2 * r, b = TW + 32 * bm_nk(r) - 16;
    const int need = a > b ? a : b;
    return ((need + 31) / 64) * 64 + 32;  // smallest value >= need with value mod 64 == 32
}
__host__ __device__ constexpr size_t bm_smem(int TW, int r) {
    // planes | per-warp transpose buffers
    return (size_t)BM_PLANES * bm_pitch(TW, r) + (size_t)(TW / 16) * BM_TBUF;
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
// bins 2i | 2i+1 << 16); leaves in k the rank within bin b.  If the 16 bins
// hold fewer than k, the result is bin 15 with k above that bin's count.
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

// One product: 8*NTL planes (plane of bin i: row(i)) for the 16 pixels whose
// windows start at stripe columns xa .. xa+15.  n-tile t holds bins 8t..8t+7
// and lane (g, q)'s B-fragment column is bin 8t+g: the four plane rows a
// half-warp reads are consecutive, so with the pitch = 32 (mod 64) they sit
// in distinct bank groups.  After the k-loop lane (g, q) holds bins 8t+2q and
// 8t+2q+1 of pixels g and g+8: record word 4t+q (bins 2i | 2i+1 << 16 in word
// i) of the two pixels' records in tb.
template <int NK, int NTL, typename RowOf>
__device__ __forceinline__ void bm_product(const uint8_t *planes, int NP, int xa, int lane,
                                           const uint32_t (&af)[3][4], unsigned char *tb, RowOf row) {
    const int g = lane >> 2, q = lane & 3;
    const uint32_t ones[4] = {0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u};
    __syncwarp();  // the previous product's records have been read
#pragma unroll
    for (int t = 0; t < NTL; ++t) {
        const uint8_t *rp = planes + (size_t)row(8 * t + g) * NP + xa + 8 * q;
        int acc[4] = {0, 0, 0, 0};
#pragma unroll
        for (int kt = 0; kt < NK; ++kt) {
            const uint2 b = *reinterpret_cast<const uint2 *>(rp + 32 * kt);
            if (kt == 0)
                bm_mma(acc, af[0], b.x, b.y);
            else if (kt == NK - 1)
                bm_mma(acc, af[2], b.x, b.y);
            else if (kt == NK - 2)
                bm_mma(acc, af[1], b.x, b.y);
            else
                bm_mma(acc, ones, b.x, b.y);
        }
        *reinterpret_cast<uint32_t *>(tb + g * BM_REC + (4 * t + q) * 4) = __byte_perm(acc[0], acc[1], 0x5410);
        *reinterpret_cast<uint32_t *>(tb + (g + 8) * BM_REC + (4 * t + q) * 4) = __byte_perm(acc[2], acc[3], 0x5410);
    }
    __syncwarp();
}

// NK: k-tiles of a group of 16 pixels.  Block = 32 * (TW / 16) threads (one
// warp per 16 output columns); grid = (stripes, row slabs, images).
// PX = uint16_t: the same kernel on the coarse keys min(v >> s, 255) of 16-bit
// pixels (key_shift), as the first pass of the 16-bit candidate-bucket path
// from r = 32 (kernels_lowsel16.cuh): instead of a result pixel it writes
// H << 16 | k' per pixel to a u32 plane (p.dst, pitch in words), H = the
// result's key, k' = the rank of the result among the window values with that
// key (what the last descent leaves).
template <int NK, bool STREAM, typename PX = uint8_t>
__global__ void __launch_bounds__(BM_MAXT, 1) k_bandmma_u8(SlabParams p, int TW) {
    constexpr bool HI16 = sizeof(PX) == 2;
    using OUT = typename std::conditional<HI16, uint32_t, uint8_t>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (HI16 && gate_off(p)) return;  // (uniform over the grid)
    const int ks = HI16 ? key_shift(p) : 0;
    auto keyof = [&](unsigned v) -> unsigned { return HI16 ? min(v >> ks, 255u) : v; };
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NTH = blockDim.x;
    const int r = p.radius, r2 = 2 * r, H = p.H, W = p.W;
    const int NC = TW + r2, NP = bm_pitch(TW, r), NPW = NP >> 2;
    uint8_t *planes = smem_raw;
    uint32_t *planew = reinterpret_cast<uint32_t *>(smem_raw);
    unsigned char *tb = smem_raw + (size_t)BM_PLANES * NP + (size_t)warp * BM_TBUF;
#ifdef BM_TIMING
    const long long tstart = clock64();
#endif
    const int X0 = blockIdx.x * TW;
    const int y0 = p.row_begin + blockIdx.y * p.rows_per_cta;
    if (y0 >= p.row_end) return;  // CTA-uniform (barriers below)
    const int y1 = min(y0 + p.rows_per_cta, p.row_end);
    if (STREAM) stream_wait_rows(p, y1 + r);
    const PX *src = static_cast<const PX *>(p.src) + blockIdx.z * p.src_img_stride;
    OUT *dst = static_cast<OUT *>(p.dst) + blockIdx.z * p.dst_img_stride;
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
            for (int u = 0; u < 8; ++u) v[u] = keyof(__ldg(src_row(p, src, clampi(y0 + j + u, 0, H - 1)) + gx));
#pragma unroll
            for (int u = 0; u < 8; ++u) atomicAdd(planew + (16 + v[u]) * NPW + wd, one);
        }
        for (; j <= r; ++j)
            atomicAdd(planew + (16 + keyof(__ldg(src_row(p, src, clampi(y0 + j, 0, H - 1)) + gx))) * NPW + wd, one);
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

    // ---- row updates: one slot per thread (more: a loop), leaving / entering
    // pixels loaded a row ahead
    uint32_t *pw = nullptr;  // plane word of the slot (row 0), nullptr: no slot
    uint32_t pone = 0;
    const PX *pin = src;  // the slot's column in source row 0 of this image
    {
        const int bl = tid / nwords, wd = tid - bl * nwords, c = 4 * wd + bl;
        if (tid < nslots && c < NC) pw = planew + wd;
        pin = src_row(p, src, p.src_row0) + clampi(X0 - r + min(c, NC - 1), 0, W - 1);
        pone = 1u << (8 * (bl & 3));
    }
    unsigned pvo = 0, pvi = 0;
    // running pointers to the slot's column in the leaving / entering row of
    // the next update (a clamped row index repeats the edge row: no step)
    const PX *pout = pin + (int64_t)(clampi(y0 - r, 0, H - 1) - p.src_row0) * p.src_pitch;
    const PX *pent = pin + (int64_t)(clampi(y0 + 1 + r, 0, H - 1) - p.src_row0) * p.src_pitch;
    // rows of the update y-1 -> y: leaving y-r-1, entering y+r; called for yn = y0+1, y0+2, ...
    auto prefetch = [&](int yn) {
        if (pw) {
            pvo = keyof(__ldg(pout));
            pvi = keyof(__ldg(pent));
        }
        // next update (yn + 1): leaving row yn - r, entering row yn + 1 + r
        if (yn - r > 0 && yn - r <= H - 1) pout += p.src_pitch;
        if (yn + 1 + r <= H - 1) pent += p.src_pitch;
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

    // ---- the warp's 16 output pixels; lanes l and l + 16 share pixel l & 15:
    // each descends one half (16 bins) of the pixel's record
    const int xa = 16 * warp;                 // first pixel (stripe-relative) = first window column
    const int px = lane & 15, half = lane >> 4;
    const bool valid = X0 + xa + px < W;
    const bool live = X0 + xa < W;            // (warp-uniform) some pixel of the warp is in the image
    const unsigned char *myrec = tb + px * BM_REC + half * 32;
    OUT *dpx = dst + (int64_t)(y0 - p.row_begin) * p.dst_pitch + X0 + xa + px;
    int Bp = 0xff;  // predicted window base (coarse bin); 0xff: none yet
    const uint32_t rank = p.rank;

#ifdef BM_TIMING
    long long tA = 0, tB1 = 0, tB = 0, tB2 = 0, t0 = clock64(), tinit = t0 - tstart;
#endif
    for (int y = y0; y < y1; ++y, dpx += p.dst_pitch) {
        if (y > y0) {
            if (pw) move(pw, pone, pvo, pvi);
            if (nslots > NTH) {
                const PX *ro = src_row(p, src, clampi(y - r - 1, 0, H - 1));
                const PX *ri = src_row(p, src, clampi(y + r, 0, H - 1));
                for (int s = tid + NTH; s < nslots; s += NTH) {
                    const int bl = s / nwords, wd = s - bl * nwords, c = 4 * wd + bl;
                    if (c >= NC) continue;
                    const int gx = clampi(X0 - r + c, 0, W - 1);
                    move(planew + wd, 1u << (8 * bl), keyof(__ldg(ro + gx)), keyof(__ldg(ri + gx)));
                }
            }
        }
        if (y + 1 < y1) prefetch(y + 1);
#ifdef BM_TIMING
        { const long long t = clock64(); tA += t - t0; t0 = t; }
#endif
        __syncthreads();
#ifdef BM_TIMING
        { const long long t = clock64(); tB1 += t - t0; t0 = t; }
#endif
        if (live) {
            int B = Bp;
            uint32_t open = 0xffffffffu;  // lanes whose pixel is not yet resolved
            unsigned val = 0;
            for (int pass = 0;; ++pass) {
                if (pass > 0 || B == 0xff) {
                    // coarse bin of every open pixel from the 16 cumulative planes
                    bm_product<NK, 2>(planes, NP, xa, lane, af, tb, [](int bin) { return bin; });
                    const uint4 u = *reinterpret_cast<const uint4 *>(tb + px * BM_REC);
                    const uint4 v = *reinterpret_cast<const uint4 *>(tb + px * BM_REC + 16);
                    const uint32_t cw[8] = {u.x, u.y, u.z, u.w, v.x, v.y, v.z, v.w};
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
                bm_product<NK, 4>(planes, NP, xa, lane, af, tb, [B](int bin) {
                    const int v = 16 * B + bin - 1;  // value plane; bin 0: cum[B]
                    return bin == 0 ? B : (v <= 255 ? 16 + v : 0);  // past 255: the zero plane
                });
                // this lane's 16 bins: 0..15 (half 0, bin 0 = below the window) or 16..31
                const uint4 u = *reinterpret_cast<const uint4 *>(myrec);
                const uint4 v = *reinterpret_cast<const uint4 *>(myrec + 16);
                const uint32_t c8[8] = {u.x, u.y, u.z, u.w, v.x, v.y, v.z, v.w};
                const uint32_t mine = bm_hsum16(c8[0] + c8[1] + c8[2] + c8[3] + c8[4] + c8[5] + c8[6] + c8[7]);
                const uint32_t other = __shfl_xor_sync(0xffffffffu, mine, 16);
                // rank within this half; the upper half only counts when the lower holds fewer than rank
                uint32_t k = half ? rank - min(other, rank) : rank;
                const bool here = half ? (other < rank && k <= mine) : (rank <= mine);
                const int b16 = bm_descend(c8, k);
                const int bin = 16 * half + b16;
                // (bin 0 is "below the window": a miss, like a rank above the window's total)
                // (16-bit keys: the rank within the value rides along below the value)
                const unsigned found = (unsigned)(16 * B + bin - 1);
                const unsigned cand = (here && bin > 0) ? (HI16 ? (found << 16) | k : found) : 0xffffffffu;
                const unsigned both = min(cand, __shfl_xor_sync(0xffffffffu, cand, 16));  // the pair's result
                const bool hit = both != 0xffffffffu;
                if (hit && ((open >> lane) & 1u)) val = both;
                open &= ~__ballot_sync(0xffffffffu, hit || !valid);
                if (!open) break;
            }
            // prediction for the next row: the lowest result of the warp, one below for drift
            const int lo = __reduce_min_sync(0xffffffffu, valid ? (int)(HI16 ? val >> 16 : val) : 255);
            Bp = min(max(lo - 1, 0) >> 4, 15);
            if (valid && half == 0) {
                if (HI16)
                    *dpx = (OUT)val;
                else
                    *dpx = (OUT)(lut ? __ldg(lut + val) : (uint8_t)val);
            }
        }
#ifdef BM_TIMING
        { const long long t = clock64(); tB += t - t0; t0 = t; }
#endif
        __syncthreads();
#ifdef BM_TIMING
        { const long long t = clock64(); tB2 += t - t0; t0 = t; }
#endif
    }
#ifdef BM_TIMING
    if ((p.gate & 32) && lane == 0 && (warp == 0 || warp == 17) && blockIdx.x == 3 && blockIdx.y == 5)
        printf("warp %d rows %d: init %lld, A %lld, bar1 %lld, B %lld, bar2 %lld (cycles per row: A %lld bar1 %lld B %lld bar2 %lld)\n",
               warp, y1 - y0, tinit, tA, tB1, tB, tB2, tA / (y1 - y0), tB1 / (y1 - y0), tB / (y1 - y0), tB2 / (y1 - y0));
#endif
    if (STREAM) stream_signal(p, y0, y1, X0, X0 + TW);
}

}  // namespace mtb
