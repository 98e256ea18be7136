// kernels_lowsel16.cuh -- 16-bit rank filter on widely spread data, second
// pass: "low byte from shared candidate buckets".
//
// The reference descends a 3-level tree per pixel (_kernels.py:229-253
// extract_u on the 16-bit tree): the top levels pick the coarse bin, the last
// one the value inside it.  Here the first pass (k_colhist4p_u8 keyed by the
// high byte, kernels_colhist.cuh) leaves, per output pixel, the high byte H of
// the result and the rank k' of the result among the window values whose high
// byte is H.  On spread data only ~n^2/256 window values have that high byte,
// and neighbouring pixels want nearby H, so ONE WARP resolves a block of
// 32 x PH output pixels together:
//   1. [Hmin, Hmax] = the range of H over the block, taken in chunks of up to
//      64 consecutive keys;
//   2. the warp scans the union of the block's windows, (32 + 2r) x (PH + 2r)
//      replicate-clamped source values, once per chunk, and stages every value
//      whose key lies in the chunk in shared memory together with its window
//      coordinates (value << 16 | dy << 8 | dx; up to 512 entries);
//   3. the staged entries are counted per key, placed into one bucket per key
//      (exclusive prefix of the counts: no slot is wasted on an empty key), and
//      every bucket is sorted by counting ranks (entries are distinct, so an
//      entry's place is the number of smaller entries of its bucket);
//   4. every pixel walks the bucket of its H in ascending order, counts the
//      entries inside its own window, and stops at the k'-th: that entry's
//      value is the result.
// The scan is shared by 32 PH pixels, so a pixel pays (32 + 2r)(PH + 2r) /
// (32 PH) loads instead of the n per level of the gather kernels or the
// per-column run lookups of k_colhist16c_u16.
//
// A chunk whose entries do not fit is halved (fewer keys per chunk) and
// repeated; a block where one key alone overflows 512 entries (locally compact data) is flagged in SlabParams::todo and left to
// k_colhist16_u16, which then works on the tiles holding such blocks only.
// Exact for any image; the data only decide which kernel resolves a block.
#pragma once
#include "common.cuh"

namespace mtb {

constexpr int LS_WARPS = 8;    // warps per CTA, side by side (256 output columns)
constexpr int LS_CAP = 512;    // bucket entries per warp (NB buckets x BCAP)
constexpr int LS_KEYS = 64;    // keys (buckets) per chunk at most

// One block: the 32 x PH output pixels at columns xb.., block row `by` of image
// blockIdx.z; called by a whole warp.  buf / srt / ctr / kmap: the warp's buckets and counters.
// PH > 0: compile-time block height, the block's (H, k') words in registers;
// PH == 0: block height p.todo_bh, the words re-read where they are used.
template <int PH, int NI>
__device__ __forceinline__ void ls_block(const SlabParams &p, const uint32_t *__restrict__ hk, int xb, int by,
                                         uint32_t *buf, uint32_t *srt, int *ctr, unsigned char *kmap) {
    const int lane = threadIdx.x & 31;
    const int r = p.radius, r2 = 2 * r, W = p.W, H = p.H;
    const int PHR = PH ? PH : p.todo_bh;
    const int yb = p.row_begin + by * PHR;
    const int ph = min(PHR, p.row_end - yb);
    const int rows = p.row_end - p.row_begin;
    const uint16_t *src = static_cast<const uint16_t *>(p.src) + blockIdx.z * p.src_img_stride;
    uint16_t *dst = static_cast<uint16_t *>(p.dst) + blockIdx.z * p.dst_img_stride;
    const uint16_t *lut = static_cast<const uint16_t *>(p.lut);
    const uint32_t *hkp = hk + ((int64_t)blockIdx.z * rows + (yb - p.row_begin)) * W + xb + lane;
    const bool valid = xb + lane < W;
    const int ks = key_shift(p);  // coarse key of a pixel: min(v >> ks, 255) (8: the high byte)

    // ---- the block's (H, k') and the range of H
    uint32_t myhk[PH ? PH : 1];
    auto hk_at = [&](int py) -> uint32_t {  // 0xffffffff: no pixel
        if (PH) return myhk[py];
        return valid && py < ph ? __ldg(hkp + (int64_t)py * W) : 0xffffffffu;
    };
    int hmin = 255, hmax = 0;
#pragma unroll
    for (int py = 0; py < PHR; ++py) {
        uint32_t w = 0xffffffffu;
        if (valid && py < ph) {
            w = __ldg(hkp + (int64_t)py * W);
            const int h = (int)(w >> 16);
            hmin = min(hmin, h);
            hmax = max(hmax, h);
        }
        if (PH) myhk[py] = w;
    }
    hmin = __reduce_min_sync(0xffffffffu, hmin);
    hmax = __reduce_max_sync(0xffffffffu, hmax);

    // the union of the windows: virtual columns xb-r .. xb+31+r (dx = 0 .. UW-1),
    // virtual rows yb-r .. yb+ph-1+r (dy = 0 .. UH-1), replicate-clamped into
    // the image.  Only the cells inside the image are scanned (dx in [cL, cR],
    // dy in [jT, jB]); a border pixel stands for every virtual cell clamped
    // onto it, and the walk below weighs it by how many of those lie in the
    // pixel's window.
    const int UW = 32 + r2, UH = ph + r2;
    const int cL = max(0, r - xb), cR = min(UW - 1, W - 1 - xb + r);
    const int jT = max(0, r - yb), jB = min(UH - 1, H - 1 - yb + r);
    const bool border = cL > 0 || cR < UW - 1 || jT > 0 || jB < UH - 1;  // (warp-uniform)
    // image borders in window coordinates (out of reach when the border is not in the union)
    const int dxL = xb - r <= 0 ? r - xb : -1000, dxR = xb + 31 + r >= W - 1 ? W - 1 - xb + r : 1000;
    const int dyT = yb - r <= 0 ? r - yb : -1000, dyB = yb + ph - 1 + r >= H - 1 ? H - 1 - yb + r : 1000;
    int gx[NI];
    unsigned okc = 0;  // bit i: this lane's column of step i is inside the image
#pragma unroll
    for (int i = 0; i < NI; ++i) {
        const int c = lane + 32 * i;
        gx[i] = clampi(xb - r + c, 0, W - 1);
        okc |= (c >= cL && c <= cR) ? 1u << i : 0u;
    }
    const uint16_t *row0 = src_row(p, src, yb - r + jT);

    // chunks of up to LS_KEYS consecutive keys; a chunk whose entries do not fit
    // LS_CAP is halved and repeated
    int width = min(hmax - hmin + 1, LS_KEYS);
    int *kcnt = ctr, *koff = ctr + LS_KEYS, *kfill = ctr + 2 * LS_KEYS, *staged = ctr + 3 * LS_KEYS;
    for (int h0 = hmin; h0 <= hmax;) {
        const int h1 = min(h0 + width - 1, hmax);
        const unsigned hspan = (unsigned)(h1 - h0);
        bool want = false;
#pragma unroll
        for (int py = 0; py < PHR; ++py) want |= (hk_at(py) >> 16) - (unsigned)h0 <= hspan;
        if (!__any_sync(0xffffffffu, want)) {  // no pixel of the block has its H here
            h0 = h1 + 1;
            continue;
        }
        kcnt[lane] = kcnt[lane + 32] = 0;
        kfill[lane] = kfill[lane + 32] = 0;
        for (int i = lane; i < LS_CAP / 4; i += 32) reinterpret_cast<uint32_t *>(kmap)[i] = 0xffffffffu;
        if (lane == 0) *staged = 0;
        __syncwarp();
        // ---- scan, two rows per step (all loads of a step in flight together):
        // matching values are staged in scan order (in srt)
        auto drop = [&](unsigned v, int j, int i, bool on) {
            const unsigned b = min(v >> ks, 255u) - (unsigned)h0;
            if (on && ((okc >> i) & 1u) && b <= hspan) {
                const int pos = atomicAdd(staged, 1);
                if (pos < LS_CAP) srt[pos] = (v << 16) | ((unsigned)j << 8) | (unsigned)(lane + 32 * i);
            }
        };
        const uint16_t *row = row0;
        for (int j = jT; j <= jB; j += 2, row += 2 * p.src_pitch) {
            const bool two = j < jB;
            unsigned v0[NI], v1[NI];
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                v0[i] = __ldg(row + gx[i]);
                v1[i] = two ? (unsigned)__ldg(row + p.src_pitch + gx[i]) : 0u;
            }
#pragma unroll
            for (int i = 0; i < NI; ++i) drop(v0[i], j, i, true);
#pragma unroll
            for (int i = 0; i < NI; ++i) drop(v1[i], j + 1, i, two);
        }
        __syncwarp();
        // ---- entries per key (one lane per staged entry), then the bucket offsets:
        // exclusive prefix of the counts, every bucket on an even slot (the walk
        // reads entry pairs); lane l owns keys 2l and 2l + 1
        const int cnt = *staged;
        auto key_of = [&](uint32_t e) -> int { return (int)(min((e >> 16) >> ks, 255u) - (unsigned)h0); };
        for (int t = lane; t < min(cnt, LS_CAP); t += 32) atomicAdd(kcnt + key_of(srt[t]), 1);
        __syncwarp();
        const int ca = (kcnt[2 * lane] + 1) & ~1, cb = (kcnt[2 * lane + 1] + 1) & ~1;
        int incl = ca + cb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int padded = __shfl_sync(0xffffffffu, incl, 31);
        if (cnt > LS_CAP || padded > LS_CAP) {
            if (width == 1) {  // locally compact data: leave the block to the two-phase kernel
                if (lane == 0) p.todo[((size_t)blockIdx.z * p.todo_nby + by) * p.todo_nbx + (xb >> 5)] = 1;
                __syncwarp();
                return;
            }
            width = (width + 1) >> 1;  // fewer keys per chunk; repeat from h0
            __syncwarp();
            continue;
        }
        koff[2 * lane] = incl - ca - cb;
        koff[2 * lane + 1] = incl - cb;
        __syncwarp();
        // ---- place the staged entries into their buckets (srt -> buf; kmap: the key
        // of every occupied slot), then sort every bucket (buf -> srt): an entry goes
        // to the count of smaller entries of its bucket (entries are distinct).  One
        // lane per entry / per slot.
        for (int t = lane; t < cnt; t += 32) {
            const uint32_t e = srt[t];
            const int k = key_of(e);
            const int slot = koff[k] + atomicAdd(kfill + k, 1);
            buf[slot] = e;
            kmap[slot] = (unsigned char)k;
        }
        __syncwarp();
        for (int t = lane; t < padded; t += 32) {
            const int k = kmap[t];
            if (k != 0xff) {
                const uint32_t *bk = buf + koff[k];
                const uint32_t e = buf[t];
                const int nb = kcnt[k];
                int rank = 0;
                for (int q = 0; q < nb; ++q) rank += bk[q] < e ? 1 : 0;
                srt[koff[k] + rank] = e;
            }
        }
        __syncwarp();
        // ---- every pixel of the chunk: the k'-th entry of its bucket inside its
        // window (pixel (lane, py): dx in [lane, lane + 2r], dy in [py, py + 2r])
#pragma unroll
        for (int py = 0; py < PHR; ++py) {
            const uint32_t w = hk_at(py);
            const unsigned b = (w >> 16) - (unsigned)h0;
            if (b > hspan) continue;
            const uint32_t k = w & 0xffffu;
            const uint32_t *bk = srt + koff[b];
            const int nb = kcnt[b];
            uint32_t c = 0, res = 0;
            if (!border) {
                // two entries per step (buckets are 64-byte aligned; an odd bucket's last
                // partner is not counted)
                // both coordinate tests of an entry at once: dx and dy spread into two 16-bit
                // fields g; d >= q sets bit 8 of the field d - q + 256, d <= q + 2r sets bit 8
                // of q + 2r - d + 256 (no borrow or carry crosses a field: d, q < 256, 2r < 256)
                const uint32_t P = ((uint32_t)py << 16) | (uint32_t)lane, M = 0x01000100u;
                const uint32_t C1 = M - P, C2 = P + (((uint32_t)r2 << 16) | (uint32_t)r2) + M;
                auto inside = [&](uint32_t e) -> bool {
                    const uint32_t g = __byte_perm(e, 0, 0x4140);  // dx | dy << 16
                    return ((g + C1) & (C2 - g) & M) == M;
                };
                for (int i = 0; i < nb; i += 2) {
                    const uint2 ee = *reinterpret_cast<const uint2 *>(bk + i);
                    const bool in0 = inside(ee.x), in1 = i + 1 < nb && inside(ee.y);
                    const uint32_t c0 = c + (in0 ? 1u : 0u), c1 = c0 + (in1 ? 1u : 0u);
                    if (c1 >= k) {  // (c < k before: the first of the two to reach k)
                        res = (c0 == k ? ee.x : ee.y) >> 16;
                        break;
                    }
                    c = c1;
                }
            } else {
                // weight of an entry = virtual cells of the window clamped onto it:
                // [dx, dx] x [dy, dy] for an interior pixel, open-ended towards a border it lies on
                for (int i = 0; i < nb; ++i) {
                    const uint32_t e = bk[i];
                    const int dx = (int)(e & 0xffu), dy = (int)((e >> 8) & 0xffu);
                    const int xa = dx == dxL ? -1000 : dx, xz = dx == dxR ? 1000 : dx;
                    const int ya = dy == dyT ? -1000 : dy, yz = dy == dyB ? 1000 : dy;
                    const int wx = max(0, min(xz, lane + r2) - max(xa, lane) + 1);
                    const int wy = max(0, min(yz, py + r2) - max(ya, py) + 1);
                    c += (uint32_t)(wx * wy);
                    if (c >= k) {
                        res = e >> 16;
                        break;
                    }
                }
            }
            dst[(int64_t)(yb + py - p.row_begin) * p.dst_pitch + xb + lane] = lut ? __ldg(lut + res) : (uint16_t)res;
        }
        __syncwarp();  // the buckets are reused by the next chunk
        h0 = h1 + 1;
    }
}

// hk: [image][row - row_begin][x] words H << 16 | k' (pitch W); PH output rows
// per block; NI = ceil((32 + 2r) / 32) column steps of the scan.  A CTA takes `seg` vertically adjacent block
// rows of its 256 columns (grid.y = ceil(block rows / seg)): consecutive
// blocks share all but PH of their PH + 2r source rows in L1, and a gated
// launch that has nothing to do (compact data) is a few thousand CTAs, not
// one per block row.
template <int PH, int NI>
__global__ void __launch_bounds__(32 * LS_WARPS, 4) k_lowsel_u16(SlabParams p, const uint32_t *__restrict__ hk, int seg) {
    __shared__ uint32_t bufs[LS_WARPS][LS_CAP];  // buckets as scanned
    __shared__ uint32_t srts[LS_WARPS][LS_CAP];  // buckets sorted
    __shared__ int ctrs[LS_WARPS][3 * LS_KEYS + 2];      // per key: entries, first slot, placed; then: staged
    __shared__ __align__(4) unsigned char kmaps[LS_WARPS][LS_CAP];  // the key of every bucket slot
    if (gate_off(p)) return;
    const int warp = threadIdx.x >> 5;
    const int xb = (blockIdx.x * LS_WARPS + warp) * 32;  // first output column of the warp's blocks
    if (xb >= p.W) return;                                // (warp-uniform; the kernel has no CTA barriers)
    const int by1 = min((int)(blockIdx.y + 1) * seg, p.todo_nby);
    for (int by = blockIdx.y * seg; by < by1; ++by) {
        ls_block<PH, NI>(p, hk, xb, by, bufs[warp], srts[warp], ctrs[warp], kmaps[warp]);
        __syncwarp();  // the buckets are reused by the next block
    }
}

}  // namespace mtb
