// kernels_lob.cuh -- 8-bit rank filter, "lanes own bins".
//
// The window histogram of one output pixel (256 bins, u16) is spread over a
// HALF-WARP: lane q of the half-warp owns bins [16q, 16q+16) as 8 packed
// u16 words in registers.  Each warp runs two independent streams (one per
// half-warp), each sliding right along a row segment of L outputs.
//
// Column histograms.  The warp tile (2L output columns + 2r halo columns,
// rows [Y0,Y1)) keeps one 256-bin u8 histogram per column of its current
// row in shared memory (column counts <= n <= 255).  Moving down a row
// removes the pixel leaving each column's vertical span and adds the one
// entering it (the reference's column-tree update, _kernels.py:115-127).
//
// Horizontal step (the reference's window sync, _kernels.py:145-194, made
// eager and bin-parallel): every lane adds its 16-byte slice of the column
// entering the window and subtracts the slice of the column leaving it --
// one LDS.128 each, d = in + 0x80 - out per byte, widened into the u16 bins
// (IADD3 + PRMT).  Rank descent (the reference's extract_u,
// _kernels.py:229-253): per-lane bin sums, a segmented inclusive warp scan
// over the 16 lanes, a ballot for the first lane whose prefix reaches the
// rank, and a 16-bin binary descent inside that lane.
//
// The window at the start of each stream's row segment is re-summed from
// its 2r+1 columns (O(r) per row, amortised over L outputs).  Everything
// else is O(1) in the radius.  Exact integer counting throughout.
#pragma once
#include "common.cuh"
#include "kernels_ctmf.cuh"  // hsum16, ct_descend

namespace mtb {

struct LobGeom {
    int L, TW, NC, NCP;  // outputs per stream, tile width, halo'd columns, padded
    int col_bytes;       // NCP x 256
    int cum_bytes;       // NCP x 16
    int stage_bytes;     // staged rows
    int out_bytes;       // one output row of the tile
    int warp_bytes;
};

constexpr int LOB_STAGE_ROWS = 4;

__host__ __device__ inline LobGeom lob_geom(int L, int r) {
    LobGeom g;
    g.L = L;
    g.TW = 2 * L;
    g.NC = g.TW + 2 * r;
    g.NCP = (g.NC + 31) & ~31;
    g.col_bytes = g.NCP * 256;
    g.cum_bytes = g.NCP * 16;
    g.stage_bytes = LOB_STAGE_ROWS * ((g.NC + 16 + 15) & ~15);
    g.out_bytes = (g.TW + 15) & ~15;
    g.warp_bytes = g.col_bytes + g.cum_bytes + g.stage_bytes + g.out_bytes;
    return g;
}

// Column c stores its 16-bin chunk k at physical chunk (k + c) & 15, so
// that lanes updating neighbouring columns with similar values, and the two
// streams reading their slices, spread over the shared-memory banks.
__device__ __forceinline__ int lob_byte(int c, unsigned v) {
    return c * 256 + ((((int)(v >> 4) + c) & 15) << 4) + (int)(v & 15);
}
__device__ __forceinline__ const uint4 *lob_slice(const uint8_t *colh, int c, int q) {
    return reinterpret_cast<const uint4 *>(colh + c * 256 + (((q + c) & 15) << 4));
}

// W[0..7] += widened(in - out) for 16 u8 bins (in, out <= 127)
__device__ __forceinline__ void lob_step(uint32_t (&w)[8], const uint4 in, const uint4 out) {
    const uint32_t iv[4] = {in.x, in.y, in.z, in.w};
    const uint32_t ov[4] = {out.x, out.y, out.z, out.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t d = iv[j] + 0x80808080u - ov[j];
        w[2 * j] = w[2 * j] + __byte_perm(d, 0, 0x4140) - 0x00800080u;
        w[2 * j + 1] = w[2 * j + 1] + __byte_perm(d, 0, 0x4342) - 0x00800080u;
    }
}

__device__ __forceinline__ void lob_add(uint32_t (&w)[8], const uint4 in) {
    const uint32_t iv[4] = {in.x, in.y, in.z, in.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        w[2 * j] += __byte_perm(iv[j], 0, 0x4140);
        w[2 * j + 1] += __byte_perm(iv[j], 0, 0x4342);
    }
}

// cum[c][g] = number of pixels of column c below 16*g (g = 0..15), u8.
// A one-hot at value v changes cum[c][g] for every g > v>>4: a 16-byte add
// of 0x01 bytes above byte v>>4.
__device__ __forceinline__ void lob_cum_bump(uint8_t *cum, int c, unsigned v, bool add) {
    uint4 *p = reinterpret_cast<uint4 *>(cum + c * 16);
    uint4 t = *p;
    const int b = (int)(v >> 4) + 1;  // first g that counts v
    uint32_t m[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int sh = 8 * (b - 4 * j);  // bytes >= b within word j
        m[j] = sh <= 0 ? 0x01010101u : (sh >= 32 ? 0u : (0x01010101u << sh));
    }
    if (add) {
        t.x += m[0]; t.y += m[1]; t.z += m[2]; t.w += m[3];
    } else {
        t.x -= m[0]; t.y -= m[1]; t.z -= m[2]; t.w -= m[3];
    }
    *p = t;
}

template <int L>
__global__ void __launch_bounds__(32) k_lob_u8(SlabParams p, int tiles_x, int tiles_y) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x;
    const int tile = blockIdx.x;
    if (tile >= tiles_x * tiles_y) return;
    const int r = p.radius;
    const LobGeom g = lob_geom(L, r);
    uint8_t *colh = smem_raw;                       // [NCP][256]
    uint8_t *cum = smem_raw + g.col_bytes;          // [NCP][16]
    uint8_t *stage = cum + g.cum_bytes;             // [LOB_STAGE_ROWS][SPB]
    uint8_t *orow = stage + g.stage_bytes;          // [TW]
    const int SPB = (g.NC + 16 + 15) & ~15;

    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int W = p.W, H = p.H;
    const int X0 = tx * g.TW;
    const int Y0 = p.row_begin + ty * p.rows_per_cta;
    const int Y1 = min(Y0 + p.rows_per_cta, p.row_end);
    const uint8_t *src = static_cast<const uint8_t *>(p.src) + blockIdx.z * p.src_img_stride;
    uint8_t *dst = static_cast<uint8_t *>(p.dst) + blockIdx.z * p.dst_img_stride;
    const uint8_t *lut = static_cast<const uint8_t *>(p.lut);
    const uint32_t rank = p.rank;
    const int sx0 = max(0, X0 - r);
    const int sx1 = min(W, X0 + g.TW + r);
    const int A = ct_span_base(sx0);
    const bool aligned = ct_rows_aligned16(src, p.src_pitch);
    StageBar sbar = ct_stage_init(lane);

    const int q = lane & 15;        // bin slice [16q, 16q+16)
    const int sid = lane >> 4;      // stream
    const int cs = sid * L;         // stream's first window column index

    // --- column histograms at row Y0
    for (int i = lane; i < g.NCP * 16; i += 32) reinterpret_cast<uint4 *>(colh)[i] = make_uint4(0, 0, 0, 0);
    for (int j0 = -r; j0 <= r; j0 += LOB_STAGE_ROWS) {
        const int nr = min(LOB_STAGE_ROWS, r - j0 + 1);
        int gr[LOB_STAGE_ROWS];
#pragma unroll
        for (int k = 0; k < LOB_STAGE_ROWS; ++k) gr[k] = clampi(Y0 + j0 + k, 0, H - 1);
        __syncwarp();
        ct_stage(p, src, stage, SPB, gr, nr, A, sx1, aligned, lane, &sbar);
        __syncwarp();
        for (int c = lane; c < g.NC; c += 32) {
            const int si = clampi(X0 - r + c, 0, W - 1) - A;
            for (int k = 0; k < nr; ++k) colh[lob_byte(c, stage[k * SPB + si])] += 1;
        }
    }
    __syncwarp();
    // cumulative chunk counts per column
    for (int c = lane; c < g.NCP; c += 32) {
        uint32_t acc = 0;
        uint32_t out[4] = {0, 0, 0, 0};
        for (int k = 0; k < 16; ++k) {
            out[k >> 2] |= acc << (8 * (k & 3));
            const uint4 v = *reinterpret_cast<const uint4 *>(colh + c * 256 + (((k + c) & 15) << 4));
            // byte sum of 16 bytes (each <= 127, sum <= 127 per column)
            uint32_t t = __vsadu4(v.x, 0) + __vsadu4(v.y, 0) + __vsadu4(v.z, 0) + __vsadu4(v.w, 0);
            acc += t;
        }
        *reinterpret_cast<uint4 *>(cum + c * 16) = make_uint4(out[0], out[1], out[2], out[3]);
    }
    __syncwarp();

    // column c's slice for lane q: byte offset c*256 + ((q + c) & 15)*16
    auto slice_off = [&](int c) -> uint32_t { return (uint32_t)(c * 256 + (((q + c) & 15) << 4)); };

    for (int y = Y0; y < Y1; ++y) {
        if (y > Y0) {
            int gr[LOB_STAGE_ROWS];
            gr[0] = clampi(y - r - 1, 0, H - 1);
            gr[1] = clampi(y + r, 0, H - 1);
            if (gr[0] != gr[1]) {
                ct_stage(p, src, stage, SPB, gr, 2, A, sx1, aligned, lane, &sbar);
                __syncwarp();
                for (int c = lane; c < g.NC; c += 32) {
                    const int si = clampi(X0 - r + c, 0, W - 1) - A;
                    const unsigned vo = stage[si], vi = stage[SPB + si];
                    if (vo != vi) {
                        colh[lob_byte(c, vo)] -= 1;
                        colh[lob_byte(c, vi)] += 1;
                        if ((vo >> 4) != (vi >> 4)) {
                            lob_cum_bump(cum, c, vo, false);
                            lob_cum_bump(cum, c, vi, true);
                        }
                    }
                }
                __syncwarp();
            }
        }
        // --- stream window at its first output: columns cs .. cs+2r
        uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        {
            int c = cs;
            for (; c + 1 <= cs + 2 * r; c += 2) {
                const uint4 a = *reinterpret_cast<const uint4 *>(colh + slice_off(c));
                const uint4 b = *reinterpret_cast<const uint4 *>(colh + slice_off(c + 1));
                lob_add(w, make_uint4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w));
            }
            if (c <= cs + 2 * r) lob_add(w, *reinterpret_cast<const uint4 *>(colh + slice_off(c)));
        }
        int gq = 0;          // lane (bin slice) holding this stream's rank value
        uint32_t E = 0;      // number of window pixels below 16*gq
        bool known = false;  // gq/E valid for the current window
        for (int s = 0; s < L; ++s) {
            if (s > 0) {
                const int cin = cs + s + 2 * r, cout = cs + s - 1;
                const uint4 iv = *reinterpret_cast<const uint4 *>(colh + slice_off(cin));
                const uint4 ov = *reinterpret_cast<const uint4 *>(colh + slice_off(cout));
                lob_step(w, iv, ov);
                E = E + cum[cin * 16 + gq] - cum[cout * 16 + gq];
            }
            const uint32_t tsum = hsum16(((w[0] + w[1]) + (w[2] + w[3])) + ((w[4] + w[5]) + (w[6] + w[7])));
            // fast path: the rank value stayed in slice gq
            const bool ok_here = known && (q != gq || (E < rank && rank <= E + tsum));
            if (!__all_sync(0xffffffffu, ok_here)) {
                uint32_t incl = tsum;
#pragma unroll
                for (int d = 1; d < 16; d <<= 1) {
                    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d, 16);
                    incl += (q >= d) ? t : 0u;
                }
                const uint32_t ball = __ballot_sync(0xffffffffu, incl >= rank);
                gq = __ffs((ball >> (16 * sid)) & 0xffffu) - 1;
                E = __shfl_sync(0xffffffffu, incl - tsum, (sid << 4) | gq);
                known = true;
            }
            if (q == gq) {
                uint32_t k = rank - E;
                const int b = ct_descend(w, k);
                orow[cs + s] = (uint8_t)(16 * q + b);
            }
        }
        __syncwarp();
        // --- store the row (optionally through the value map)
        uint8_t *drow = dst + (int64_t)(y - p.row_begin) * p.dst_pitch;
        for (int i = lane; i < g.TW; i += 32) {
            const int x = X0 + i;
            if (x < W) {
                const uint8_t v = orow[i];
                drow[x] = lut ? __ldg(lut + v) : v;
            }
        }
        __syncwarp();
    }
}

}  // namespace mtb
