// kernels_colhist.cuh -- 8-bit rank filter from u8 column histograms with a
// per-pixel window GATHER (one pass, no per-tile fine passes).
//
// The CTA owns output columns [X0, X0 + T*S) for rows [y0, y1) of a slab and
// keeps, for every column of the halo'd stripe [X0-r, X0+T*S+r), the full
// 256-bin histogram of the column's current vertical span (u8 counts: a
// column holds n <= 255 pixels) plus its 16 coarse counts.  Moving down a row
// is one decrement + one increment per column and level (the reference's
// per-column trees, _kernels.py:115-165, with the sync step replaced by a
// gather).
//
// Thread t outputs the S pixels x = X0 + t*S + s.  For the first it GATHERS
// the window's coarse histogram from its 2r+1 columns: a column's 16 coarse
// counts are one 16-B record (4 words of 4 u8 lanes) and G records with
// G*n <= 255 add with plain 32-bit adds without a carry crossing a byte
// lane; each group is then widened into 8 packed u16 pairs.  A 4-step
// binary descent (ct_descend) picks the coarse bin B and the residual rank;
// the same gather over the columns' 16-B fine record of bin B gives the low
// nibble.  Pixels s > 0 slide the coarse window by one column
// (+C[x+r] - C[x-r-1]) and slide the fine window as well when their coarse
// bin equals the previous pixel's (regather otherwise).
//
// Shared-memory layout (bank-conflict free gathers): records are stored as
// [chunk][column position] with pos(c) = (c % S) * NCS + c / S, so the 32
// threads of a warp, which read columns c = t*S + j for the same j, hit 32
// consecutive 16-B records.  Chunks 0..15 are the fine records (bins
// 16B..16B+15), chunk 16 the coarse record.
#pragma once
#include "common.cuh"
#include "kernels_ctmf.cuh"  // ct_descend
#include "kernels_vert.cuh"  // lower_bound_multi

namespace mtb {

struct ColhistGeom {
    int TW, NC, NCS, NPOS;  // tile width, stripe columns, columns per phase, positions
    int bytes;              // dynamic shared memory
};

__host__ __device__ inline ColhistGeom colhist_geom(int T, int S, int r) {
    ColhistGeom g;
    g.TW = T * S;
    g.NC = g.TW + 2 * r;
    // phase length padded so a record row is a multiple of 8 records (32
    // words): the per-column byte updates then fall in bank 4c+byte/4
    // whatever the chunk (measured: a radix-4 kernel gained 20% this way)
    g.NCS = (g.NC + S - 1) / S;
    g.NCS = (g.NCS + (8 / S > 0 ? 8 / S : 1) - 1) / (8 / S > 0 ? 8 / S : 1) * (8 / S > 0 ? 8 / S : 1);
    g.NPOS = g.NCS * S;
    g.bytes = 17 * g.NPOS * 16;
    return g;
}

template <int S>
__device__ __forceinline__ int ch_pos(int c, int NCS) {
    return (c % S) * NCS + c / S;
}

// widen 4 u8 lanes into two packed u16 pairs and add
__device__ __forceinline__ void ch_widen_add(uint32_t (&w)[8], const uint4 &t) {
    w[0] += __byte_perm(t.x, 0, 0x4140);
    w[1] += __byte_perm(t.x, 0, 0x4342);
    w[2] += __byte_perm(t.y, 0, 0x4140);
    w[3] += __byte_perm(t.y, 0, 0x4342);
    w[4] += __byte_perm(t.z, 0, 0x4140);
    w[5] += __byte_perm(t.z, 0, 0x4342);
    w[6] += __byte_perm(t.w, 0, 0x4140);
    w[7] += __byte_perm(t.w, 0, 0x4342);
}

// w += widen(a) - widen(b): per-lane results stay >= 0, so no borrow crosses lanes
__device__ __forceinline__ void ch_widen_slide(uint32_t (&w)[8], const uint4 &a, const uint4 &b) {
    w[0] += __byte_perm(a.x, 0, 0x4140) - __byte_perm(b.x, 0, 0x4140);
    w[1] += __byte_perm(a.x, 0, 0x4342) - __byte_perm(b.x, 0, 0x4342);
    w[2] += __byte_perm(a.y, 0, 0x4140) - __byte_perm(b.y, 0, 0x4140);
    w[3] += __byte_perm(a.y, 0, 0x4342) - __byte_perm(b.y, 0, 0x4342);
    w[4] += __byte_perm(a.z, 0, 0x4140) - __byte_perm(b.z, 0, 0x4140);
    w[5] += __byte_perm(a.z, 0, 0x4342) - __byte_perm(b.z, 0, 0x4342);
    w[6] += __byte_perm(a.w, 0, 0x4140) - __byte_perm(b.w, 0, 0x4140);
    w[7] += __byte_perm(a.w, 0, 0x4342) - __byte_perm(b.w, 0, 0x4342);
}

// window histogram (16 bins, packed u16 pairs) of chunk `chunk` over the
// columns k0 .. k0+n-1: groups of G records (G*n <= 255, so the u8 lanes of a
// group sum never carry) added with IADD3, then widened into the u16 pairs.
// Fully unrolled groups; the ragged tail is a predicated group.
template <int S, int G, int M>
__device__ __forceinline__ void ch_gather(const uint4 *rec, int chunk, int k0, int n, int NCS,
                                          uint32_t (&w)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = 0;
    const uint4 *base = rec + chunk * (NCS * S);
    int j = 0;
    for (; j < n - M; j += G) {
        uint4 t = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int q = 0; q < G; q += 2) {
            const uint4 a = base[ch_pos<S>(k0 + j + q, NCS)];
            const uint4 b = q + 1 < G ? base[ch_pos<S>(k0 + j + q + 1, NCS)] : make_uint4(0, 0, 0, 0);
            t.x += a.x + b.x;
            t.y += a.y + b.y;
            t.z += a.z + b.z;
            t.w += a.w + b.w;
        }
        ch_widen_add(w, t);
    }
    if (M > 0) {
        uint4 t = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int q = 0; q < M; ++q) {
            const uint4 a = base[ch_pos<S>(k0 + j + q, NCS)];
            t.x += a.x;
            t.y += a.y;
            t.z += a.z;
            t.w += a.w;
        }
        ch_widen_add(w, t);
    }
}

// NF > 0: the window side as a compile-time constant (fully unrolled
// gathers; measured 16-23% faster than the runtime-n loops at r = 6..15)
template <int T, int S, int G, int M, int NF = 0>
__global__ void __launch_bounds__(T) k_colhist_u8(SlabParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    const int r = NF ? NF / 2 : p.radius, H = p.H, W = p.W, n = NF ? NF : 2 * r + 1;
    const ColhistGeom g = colhist_geom(T, S, r);
    const int NCS = g.NCS, NPOS = g.NPOS;
    uint4 *rec = reinterpret_cast<uint4 *>(smem_raw);       // [17][NPOS] 16-B records
    uint8_t *recb = smem_raw;
    const int X0 = blockIdx.x * g.TW;
    const int y0 = p.row_begin + blockIdx.y * p.rows_per_cta;
    if (y0 >= p.row_end) return;  // CTA-uniform (barriers below)
    const int y1 = min(y0 + p.rows_per_cta, p.row_end);
    stream_wait_rows(p, y1 + r);
    const uint8_t *src = static_cast<const uint8_t *>(p.src) + blockIdx.z * p.src_img_stride;
    uint8_t *dst = static_cast<uint8_t *>(p.dst) + blockIdx.z * p.dst_img_stride;
    const uint8_t *lut = static_cast<const uint8_t *>(p.lut);
    const uint32_t rank = p.rank;

    // ---- column histograms of rows clamp(y0-r .. y0+r)
    for (int pos = tid; pos < 17 * NPOS; pos += T) rec[pos] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    for (int c = tid; c < g.NC; c += T) {
        const int gx = clampi(X0 - r + c, 0, W - 1);
        const int pc = ch_pos<S>(c, NCS);
        uint32_t *rw = reinterpret_cast<uint32_t *>(smem_raw);
        for (int j = -r; j <= r; ++j) {
            const unsigned v = __ldg(src_row(p, src, clampi(y0 + j, 0, H - 1)) + gx);
            atomicAdd(rw + ((v >> 4) * NPOS + pc) * 4 + ((v & 15) >> 2), 1u << (8 * (v & 3)));
            atomicAdd(rw + (16 * NPOS + pc) * 4 + (v >> 6), 1u << (8 * ((v >> 4) & 3)));
        }
    }
    __syncthreads();

    const int k0 = tid * S;  // stripe column of the first window's left edge
    const int xt = X0 + k0;
    // one shared-memory atomic add per counter (see ch4_bump_upd): the
    // 32-bit word holding the byte, +-1 shifted into it
    uint32_t *recw = reinterpret_cast<uint32_t *>(smem_raw);
    auto bump = [&](int c, unsigned vo, unsigned vi) {
        const int pc = ch_pos<S>(c, NCS);
        atomicAdd(recw + ((vo >> 4) * NPOS + pc) * 4 + ((vo & 15) >> 2), 0xffffffffu << (8 * (vo & 3)));
        atomicAdd(recw + ((vi >> 4) * NPOS + pc) * 4 + ((vi & 15) >> 2), 1u << (8 * (vi & 3)));
        atomicAdd(recw + (16 * NPOS + pc) * 4 + (vo >> 6), 0xffffffffu << (8 * ((vo >> 4) & 3)));
        atomicAdd(recw + (16 * NPOS + pc) * 4 + (vi >> 6), 1u << (8 * ((vi >> 4) & 3)));
    };
    // the stripe columns this thread moves down each row; their leaving /
    // entering pixels of the NEXT row are loaded a row ahead (latency hidden
    // behind the gathers)
    constexpr int CH_PF = 2;
    int gxs[CH_PF];
#pragma unroll
    for (int u = 0; u < CH_PF; ++u) gxs[u] = clampi(X0 - r + min(tid + u * T, g.NC - 1), 0, W - 1);
    unsigned pvo[CH_PF], pvi[CH_PF];
    auto prefetch = [&](int yn) {
        const uint8_t *ro = src_row(p, src, clampi(yn - r - 1, 0, H - 1));
        const uint8_t *ri = src_row(p, src, clampi(yn + r, 0, H - 1));
#pragma unroll
        for (int u = 0; u < CH_PF; ++u) {
            pvo[u] = __ldg(ro + gxs[u]);
            pvi[u] = __ldg(ri + gxs[u]);
        }
    };
    if (y0 + 1 < y1) prefetch(y0 + 1);
    for (int y = y0; y < y1; ++y) {
        if (y > y0) {
            __syncthreads();  // previous row's gathers done
#pragma unroll
            for (int u = 0; u < CH_PF; ++u) {
                const int c = tid + u * T;
                if (c < g.NC) bump(c, pvo[u], pvi[u]);  // (vo == vi cancels: no data-dependent branch)
            }
            if (g.NC > CH_PF * T) {  // narrow CTA, wide halo: the rest without prefetch
                const uint8_t *ro = src_row(p, src, clampi(y - r - 1, 0, H - 1));
                const uint8_t *ri = src_row(p, src, clampi(y + r, 0, H - 1));
                for (int c = tid + CH_PF * T; c < g.NC; c += T) {
                    const int gx = clampi(X0 - r + c, 0, W - 1);
                    const unsigned vo = __ldg(ro + gx), vi = __ldg(ri + gx);
                    if (vo != vi) bump(c, vo, vi);
                }
            }
            if (y + 1 < y1) prefetch(y + 1);
            __syncthreads();
        }
        uint32_t wc[8], wf[8];
        int prevB = -1;
        uint32_t outw = 0;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (s == 0) {
                ch_gather<S, G, M>(rec, 16, k0, n, NCS, wc);
            } else {
                ch_widen_slide(wc, rec[16 * NPOS + ch_pos<S>(k0 + s + 2 * r, NCS)],
                               rec[16 * NPOS + ch_pos<S>(k0 + s - 1, NCS)]);
            }
            uint32_t k = rank;
            const int B = ct_descend(wc, k);
            if (B == prevB) {
                ch_widen_slide(wf, rec[B * NPOS + ch_pos<S>(k0 + s + 2 * r, NCS)],
                               rec[B * NPOS + ch_pos<S>(k0 + s - 1, NCS)]);
            } else {
                ch_gather<S, G, M>(rec, B, k0 + s, n, NCS, wf);
                prevB = B;
            }
            const int lo = ct_descend(wf, k);
            unsigned v = (unsigned)(B * 16 + lo);
            if (lut) v = xt + s < W ? __ldg(lut + v) : 0u;
            outw |= v << (8 * (s & 3));
            if ((s & 3) == 3 || s == S - 1) {
                // store the (up to) 4 bytes of this group
                const int xs = xt + (s & ~3);
                uint8_t *o = dst + (int64_t)(y - p.row_begin) * p.dst_pitch + xs;
                const int cnt = (s & 3) + 1;
                if (xs + cnt <= W && cnt == 4 && (reinterpret_cast<uintptr_t>(o) & 3) == 0) {
                    *reinterpret_cast<uint32_t *>(o) = outw;
                } else {
                    for (int q = 0; q < cnt; ++q)
                        if (xs + q < W) o[q] = (uint8_t)(outw >> (8 * q));
                }
                outw = 0;
            }
        }
    }
    stream_signal(p, y0, y1, X0, X0 + g.TW);
}

}  // namespace mtb

namespace mtb {

// ---------------------------------------------------------------------------
// Radix-4 variant: four levels of 4 bins (base-4 digits of the value), every
// column record one u32 of 4 u8 counts.  Per pixel the thread gathers 4 x n
// words (16 B per window column instead of 32 B for the 16 x 16 split: the
// 16-bin gathers above are bound by shared-memory bandwidth) and descends 2
// steps per level.  Records per column: level 0 (1), level 1 (4, by the top
// digit), level 2 (16, by the top two digits), level 3 (64) = 85 words.
// Layout [record id][column]: thread t reads column t + j, so a warp's 32
// loads are 32 consecutive words.
constexpr int CH4_RECS = 85;

// record row stride: a multiple of 32 words, so a warp's per-column byte
// updates (column c -> bank c mod 32, whatever the record row) never
// conflict
__host__ __device__ constexpr int ch4_stride(int ncol) { return (ncol + 31) & ~31; }
__host__ __device__ constexpr int colhist4_bytes(int T, int r) { return CH4_RECS * ch4_stride(T + 2 * r) * 4; }

// 4 bins (packed u16 pairs w0 = {b0, b1}, w1 = {b2, b3}): smallest digit d
// with cumsum(bins[0..d]) >= k; leaves the rank within bin d in k
__device__ __forceinline__ int ch4_descend(uint32_t w0, uint32_t w1, uint32_t &k) {
    const uint32_t s = hsum16(w0);
    const bool r1 = s < k;
    k -= r1 ? s : 0u;
    const uint32_t w = r1 ? w1 : w0;
    const uint32_t s2 = w & 0xffffu;
    const bool r2 = s2 < k;
    k -= r2 ? s2 : 0u;
    return (r1 ? 2 : 0) | (r2 ? 1 : 0);
}

// window counts of record row `rp` over columns k0 .. k0+n-1: full groups of
// G words (carry-free), then the M = n mod G tail words (compile-time)
template <int G, int M>
__device__ __forceinline__ void ch4_gather(const uint32_t *rp, int n, uint32_t &w0, uint32_t &w1) {
    w0 = 0;
    w1 = 0;
    const uint32_t *e = rp + (n - M);
    for (; rp < e; rp += G) {
        uint32_t t = 0;
#pragma unroll
        for (int q = 0; q < G; q += 2) t += rp[q] + (q + 1 < G ? rp[q + 1] : 0u);
        w0 += __byte_perm(t, 0, 0x4140);
        w1 += __byte_perm(t, 0, 0x4342);
    }
    if (M > 0) {
        uint32_t t = 0;
#pragma unroll
        for (int q = 0; q < M; ++q) t += rp[q];
        w0 += __byte_perm(t, 0, 0x4140);
        w1 += __byte_perm(t, 0, 0x4342);
    }
}

__device__ __forceinline__ void ch4_bump(uint8_t *recb, int NCOL, int c, unsigned v, int d) {
    // record ids: 0 | 1 + (v>>6) | 5 + (v>>4) | 21 + (v>>2); byte = next digit
    recb[(0 * NCOL + c) * 4 + (v >> 6)] += d;
    recb[((1 + (v >> 6)) * NCOL + c) * 4 + ((v >> 4) & 3)] += d;
    recb[((5 + (v >> 4)) * NCOL + c) * 4 + ((v >> 2) & 3)] += d;
    recb[((21 + (v >> 2)) * NCOL + c) * 4 + (v & 3)] += d;
}

// The same for the per-row updates: one shared-memory atomic add per level
// (a single instruction; the word belongs to this thread's column, so
// there is no contention), the +-1 shifted into the byte of the digit (a
// decrement never borrows: the count it decrements is >= 1).  Measured
// 9-20% faster kernels at r = 5..31 than byte read-modify-writes.  The
// column builds of ch4_sweep and k_colhist16s keep the byte form (atomic
// builds made the 16-bit keyed sweeps 20% slower); k_colhist4p uses atomics
// for its build as well.
__device__ __forceinline__ void ch4_bump_upd(uint8_t *recb, int NCOL, int c, unsigned v, int d) {
    uint32_t *rw = reinterpret_cast<uint32_t *>(recb);
    const unsigned one = (unsigned)d;
    atomicAdd(rw + (0 * NCOL + c), one << (8 * (v >> 6)));
    atomicAdd(rw + ((1 + (v >> 6)) * NCOL + c), one << (8 * ((v >> 4) & 3)));
    atomicAdd(rw + ((5 + (v >> 4)) * NCOL + c), one << (8 * ((v >> 2) & 3)));
    atomicAdd(rw + ((21 + (v >> 2)) * NCOL + c), one << (8 * (v & 3)));
}

// PL = number of levels with pair records (3: levels 0-2, 21 record rows;
// 2: levels 0-1, 5 rows) -- fewer when shared memory would otherwise drop
// the CTA below two per SM.
__host__ __device__ constexpr int ch4p_recs(int PL) { return PL >= 3 ? 21 : (PL == 2 ? 5 : 1); }

// record rows padded to a multiple of 32 columns (conflict-free updates;
// pair and quad alignment)
__host__ __device__ constexpr int colhist4p_ncolp(int T, int r) { return (T + 2 * r + 31) & ~31; }
__host__ __device__ constexpr int colhist4p_bytes(int T, int r, int PL) {
    const int ncp = colhist4p_ncolp(T, r);
    return (CH4_RECS * ncp + ch4p_recs(PL) * (ncp / 2)) * 4;
}

// PL = 4: three pair levels and NO level-2 single records (see
// k_colhist4p_u8): singles are level 0 (row 0), level 1 (rows 1-4) and
// level 3 (rows 5-68); the one single column of a level-2 pair gather
// derives its word from its four level-3 words.
__host__ __device__ constexpr int ch4p_singles(int PL) { return PL == 4 ? 69 : CH4_RECS; }
__host__ __device__ constexpr int ch4p_pair_levels(int PL) { return PL == 4 ? 3 : PL; }
__host__ __device__ constexpr int colhist4q_bytes(int T, int r, int PL) {
    const int ncp = colhist4p_ncolp(T, r);
    return (ch4p_singles(PL) * ncp + ch4p_recs(ch4p_pair_levels(PL)) * (ncp / 2)) * 4;
}

// level-2 word of column c for record p2 from its four level-3 words (PL = 4)
__device__ __forceinline__ uint32_t ch4_l2_from_l3(const uint32_t *rec, int NCP, int p2, int c) {
    const uint32_t *q = rec + (5 + 4 * p2) * NCP + c;
    return __dp4a(q[0], 0x01010101u, 0u) | (__dp4a(q[NCP], 0x01010101u, 0u) << 8) |
           (__dp4a(q[2 * NCP], 0x01010101u, 0u) << 16) | (__dp4a(q[3 * NCP], 0x01010101u, 0u) << 24);
}

// record updates for the PL = 4 layout: byte read-modify-writes (builds)
// and shared-memory atomics (row updates)
__device__ __forceinline__ void ch4q_bump(uint8_t *recb, int NCOL, int c, unsigned v, int d) {
    recb[(0 * NCOL + c) * 4 + (v >> 6)] += d;
    recb[((1 + (v >> 6)) * NCOL + c) * 4 + ((v >> 4) & 3)] += d;
    recb[((5 + (v >> 2)) * NCOL + c) * 4 + (v & 3)] += d;
}
__device__ __forceinline__ void ch4q_bump_upd(uint8_t *recb, int NCOL, int c, unsigned v, int d) {
    uint32_t *rw = reinterpret_cast<uint32_t *>(recb);
    const unsigned one = (unsigned)d;
    atomicAdd(rw + (0 * NCOL + c), one << (8 * (v >> 6)));
    atomicAdd(rw + ((1 + (v >> 6)) * NCOL + c), one << (8 * ((v >> 4) & 3)));
    atomicAdd(rw + ((5 + (v >> 2)) * NCOL + c), one << (8 * (v & 3)));
}

// window of one level from pair records (np = (n-1)/2 pairs from kp) plus
// the single column cs; GP pairs per carry-free group, runtime tail
template <int GP>
__device__ __forceinline__ void ch4p_gather(const uint32_t *pr, const uint32_t *sr, int kp, int cs, int np,
                                            uint32_t &w0, uint32_t &w1) {
    const uint32_t sv = sr[cs];
    w0 = __byte_perm(sv, 0, 0x4140);
    w1 = __byte_perm(sv, 0, 0x4342);
    const uint32_t *rp = pr + kp;
    const int full = np - np % GP;
    int j = 0;
    for (; j < full; j += GP) {
        uint32_t t = 0;
#pragma unroll
        for (int q = 0; q < GP; q += 2) t += rp[j + q] + (q + 1 < GP ? rp[j + q + 1] : 0u);
        w0 += __byte_perm(t, 0, 0x4140);
        w1 += __byte_perm(t, 0, 0x4342);
    }
    if (j < np) {
        uint32_t t = 0;
#pragma unroll
        for (int q = 0; q < GP - 1; ++q)
            if (j + q < np) t += rp[j + q];
        w0 += __byte_perm(t, 0, 0x4140);
        w1 += __byte_perm(t, 0, 0x4342);
    }
}


// the same with the single column's word supplied by the caller
template <int GP>
__device__ __forceinline__ void ch4p_gather_sv(const uint32_t *pr, uint32_t sv, int kp, int np, uint32_t &w0,
                                               uint32_t &w1) {
    w0 = __byte_perm(sv, 0, 0x4140);
    w1 = __byte_perm(sv, 0, 0x4342);
    const uint32_t *rp = pr + kp;
    const int full = np - np % GP;
    int j = 0;
    for (; j < full; j += GP) {
        uint32_t t = 0;
#pragma unroll
        for (int q = 0; q < GP; q += 2) t += rp[j + q] + (q + 1 < GP ? rp[j + q + 1] : 0u);
        w0 += __byte_perm(t, 0, 0x4140);
        w1 += __byte_perm(t, 0, 0x4342);
    }
    if (j < np) {
        uint32_t t = 0;
#pragma unroll
        for (int q = 0; q < GP - 1; ++q)
            if (j + q < np) t += rp[j + q];
        w0 += __byte_perm(t, 0, 0x4140);
        w1 += __byte_perm(t, 0, 0x4342);
    }
}

// the 4-level selection of the rank-k element (k updated to the rank within
// the selected value) from the records of the window starting at rp (= record
// row 0, thread column applied)
// the same with pair records for the upper PL levels (prs: [PR][NPR]);
// the thread's window is stripe columns tid .. tid+n-1
template <int G, int M, int PL>
__device__ __forceinline__ unsigned ch4_select_p(const uint32_t *rec, const uint32_t *prs, int NCP, int NPR, int tid,
                                                 int n, uint32_t &k) {
    if (PL == 0) {
        uint32_t w0, w1;
        ch4_gather<G, M>(rec + tid, n, w0, w1);
        const int d3 = ch4_descend(w0, w1, k);
        ch4_gather<G, M>(rec + (1 + d3) * NCP + tid, n, w0, w1);
        const int d2 = ch4_descend(w0, w1, k);
        const int p2 = d3 * 4 + d2;
        ch4_gather<G, M>(rec + (5 + p2) * NCP + tid, n, w0, w1);
        const int d1 = ch4_descend(w0, w1, k);
        const int p3 = p2 * 4 + d1;
        ch4_gather<G, M>(rec + (21 + p3) * NCP + tid, n, w0, w1);
        const int d0 = ch4_descend(w0, w1, k);
        return (unsigned)(p3 * 4 + d0);
    }
    constexpr int GP = G / 2;
    constexpr bool DL2 = PL == 4;
    constexpr int PLP = ch4p_pair_levels(PL), R3 = DL2 ? 5 : 21;
    const int kp = (tid + 1) >> 1, cs = (tid & 1) ? tid : tid + n - 1, np = (n - 1) >> 1;
    uint32_t w0, w1;
    ch4p_gather<GP>(prs, rec, kp, cs, np, w0, w1);
    const int d3 = ch4_descend(w0, w1, k);
    if (PLP >= 2)
        ch4p_gather<GP>(prs + (1 + d3) * NPR, rec + (1 + d3) * NCP, kp, cs, np, w0, w1);
    else
        ch4_gather<G, M>(rec + (1 + d3) * NCP + tid, n, w0, w1);
    const int d2 = ch4_descend(w0, w1, k);
    const int p2 = d3 * 4 + d2;
    if (DL2)
        ch4p_gather_sv<GP>(prs + (5 + p2) * NPR, ch4_l2_from_l3(rec, NCP, p2, cs), kp, np, w0, w1);
    else if (PLP >= 3)
        ch4p_gather<GP>(prs + (5 + p2) * NPR, rec + (5 + p2) * NCP, kp, cs, np, w0, w1);
    else
        ch4_gather<G, M>(rec + (5 + p2) * NCP + tid, n, w0, w1);
    const int d1 = ch4_descend(w0, w1, k);
    const int p3 = p2 * 4 + d1;
    ch4_gather<G, M>(rec + (R3 + p3) * NCP + tid, n, w0, w1);
    const int d0 = ch4_descend(w0, w1, k);
    return (unsigned)(p3 * 4 + d0);
}

template <int G, int M>
__device__ __forceinline__ unsigned ch4_select(const uint32_t *rp, int NCOL, int n, uint32_t &k) {
    uint32_t w0, w1;
    ch4_gather<G, M>(rp, n, w0, w1);
    const int d3 = ch4_descend(w0, w1, k);
    ch4_gather<G, M>(rp + (1 + d3) * NCOL, n, w0, w1);
    const int d2 = ch4_descend(w0, w1, k);
    const int p2 = d3 * 4 + d2;
    ch4_gather<G, M>(rp + (5 + p2) * NCOL, n, w0, w1);
    const int d1 = ch4_descend(w0, w1, k);
    const int p3 = p2 * 4 + d1;
    ch4_gather<G, M>(rp + (21 + p3) * NCOL, n, w0, w1);
    const int d0 = ch4_descend(w0, w1, k);
    return (unsigned)(p3 * 4 + d0);
}

// One downward sweep of a CTA stripe over rows [ya, yb]: the column records
// are built for row ya from the (clamped) spans, then moved down a row at a
// time; `key(v)` maps a pixel to its 8-bit record key (or -1: not counted),
// `pixel(y)` runs after each row's records are final.  Next-row pixels are
// prefetched a row ahead so their latency hides behind the gathers.
// PL > 0: also pair records prs [ch4p_recs(PL)][NCP/2] for the upper PL
// levels (rec row stride NCP even, pad column zero); updated with
// shared-memory atomics.
struct Ch4NoExtra {
    __device__ void operator()(int, unsigned, int) const {}
};

// extra(c, v, d): optional additional per-pixel record maintenance
// (called for every pixel entering (+1) / leaving (-1) column c)
template <int T, int PL = 0, typename P, typename Key, typename Pixel, typename Extra = Ch4NoExtra>
__device__ __forceinline__ void ch4_sweep(const SlabParams &p, const P *src, uint32_t *rec, int NCOL, int X0,
                                          int ya, int yb, Key key, Pixel pixel, uint32_t *prs = nullptr,
                                          int NCP = 0, Extra extra = Extra()) {
    const int tid = threadIdx.x;
    const int r = p.radius, H = p.H, W = p.W;
    const int RS = PL > 0 ? NCP : ch4_stride(NCOL);  // record row stride
    const int NPR = RS / 2;
    constexpr bool DL2 = PL == 4;  // no level-2 singles (ch4p_singles)
    constexpr int PLP = ch4p_pair_levels(PL);
    uint8_t *recb = reinterpret_cast<uint8_t *>(rec);
    auto pbump = [&](int c, unsigned v, int d) {
        const int kk = c >> 1;
        const unsigned one = (unsigned)d;
        atomicAdd(prs + kk, one << (8 * (v >> 6)));
        if (PLP >= 2) atomicAdd(prs + (1 + (v >> 6)) * NPR + kk, one << (8 * ((v >> 4) & 3)));
        if (PLP >= 3) atomicAdd(prs + (5 + (v >> 4)) * NPR + kk, one << (8 * ((v >> 2) & 3)));
    };
    auto bump2 = [&](int c, unsigned vo, unsigned vi) {
        extra(c, vo, -1);
        extra(c, vi, 1);
        const int ko = key(vo), ki = key(vi);  // (ko == ki cancels: no data-dependent branch)
        if (ko >= 0) {
            if (DL2)
                ch4q_bump_upd(recb, RS, c, (unsigned)ko, -1);
            else
                ch4_bump_upd(recb, RS, c, (unsigned)ko, -1);
            if (PL > 0) pbump(c, (unsigned)ko, -1);
        }
        if (ki >= 0) {
            if (DL2)
                ch4q_bump_upd(recb, RS, c, (unsigned)ki, 1);
            else
                ch4_bump_upd(recb, RS, c, (unsigned)ki, 1);
            if (PL > 0) pbump(c, (unsigned)ki, 1);
        }
    };
    __syncthreads();  // previous users of rec are done
    for (int i = tid; i < ch4p_singles(PL) * RS; i += T) rec[i] = 0;
    __syncthreads();
    for (int c = tid; c < NCOL; c += T) {
        const int gx = clampi(X0 - r + c, 0, W - 1);
        for (int j = -r; j <= r; ++j) {
            const unsigned v = src_row(p, src, clampi(ya + j, 0, H - 1))[gx];
            extra(c, v, 1);
            const int kv = key(v);
            if (kv >= 0) {
                if (DL2)
                    ch4q_bump(recb, RS, c, (unsigned)kv, 1);
                else
                    ch4_bump(recb, RS, c, (unsigned)kv, 1);
            }
        }
    }
    __syncthreads();
    if (PL > 0) {
        for (int i = tid; i < ch4p_recs(PLP) * NPR; i += T) {
            const int row = i / NPR, kk = i - row * NPR;
            if (DL2 && row >= 5)
                prs[i] = ch4_l2_from_l3(rec, RS, row - 5, 2 * kk) + ch4_l2_from_l3(rec, RS, row - 5, 2 * kk + 1);
            else
                prs[i] = rec[row * RS + 2 * kk] + rec[row * RS + 2 * kk + 1];
        }
        __syncthreads();
    }
    constexpr int CH_PF = 2;
    int gxs[CH_PF];
#pragma unroll
    for (int u = 0; u < CH_PF; ++u) gxs[u] = clampi(X0 - r + min(tid + u * T, NCOL - 1), 0, W - 1);
    unsigned pvo[CH_PF], pvi[CH_PF];
    auto prefetch = [&](int yn) {
        const P *ro = src_row(p, src, clampi(yn - r - 1, 0, H - 1));
        const P *ri = src_row(p, src, clampi(yn + r, 0, H - 1));
#pragma unroll
        for (int u = 0; u < CH_PF; ++u) {
            pvo[u] = __ldg(ro + gxs[u]);
            pvi[u] = __ldg(ri + gxs[u]);
        }
    };
    if (ya < yb) prefetch(ya + 1);
    for (int y = ya; y <= yb; ++y) {
        if (y > ya) {
            __syncthreads();  // previous row's gathers done
#pragma unroll
            for (int u = 0; u < CH_PF; ++u) {
                const int c = tid + u * T;
                if (c < NCOL) bump2(c, pvo[u], pvi[u]);
            }
            if (NCOL > CH_PF * T) {  // narrow CTA, wide halo: the rest without prefetch
                const P *ro = src_row(p, src, clampi(y - r - 1, 0, H - 1));
                const P *ri = src_row(p, src, clampi(y + r, 0, H - 1));
                for (int c = tid + CH_PF * T; c < NCOL; c += T) {
                    const int gx = clampi(X0 - r + c, 0, W - 1);
                    const unsigned vo = __ldg(ro + gx), vi = __ldg(ri + gx);
                    if (vo != vi) bump2(c, vo, vi);
                }
            }
            if (y < yb) prefetch(y + 1);
            __syncthreads();
        }
        pixel(y);
    }
}

// STREAM: the streaming host path's instantiation (row waits / chunk
// signals); the plain one has no hooks (they cost ~2% here when inlined).
// NF > 0: the window side as a compile-time constant (fully unrolled gathers)
template <int T, int G, int M, bool STREAM, int NF = 0>
__global__ void __launch_bounds__(T) k_colhist4_u8(SlabParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    const int r = NF ? NF / 2 : p.radius, W = p.W, n = NF ? NF : 2 * r + 1;
    const int NCOL = T + 2 * r, RS = ch4_stride(NCOL);
    uint32_t *rec = reinterpret_cast<uint32_t *>(smem_raw);  // [85][RS]
    const int X0 = blockIdx.x * T;
    const int y0 = p.row_begin + blockIdx.y * p.rows_per_cta;
    if (y0 >= p.row_end) return;  // CTA-uniform (barriers below)
    const int y1 = min(y0 + p.rows_per_cta, p.row_end);
    const uint8_t *src = static_cast<const uint8_t *>(p.src) + blockIdx.z * p.src_img_stride;
    uint8_t *dst = static_cast<uint8_t *>(p.dst) + blockIdx.z * p.dst_img_stride;
    const uint8_t *lut = static_cast<const uint8_t *>(p.lut);
    const int x = X0 + tid;
    if (STREAM) stream_wait_rows(p, y1 + r);
    auto key = [](unsigned v) { return (int)v; };
    auto pix = [&](int y) {
        uint32_t k = p.rank;
        const unsigned v = ch4_select<G, M>(rec + tid, RS, n, k);
        if (x < W) dst[(int64_t)(y - p.row_begin) * p.dst_pitch + x] = lut ? __ldg(lut + v) : (uint8_t)v;
    };
    ch4_sweep<T, 0, uint8_t>(p, src, rec, NCOL, X0, y0, y1 - 1, key, pix);
    if (STREAM) stream_signal(p, y0, y1, X0, X0 + T);
}

// ---------------------------------------------------------------------------
// 16-bit images whose median high bytes are locally few (compact data, e.g.
// config 4): two phases over the CTA's tile, each a ch4_sweep.
//   A: records keyed by the high byte -> every pixel's high byte H and its
//      rank k within H (H to a u8 scratch plane, k to dst); the set of H
//      values used by the tile and their first / last row are collected.
//   B: once per H used (ascending): records keyed by the low byte of the
//      pixels whose high byte is H, swept over that H's row range; pixels
//      with this H select their low byte with rank k.
// Exact for any image; the cost grows with the number of distinct H per
// tile, so the host only picks it when the sampled high-byte spread is small.
// WK (compact data): a first sweep keyed by a guessed high byte H0 (the
// median high byte of a sample of the tile): records of the low bytes of
// the pixels with high byte H0 plus, per column, the counts below / equal
// to / above H0 (one word).  A pixel whose rank falls inside the H0 bin is
// resolved right there (5 gathers instead of phase A + phase B's 8); the
// rest (marked in the high-byte plane) go through phases A and B, which
// then skip H0.
template <int T, int G, int M, int PL, int NF = 0>
__global__ void __launch_bounds__(T) k_colhist16_u16(SlabParams p, uint8_t *__restrict__ hplane, int wk_mode) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (gate_off(p)) return;
    const bool WK = wk_mode == WK_FROM_SPREAD ? !spread_is_wide(p) : wk_mode != 0;
    const int tid = threadIdx.x;
    const int r = NF ? NF / 2 : p.radius, W = p.W, n = NF ? NF : 2 * r + 1;
    const int NCOL = T + 2 * r;
    const int NCP = PL > 0 ? colhist4p_ncolp(T, r) : ch4_stride(NCOL);  // record row stride
    const int NPR = NCP / 2;
    uint32_t *rec = reinterpret_cast<uint32_t *>(smem_raw);  // [85 or 69][NCP] singles
    uint32_t *prs = rec + ch4p_singles(PL) * NCP;             // [PR][NPR] (PL > 0)
    uint32_t *rec3 = prs + (PL > 0 ? ch4p_recs(ch4p_pair_levels(PL)) * NPR : 0);  // [NCP] below/equal/above H0 (WK)
    int *hfirst = reinterpret_cast<int *>(rec3 + NCP);             // [256]
    int *hlast = hfirst + 256;                                      // [256]
    int *flags = hlast + 256;                                       // [0]: H0, [1]: any miss
    const int X0 = blockIdx.x * T;
    const int y0 = p.row_begin + blockIdx.y * p.rows_per_cta;
    if (y0 >= p.row_end) return;  // CTA-uniform (barriers below)
    const int y1 = min(y0 + p.rows_per_cta, p.row_end);
    if (p.todo && !todo_any(p, X0, T, y0, y1)) return;  // (CTA-uniform) nothing left over in this tile
    const uint16_t *src = static_cast<const uint16_t *>(p.src) + blockIdx.z * p.src_img_stride;
    uint16_t *dst = static_cast<uint16_t *>(p.dst) + blockIdx.z * p.dst_img_stride;
    const uint16_t *lut = static_cast<const uint16_t *>(p.lut);
    const int64_t hp_img = (int64_t)(p.row_end - p.row_begin) * p.W;
    uint8_t *hpl = hplane + blockIdx.z * hp_img;
    const int x = X0 + tid;
    stream_wait_rows(p, y1 + r);
    for (int i = tid; i < 256; i += T) {
        hfirst[i] = 1 << 30;
        hlast[i] = -1;
    }
    int H0 = -1;
    if (WK) {
        // H0: median high byte of 256 pixels sampled over the tile
        if (tid == 0) flags[1] = 0;
        for (int i = tid; i < 256; i += T) hlast[i] = 0;
        __syncthreads();
        for (int i = tid; i < 256; i += T) {
            const int yy = y0 + (int)(((int64_t)i * 97) % (y1 - y0));
            const int xx = min(X0 + (int)(((int64_t)i * 61) % T), W - 1);
            atomicAdd(&hlast[src_row(p, src, yy)[xx] >> 8], 1);  // hlast as a scratch histogram
        }
        __syncthreads();
        if (tid == 0) {
            int acc = 0, h = 0;
            for (; h < 255; ++h) {
                acc += hlast[h];
                if (2 * acc >= 256) break;
            }
            flags[0] = h;
        }
        __syncthreads();
        H0 = flags[0];
        for (int i = tid; i < 256; i += T) hlast[i] = -1;
        for (int i = tid; i < NCP; i += T) rec3[i] = 0;
        const int h0 = H0;
        ch4_sweep<T, PL, uint16_t>(
            p, src, rec, NCOL, X0, y0, y1 - 1,
            [h0](unsigned v) { return (int)(v >> 8) == h0 ? (int)(v & 255) : -1; },
            [&](int y) {
                uint32_t w0, w1;
                ch4_gather<G, M>(rec3 + tid, n, w0, w1);
                const uint32_t below = w0 & 0xffffu, eq = w0 >> 16;
                uint32_t k = p.rank;
                const bool hit = k > below && k <= below + eq;
                unsigned lo = 0;
                if (hit) {
                    k -= below;
                    lo = ch4_select_p<G, M, PL>(rec, prs, NCP, NPR, tid, n, k);
                }
                if (x < W) {
                    const int64_t o = (int64_t)(y - p.row_begin) * W + x;
                    if (hit) {
                        const unsigned v = ((unsigned)h0 << 8) | lo;
                        dst[(int64_t)(y - p.row_begin) * p.dst_pitch + x] = lut ? __ldg(lut + v) : (uint16_t)v;
                        hpl[o] = (uint8_t)h0;
                    } else {
                        hpl[o] = (uint8_t)(h0 ^ 1);  // any value != H0 marks a miss
                        flags[1] = 1;
                    }
                }
            },
            prs, NCP,
            [rec3, h0](int c, unsigned v, int d) {
                // one shared-memory atomic add (see ch4_bump_upd)
                const int hb = (int)(v >> 8);
                atomicAdd(rec3 + c, (unsigned)d << (8 * (hb < h0 ? 0 : (hb == h0 ? 1 : 2))));
            });
        __syncthreads();
        if (flags[1] == 0) {  // every pixel of the tile resolved
            stream_signal(p, y0, y1, X0, X0 + T);
            return;
        }
    }
    // phase A: high byte and rank within it (WK: only the marked pixels)
    ch4_sweep<T, PL, uint16_t>(
        p, src, rec, NCOL, X0, y0, y1 - 1, [](unsigned v) { return (int)(v >> 8); },
        [&](int y) {
            if (WK && (x >= W || hpl[(int64_t)(y - p.row_begin) * W + x] == H0)) return;
            uint32_t k = p.rank;
            const unsigned hb = ch4_select_p<G, M, PL>(rec, prs, NCP, NPR, tid, n, k);
            if (x < W) {
                const int64_t o = (int64_t)(y - p.row_begin) * W + x;
                hpl[o] = (uint8_t)hb;
                dst[(int64_t)(y - p.row_begin) * p.dst_pitch + x] = (uint16_t)k;
                // rows ascend and every writer of a row stores the same y:
                // plain stores (no atomics) are race-free in effect
                if (hfirst[hb] > y) hfirst[hb] = y;
                hlast[hb] = y;
            }
        },
        prs, NCP);
    __syncthreads();
    // phase B: one sweep per high byte used by the tile (WK: H0 is done)
    for (int hb = 0; hb < 256; ++hb) {
        const int ya = hfirst[hb], yb = hlast[hb];  // CTA-uniform
        if (yb < 0 || (WK && hb == H0)) continue;
        ch4_sweep<T, PL, uint16_t>(
            p, src, rec, NCOL, X0, ya, yb,
            [hb](unsigned v) { return (int)(v >> 8) == hb ? (int)(v & 255) : -1; },
            [&](int y) {
                if (x >= W) return;
                const int64_t o = (int64_t)(y - p.row_begin) * W + x;
                if (hpl[o] != hb) return;
                uint16_t *d = dst + (int64_t)(y - p.row_begin) * p.dst_pitch + x;
                uint32_t k = *d;
                const unsigned lo = ch4_select_p<G, M, PL>(rec, prs, NCP, NPR, tid, n, k);
                const unsigned v = ((unsigned)hb << 8) | lo;
                *d = lut ? __ldg(lut + v) : (uint16_t)v;
            },
            prs, NCP);
    }
    stream_signal(p, y0, y1, X0, X0 + T);
}

}  // namespace mtb

namespace mtb {

// ---------------------------------------------------------------------------
// 16-bit, widely spread data (e.g. uniform noise): one sweep.  The high byte
// H and the rank k within it come from radix-4 column records keyed by the
// high byte (as in phase A of k_colhist16_u16, gathered per pixel); the low
// byte from per-column SORTED arrays of the stripe kept in the same shared
// memory (one delete + one insert per column and row): the window values
// with high byte H are one run per window column, starting at
// lower_bound(256H) (2r+1 interleaved branchless searches), counted per
// bits 4..7 and then per bits 0..3 of the selected 16-value sub-run.
// Replaces the per-thread high-byte counters of k_vert2_u16 (544 B per
// thread) by shared records (340 B per column): more resident threads and
// no read-modify-write chains in the high-byte step.
constexpr int CH16S_CMAX = 24;  // low-byte candidates kept per thread (k_colhist16s_u16)

template <int T, int G, int M, int NF = 0>
__global__ void __launch_bounds__(T) k_colhist16s_u16(SlabParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (gate_off(p)) return;
    const int tid = threadIdx.x;
    const int r = NF ? NF / 2 : p.radius, H = p.H, W = p.W, n = NF ? NF : 2 * r + 1;
    const int NCOL = T + 2 * r, RS = ch4_stride(NCOL);
    uint32_t *rec = reinterpret_cast<uint32_t *>(smem_raw);                  // [85][RS]
    uint16_t *sc = reinterpret_cast<uint16_t *>(rec + CH4_RECS * RS);        // [16][T]
    uint8_t *rpos = reinterpret_cast<uint8_t *>(sc + 16 * T);                // [n][T]
    uint16_t *scol = reinterpret_cast<uint16_t *>(rpos + ((n * T + 15) & ~15));  // [NCOL][n]
    uint8_t *cand = reinterpret_cast<uint8_t *>(scol + ((NCOL * n + 7) & ~7));     // [CH16S_CMAX][T]
    uint8_t *recb = reinterpret_cast<uint8_t *>(rec);
    const int X0 = blockIdx.x * T;
    const int y0 = p.row_begin + blockIdx.y * p.rows_per_cta;
    if (y0 >= p.row_end) return;  // CTA-uniform (barriers below)
    const int y1 = min(y0 + p.rows_per_cta, p.row_end);
    const uint16_t *src = static_cast<const uint16_t *>(p.src) + blockIdx.z * p.src_img_stride;
    uint16_t *dst = static_cast<uint16_t *>(p.dst) + blockIdx.z * p.dst_img_stride;
    const uint16_t *lut = static_cast<const uint16_t *>(p.lut);
    const int x = X0 + tid;
    const uint16_t *wcol = scol + tid * n;  // window column j of this thread = stripe column tid + j
    stream_wait_rows(p, y1 + r);

    // records and sorted columns for row y0
    for (int i = tid; i < CH4_RECS * RS; i += T) rec[i] = 0;
    __syncthreads();
    for (int c = tid; c < NCOL; c += T) {
        const int gx = clampi(X0 - r + c, 0, W - 1);
        uint16_t *a = scol + c * n;
        for (int j = 0; j < n; ++j) {
            const uint16_t v = __ldg(src_row(p, src, clampi(y0 - r + j, 0, H - 1)) + gx);
            ch4_bump(recb, RS, c, v >> 8, 1);
            int i = j;
            while (i > 0 && a[i - 1] > v) {
                a[i] = a[i - 1];
                --i;
            }
            a[i] = v;
        }
    }
    __syncthreads();
    for (int y = y0; y < y1; ++y) {
        if (y > y0) {
            const int yo = clampi(y - r - 1, 0, H - 1), yi = clampi(y + r, 0, H - 1);
            if (yo != yi) {
                __syncthreads();  // previous row's reads done
                const uint16_t *ro = src_row(p, src, yo), *ri = src_row(p, src, yi);
                for (int c = tid; c < NCOL; c += T) {
                    const int gx = clampi(X0 - r + c, 0, W - 1);
                    const unsigned vo = __ldg(ro + gx), vi = __ldg(ri + gx);
                    if (vo == vi) continue;
                    if ((vo >> 8) != (vi >> 8)) {
                        ch4_bump_upd(recb, RS, c, vo >> 8, -1);
                        ch4_bump_upd(recb, RS, c, vi >> 8, 1);
                    }
                    uint16_t *a = scol + c * n;
                    const uint16_t *const aa[2] = {a, a};
                    const unsigned vv[2] = {vo, vi};
                    int pos[2];
                    lower_bound_multi<2>(aa, n, vv, pos);
                    const int io = pos[0], ii = pos[1];  // a[io] == vo
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
        // high byte and rank within it
        uint32_t k = p.rank;
        const unsigned hb = ch4_select<G, M>(rec + tid, RS, n, k);
        // low byte: runs of [256H, 256H+256) in the window columns.  The
        // low bytes found are collected (a handful on spread data: ~n^2/256
        // per bin) and the k-th smallest is counted out of them; a bin with
        // more than CH16S_CMAX values takes the two counting passes below.
        const unsigned vb = hb << 8, ve = vb + 256;
        // Each window column's run of high byte H is read off the column's
        // high-byte records, no search: its start is the column's count of
        // high bytes below H (the bytes below H's digit in the four record
        // words on H's path) and its length the count of H (the last
        // word's byte) -- four independent loads per column instead of a
        // dependent binary search plus a scan to the run's end.
        int cnt = 0;
        {
            const unsigned d3 = hb >> 6, d2 = (hb >> 4) & 3, d1 = (hb >> 2) & 3, d0 = hb & 3;
            const uint32_t *r0 = rec + tid, *r1 = rec + (1 + d3) * RS + tid;
            const uint32_t *r2 = rec + (5 + (hb >> 4)) * RS + tid, *r3 = rec + (21 + (hb >> 2)) * RS + tid;
            auto below = [](uint32_t w, unsigned d) {  // sum of the bytes below byte d (<= n < 256)
                const uint32_t m = d ? (0xffffffffu >> (32 - 8 * d)) : 0u;
                return ((w & m) * 0x01010101u) >> 24;
            };
            for (int j = 0; j < n; ++j) {
                const uint32_t w3 = r3[j];
                const int e0 = (int)(below(r0[j], d3) + below(r1[j], d2) + below(r2[j], d1) + below(w3, d0));
                const int ne = (int)((w3 >> (8 * d0)) & 0xffu);
                rpos[j * T + tid] = (uint8_t)e0;
                const uint16_t *a = wcol + j * n;
                for (int e = e0; e < e0 + ne; ++e) {
                    if (cnt < CH16S_CMAX) cand[cnt * T + tid] = (uint8_t)a[e];
                    ++cnt;
                }
            }
        }
        if (cnt <= CH16S_CMAX) {
            // k-th smallest (1-based) of the cnt candidates: the value with
            // fewer than k candidates below it and at least k at or below
            unsigned lo = 0;
            for (int i = 0; i < cnt; ++i) {
                const unsigned ci = cand[i * T + tid];
                uint32_t below = 0, atmost = 0;
                for (int jj = 0; jj < cnt; ++jj) {
                    const unsigned cj = cand[jj * T + tid];
                    below += cj < ci ? 1u : 0u;
                    atmost += cj <= ci ? 1u : 0u;
                }
                if (below < k && k <= atmost) {
                    lo = ci;
                    break;
                }
            }
            const unsigned v = vb | lo;
            if (x < W) dst[(int64_t)(y - p.row_begin) * p.dst_pitch + x] = lut ? __ldg(lut + v) : (uint16_t)v;
            continue;
        }
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
        uint32_t acc = 0;
        int lb = 0;
        for (; lb < 15; ++lb) {
            const uint32_t c = sc[lb * T + tid];
            if (acc + c >= k) break;
            acc += c;
        }
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
            if (acc + c >= k) break;
            acc += c;
        }
        const unsigned v = vb | (unsigned)lo;
        if (x < W) dst[(int64_t)(y - p.row_begin) * p.dst_pitch + x] = lut ? __ldg(lut + v) : (uint16_t)v;
    }
    stream_signal(p, y0, y1, X0, X0 + T);
}

}  // namespace mtb

namespace mtb {

// ---------------------------------------------------------------------------
// Radix-4 records with PAIR records for the upper levels (8-bit, mid r).
// The gathers of k_colhist4_u8 are bound by shared-memory wavefronts (one
// word per window column and level).  Here the CTA also keeps, for levels
// 0-2 (21 record rows), the sums of column pairs (2k, 2k+1): a window of n
// (odd) columns is (n-1)/2 pairs plus one single column -- the single is
// the first column when the window starts odd, the last when it starts
// even, so the pair run always starts at (s+1)/2 -- about half the words
// for those levels (2.5n words per pixel instead of 4n).  Pair counts are
// at most 2n, so G/2 pairs per carry-free group.  Row updates add the
// pair changes with shared-memory atomics (adjacent columns belong to
// adjacent threads); counts never go below zero, so a per-byte decrement
// never borrows across bytes.
// PL = 4: three pair levels, and NO level-2 single records -- the single
// column of a level-2 pair gather derives its word from its four level-3
// words (IDP4A each), which frees 64 B per stripe column: three pair levels
// then fit two 256-thread CTAs per SM up to r = 32 (PL = 2 before), and a
// row update is 12 shared-memory atomics instead of 14.

// PX = uint16_t: the same kernel keyed by the coarse key of 16-bit pixels,
// min(v >> s, 255) -- the high byte, s = 8, unless the data leaves the top
// bits empty (key_shift) -- as the first pass of the 16-bit candidate-bucket
// path (kernels_lowsel16.cuh): instead of a result pixel it writes
// H << 16 | k' per pixel to a u32 plane (p.dst, pitch in words), H = the
// result's key, k' = the rank of the result among the window values with
// that key.
// MODE = 1 (PX = uint16_t, "window key"): compact 16-bit data as ONE 8-bit
// problem.  The CTA estimates the median V0 + 127 of its tile from 256 sampled
// pixels and keys every pixel by clamp(v - V0 + 1, 0, 255): 0 = below the
// 254-value window [V0, V0 + 253], 255 = above it, 1..254 exact.  A pixel whose
// rank lands on a key in 1..254 is resolved exactly (result V0 + key - 1); one
// that lands on 0 or 255 flags its 32 x todo_bh block in SlabParams::todo for
// the two-phase kernel (k_colhist16_u16, which then redoes the tiles holding
// flagged blocks).  With spread[2] == 0 (the sampled histogram is not peaked:
// few medians would land in the window) the CTA flags its whole tile and exits.
template <int T, int G, int M, int PL, bool STREAM, int NF = 0, typename PX = uint8_t, int MODE = 0>
__global__ void __launch_bounds__(T) k_colhist4p_u8(SlabParams p) {
    constexpr bool WK = MODE == 1;
    constexpr bool HI16 = sizeof(PX) == 2 && !WK;
    static_assert(!WK || (sizeof(PX) == 2 && T == 256 && !STREAM), "window-key mode: 16-bit pixels, one sample per thread");
    constexpr int GP = G / 2;
    constexpr bool DL2 = PL == 4;           // level-2 singles derived from level 3
    constexpr int PLP = DL2 ? 3 : PL;        // pair levels
    constexpr int PR = ch4p_recs(PLP);
    constexpr int NS = ch4p_singles(PL);     // single record rows
    constexpr int R3 = DL2 ? 5 : 21;         // first level-3 single row
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    const int r = NF ? NF / 2 : p.radius, H = p.H, W = p.W, n = NF ? NF : 2 * r + 1;
    const int NCOL = T + 2 * r, NCP = colhist4p_ncolp(T, r), NPR = NCP / 2;
    uint32_t *rec = reinterpret_cast<uint32_t *>(smem_raw);  // [NS][NCP] singles
    uint32_t *prs = rec + NS * NCP;                           // [PR][NPR] pairs
    const int X0 = blockIdx.x * T;
    const int y0 = p.row_begin + blockIdx.y * p.rows_per_cta;
    if (y0 >= p.row_end) return;  // CTA-uniform (barriers below)
    if ((HI16 || WK) && gate_off(p)) return;
    const int ks = HI16 ? key_shift(p) : 0;
    const int y1 = min(y0 + p.rows_per_cta, p.row_end);
    if (STREAM) stream_wait_rows(p, y1 + r);
    const PX *src = static_cast<const PX *>(p.src) + blockIdx.z * p.src_img_stride;
    uint8_t *dst = static_cast<uint8_t *>(p.dst) + (HI16 ? 4 : (WK ? 2 : 1)) * blockIdx.z * p.dst_img_stride;
    const uint8_t *lut = static_cast<const uint8_t *>(p.lut);
    const int x = X0 + tid;
    unsigned V0 = 0;  // window-key mode: first value of the tile's window
    unsigned char *todo = nullptr;
    if (WK) {
        todo = p.todo + (size_t)blockIdx.z * p.todo_nbx * p.todo_nby;
        if (p.spread && reinterpret_cast<const volatile int *>(p.spread)[2] == 0) {
            // not peaked: the whole tile goes to the two-phase kernel
            const int bx0 = X0 >> 5, nx = min((X0 + T + 31) >> 5, p.todo_nbx) - bx0;
            const int by0 = (y0 - p.row_begin) / p.todo_bh, ny = (y1 - p.row_begin + p.todo_bh - 1) / p.todo_bh - by0;
            for (int i = tid; i < nx * ny; i += T) todo[(size_t)(by0 + i / nx) * p.todo_nbx + bx0 + i % nx] = 1;
            return;
        }
        // the median of 256 pixels sampled over the tile, by counting ranks
        uint32_t *smp = reinterpret_cast<uint32_t *>(smem_raw);
        const int yy = y0 + (int)(((int64_t)tid * 97) % (y1 - y0));
        const int xx = min(X0 + (int)(((int64_t)tid * 61) % T), W - 1);
        const uint32_t mine = src_row(p, src, yy)[xx];
        smp[tid] = mine;
        __syncthreads();
        int rk = 0;
        for (int j = 0; j < T; ++j) {
            const uint32_t o = smp[j];
            rk += (o < mine || (o == mine && j < tid)) ? 1 : 0;
        }
        if (rk == T / 2) smp[T] = mine;
        __syncthreads();
        V0 = (unsigned)clampi((int)smp[T] - 127, 0, 65535 - 253);
        __syncthreads();  // (the records below reuse the sample's memory)
    }
    // the record key of a pixel: the pixel (8-bit), its coarse key min(v >> ks, 255) (16-bit,
    // candidate-bucket path), or its place in the tile's window (16-bit, window-key mode)
    auto keyof = [&](unsigned v) -> unsigned {
        if (WK) return v < V0 ? 0u : min(v - V0 + 1u, 255u);
        return HI16 ? min(v >> ks, 255u) : v;
    };
    // single-record updates (one atomic per level kept; the word is the
    // thread's own column, so there is no contention)
    auto sbump_upper = [&](int c, unsigned v, int d) {  // levels 1-3
        const unsigned one = (unsigned)d;
        atomicAdd(rec + ((1 + (v >> 6)) * NCP + c), one << (8 * ((v >> 4) & 3)));
        if (!DL2) atomicAdd(rec + ((5 + (v >> 4)) * NCP + c), one << (8 * ((v >> 2) & 3)));
        atomicAdd(rec + ((R3 + (v >> 2)) * NCP + c), one << (8 * (v & 3)));
    };
    auto sbump = [&](int c, unsigned v, int d) {
        atomicAdd(rec + (0 * NCP + c), (unsigned)d << (8 * (v >> 6)));
        sbump_upper(c, v, d);
    };

    for (int i = tid; i < NS * NCP; i += T) rec[i] = 0;
    __syncthreads();
    for (int c = tid; c < NCOL; c += T) {
        const int gx = clampi(X0 - r + c, 0, W - 1);
        // (atomic adds here too: measured r = 15 0.358 -> 0.319 ms, r = 31
        // 0.595 -> 0.530 against byte read-modify-writes)
        for (int j = -r; j <= r; ++j) sbump(c, keyof(__ldg(src_row(p, src, clampi(y0 + j, 0, H - 1)) + gx)), 1);
    }
    __syncthreads();
    // level-2 word of column c for record p2, from its four level-3 words
    auto l2_from_l3 = [&](int p2, int c) -> uint32_t {
        const uint32_t *q = rec + (R3 + 4 * p2) * NCP + c;
        return __dp4a(q[0], 0x01010101u, 0u) | (__dp4a(q[NCP], 0x01010101u, 0u) << 8) |
               (__dp4a(q[2 * NCP], 0x01010101u, 0u) << 16) | (__dp4a(q[3 * NCP], 0x01010101u, 0u) << 24);
    };
    for (int i = tid; i < PR * NPR; i += T) {
        const int row = i / NPR, k = i - row * NPR;
        if (DL2 && row >= 5)
            prs[i] = l2_from_l3(row - 5, 2 * k) + l2_from_l3(row - 5, 2 * k + 1);
        else
            prs[i] = rec[row * NCP + 2 * k] + rec[row * NCP + 2 * k + 1];
    }
    // pair updates: levels 1-2 of value v, +-1 in the byte of the next digit
    auto pbump = [&](int c, unsigned v, int d) {
        const int k = c >> 1;
        const unsigned one = (unsigned)d;  // +1 or 0xffffffff (-1)
        if (PLP >= 2) atomicAdd(prs + (1 + (v >> 6)) * NPR + k, one << (8 * ((v >> 4) & 3)));
        if (PLP >= 3) atomicAdd(prs + (5 + (v >> 4)) * NPR + k, one << (8 * ((v >> 2) & 3)));
    };
    // one column's row step (vo leaves, vi enters).  Level 0 is one record
    // per column (and per pair): its two changes go in as ONE atomic add of
    // the combined delta -- exact in modular arithmetic, since every byte's
    // final count is in [0, 255].
    auto move = [&](int c, unsigned vo, unsigned vi) {
        const unsigned d0 = (1u << (8 * (vi >> 6))) - (1u << (8 * (vo >> 6)));
        atomicAdd(rec + c, d0);
        atomicAdd(prs + (c >> 1), d0);
        sbump_upper(c, vo, -1);
        sbump_upper(c, vi, 1);
        pbump(c, vo, -1);
        pbump(c, vi, 1);
    };
    constexpr int CH_PF = 2;
    int gxs[CH_PF];
#pragma unroll
    for (int u = 0; u < CH_PF; ++u) gxs[u] = clampi(X0 - r + min(tid + u * T, NCOL - 1), 0, W - 1);
    unsigned pvo[CH_PF], pvi[CH_PF];
    auto prefetch = [&](int yn) {
        const PX *ro = src_row(p, src, clampi(yn - r - 1, 0, H - 1));
        const PX *ri = src_row(p, src, clampi(yn + r, 0, H - 1));
#pragma unroll
        for (int u = 0; u < CH_PF; ++u) {
            pvo[u] = keyof(__ldg(ro + gxs[u]));
            pvi[u] = keyof(__ldg(ri + gxs[u]));
        }
    };
    if (y0 + 1 < y1) prefetch(y0 + 1);
    // the thread's window: stripe columns tid .. tid+n-1
    const int kp = (tid + 1) >> 1, cs = (tid & 1) ? tid : tid + n - 1, np = (n - 1) >> 1;
    for (int y = y0; y < y1; ++y) {
        if (y > y0) {
            __syncthreads();  // previous row's gathers done (also orders the pair init)
#pragma unroll
            for (int u = 0; u < CH_PF; ++u) {
                const int c = tid + u * T;
                if (c < NCOL) move(c, pvo[u], pvi[u]);  // (vo == vi cancels: no data-dependent branch)
            }
            if (NCOL > CH_PF * T) {
                const PX *ro = src_row(p, src, clampi(y - r - 1, 0, H - 1));
                const PX *ri = src_row(p, src, clampi(y + r, 0, H - 1));
                for (int c = tid + CH_PF * T; c < NCOL; c += T) {
                    const int gx = clampi(X0 - r + c, 0, W - 1);
                    const unsigned vo = keyof(__ldg(ro + gx)), vi = keyof(__ldg(ri + gx));
                    if (vo == vi) continue;
                    move(c, vo, vi);
                }
            }
            if (y + 1 < y1) prefetch(y + 1);
        }
        __syncthreads();
        uint32_t k = p.rank, w0, w1;
        ch4p_gather<GP>(prs, rec, kp, cs, np, w0, w1);
        const int d3 = ch4_descend(w0, w1, k);
        if (PLP >= 2)
            ch4p_gather<GP>(prs + (1 + d3) * NPR, rec + (1 + d3) * NCP, kp, cs, np, w0, w1);
        else
            ch4_gather<G, M>(rec + (1 + d3) * NCP + tid, n, w0, w1);
        const int d2 = ch4_descend(w0, w1, k);
        const int p2 = d3 * 4 + d2;
        if (DL2)
            ch4p_gather_sv<GP>(prs + (5 + p2) * NPR, l2_from_l3(p2, cs), kp, np, w0, w1);
        else if (PLP >= 3)
            ch4p_gather<GP>(prs + (5 + p2) * NPR, rec + (5 + p2) * NCP, kp, cs, np, w0, w1);
        else
            ch4_gather<G, M>(rec + (5 + p2) * NCP + tid, n, w0, w1);
        const int d1 = ch4_descend(w0, w1, k);
        const int p3 = p2 * 4 + d1;
        ch4_gather<G, M>(rec + (R3 + p3) * NCP + tid, n, w0, w1);
        const int d0 = ch4_descend(w0, w1, k);
        const unsigned v = (unsigned)(p3 * 4 + d0);
        if (HI16) {
            if (x < W) reinterpret_cast<uint32_t *>(dst)[(int64_t)(y - p.row_begin) * p.dst_pitch + x] = (v << 16) | k;
        } else if (WK) {
            if (x < W) {
                if (v >= 1u && v <= 254u) {
                    const unsigned val = V0 + v - 1u;
                    const uint16_t *lut16 = reinterpret_cast<const uint16_t *>(lut);
                    reinterpret_cast<uint16_t *>(dst)[(int64_t)(y - p.row_begin) * p.dst_pitch + x] =
                        lut16 ? __ldg(lut16 + val) : (uint16_t)val;
                } else {  // the rank lies outside the window: leave the block to the two-phase kernel
                    todo[(size_t)((y - p.row_begin) / p.todo_bh) * p.todo_nbx + (x >> 5)] = 1;
                }
            }
        } else {
            if (x < W) dst[(int64_t)(y - p.row_begin) * p.dst_pitch + x] = lut ? __ldg(lut + v) : (uint8_t)v;
        }
    }
    if (STREAM) stream_signal(p, y0, y1, X0, X0 + T);
}

}  // namespace mtb
