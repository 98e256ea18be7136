// kernels_colhist16c.cuh -- 16-bit rank filter for widely spread values
// (config 3: uniform 16-bit noise), "high byte by pair records, low byte
// by candidates".
//
// The window of n^2 values has, on spread data, only ~n^2/256 values whose
// high byte equals the result's (3.75 at r = 15).  The kernel therefore
//   1. selects the high byte H and the rank k' within it from radix-4
//      column records keyed by the high byte, with pair records for the
//      upper levels -- the 8-bit pair kernel's gathers (k_colhist4p_u8),
//      applied to the high byte;
//   2. collects the c_H window values with high byte H (c_H is the count
//      of H, known from step 1): every window column keeps its n values
//      SORTED (scol), so its values with high byte H are one run, starting
//      at the column's count of high bytes below H -- the bytes below H's
//      digits in the four record words on H's path, one IDP4A per word --
//      and as long as the count of H in the column (the last word's byte);
//   3. selects the k'-th smallest low byte of the candidates: up to 8 by a
//      sorting network in registers, more by two nibble counts (high nibble
//      over all candidates, then low nibble over those in the selected one).
// Bins with more than CMAX values (compact data forced onto this kernel)
// take two counting passes over the runs instead (u16 counters in shared
// memory).  Exact for any image.
//
// Compared with k_colhist16s_u16 (which it replaces for r <= 16 on spread
// data): pair records in step 1, one IDP4A per record word instead of a
// mask-and-multiply, no divergent candidate loop for the common run length
// 0/1, and the selection without an O(c^2) rank count.
//
// Reference semantics: the rank-k element of the replicate-clamped window
// (_kernels.py:229-253 extract_u on the 16-bit tree).
#pragma once
#include "common.cuh"
#include "kernels_colhist.cuh"

namespace mtb {

// bytes 0..d-1 set to 1: the IDP4A weight vector summing the counts below digit d
__device__ __forceinline__ uint32_t ch16c_below_w(unsigned d) {
    return d == 0 ? 0u : (d == 1 ? 0x1u : (d == 2 ? 0x101u : 0x10101u));
}

// 16 u8 counts (4 words) -> smallest bin b with cumsum >= k; k -= counts below b
__device__ __forceinline__ int ch16c_descend16(const uint32_t (&c)[4], uint32_t &k) {
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        w[2 * i] = __byte_perm(c[i], 0, 0x4140);
        w[2 * i + 1] = __byte_perm(c[i], 0, 0x4342);
    }
    return ct_descend(w, k);
}

// +1 in u8 count lane `b` (0..15) of 4 words (branch-free, predicated by `on`)
__device__ __forceinline__ void ch16c_count(uint32_t (&c)[4], unsigned b, bool on) {
    const uint32_t inc = on ? (1u << (8 * (b & 3))) : 0u;
    const unsigned q = b >> 2;
    c[0] += q == 0 ? inc : 0u;
    c[1] += q == 1 ? inc : 0u;
    c[2] += q == 2 ? inc : 0u;
    c[3] += q == 3 ? inc : 0u;
}

// shared memory: records + pairs, sorted spans, and per thread either the
// candidate bytes (fast path) or 16 u16 counters (crowded bins) -- a thread
// uses one or the other for a pixel, so they share the space
constexpr int ch16c_bytes(int T, int r, int PL, int CMAX) {
    return colhist4p_bytes(T, r, PL) + (((T + 2 * r) * (2 * r + 1) * 2 + 15) & ~15) +
           (CMAX > 32 ? CMAX : 32) * T;
}

// pair levels: the most that still fit three CTAs per SM (else two)
constexpr int ch16c_pair_levels(int T, int r, int CMAX) {
    return 3 * (ch16c_bytes(T, r, 3, CMAX) + 1024) <= 228 * 1024 ? 3
           : 3 * (ch16c_bytes(T, r, 2, CMAX) + 1024) <= 228 * 1024 ? 2 : 3;
}

template <int T, int G, int M, int PL, int CMAX, bool STREAM, int NF = 0>
__global__ void __launch_bounds__(T) k_colhist16c_u16(SlabParams p) {
    constexpr int GP = G / 2;
    constexpr int PR = ch4p_recs(PL);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (gate_off(p)) return;
    const int tid = threadIdx.x;
    const int r = NF ? NF / 2 : p.radius, H = p.H, W = p.W, n = NF ? NF : 2 * r + 1;
    const int NCOL = T + 2 * r, NCP = colhist4p_ncolp(T, r), NPR = NCP / 2;
    uint32_t *rec = reinterpret_cast<uint32_t *>(smem_raw);  // [85][NCP] singles (high byte)
    uint32_t *prs = rec + CH4_RECS * NCP;                     // [PR][NPR] pairs
    uint16_t *scol = reinterpret_cast<uint16_t *>(prs + PR * NPR);  // [NCOL][n] sorted spans
    uint8_t *cand = reinterpret_cast<uint8_t *>(scol) + (((size_t)NCOL * n * 2 + 15) & ~(size_t)15);  // [CMAX][T]
    // crowded bins: 16 u16 counters per thread, counter q in the thread's own
    // candidate bytes 2q (low) and 2q + 1 (high) -- the same bytes it would
    // use for candidates, never another thread's
    auto sc_get = [&](int q) -> uint32_t { return cand[(2 * q) * T + tid] | (cand[(2 * q + 1) * T + tid] << 8); };
    auto sc_set = [&](int q, uint32_t v) {
        cand[(2 * q) * T + tid] = (uint8_t)v;
        cand[(2 * q + 1) * T + tid] = (uint8_t)(v >> 8);
    };
    uint8_t *recb = smem_raw;
    const int X0 = blockIdx.x * T;
    const int y0 = p.row_begin + blockIdx.y * p.rows_per_cta;
    if (y0 >= p.row_end) return;  // CTA-uniform (barriers below)
    const int y1 = min(y0 + p.rows_per_cta, p.row_end);
    if (STREAM) stream_wait_rows(p, y1 + r);
    const uint16_t *src = static_cast<const uint16_t *>(p.src) + blockIdx.z * p.src_img_stride;
    uint16_t *dst = static_cast<uint16_t *>(p.dst) + blockIdx.z * p.dst_img_stride;
    const uint16_t *lut = static_cast<const uint16_t *>(p.lut);
    const int x = X0 + tid;

    // ---- records and sorted spans for row y0
    for (int i = tid; i < CH4_RECS * NCP; i += T) rec[i] = 0;
    __syncthreads();
    for (int c = tid; c < NCOL; c += T) {
        const int gx = clampi(X0 - r + c, 0, W - 1);
        uint16_t *a = scol + c * n;
        for (int j = 0; j < n; ++j) {
            const uint16_t v = __ldg(src_row(p, src, clampi(y0 - r + j, 0, H - 1)) + gx);
            ch4_bump_upd(recb, NCP, c, v >> 8, 1);
            int i = j;
            while (i > 0 && a[i - 1] > v) {
                a[i] = a[i - 1];
                --i;
            }
            a[i] = v;
        }
    }
    __syncthreads();
    for (int i = tid; i < PR * NPR; i += T) {
        const int row = i / NPR, k = i - row * NPR;
        prs[i] = rec[row * NCP + 2 * k] + rec[row * NCP + 2 * k + 1];
    }
    auto pbump_upper = [&](int c, unsigned v, int d) {  // pair levels 1-2
        const int k = c >> 1;
        const unsigned one = (unsigned)d;
        if (PL >= 2) atomicAdd(prs + (1 + (v >> 6)) * NPR + k, one << (8 * ((v >> 4) & 3)));
        if (PL >= 3) atomicAdd(prs + (5 + (v >> 4)) * NPR + k, one << (8 * ((v >> 2) & 3)));
    };
    // one column's row step: records of the high bytes (the -1 and +1 cancel
    // when they agree: no data-dependent branch), then the sorted span
    auto col_step = [&](int c, unsigned vo, unsigned vi) {
        // level 0 (one record per column and per pair): one combined atomic
        // each; levels 1-3 one per value
        const unsigned ho = vo >> 8, hi = vi >> 8;
        const unsigned d0 = (1u << (8 * (hi >> 6))) - (1u << (8 * (ho >> 6)));
        atomicAdd(rec + c, d0);
        atomicAdd(prs + (c >> 1), d0);
        uint32_t *rw = rec;
        atomicAdd(rw + ((1 + (ho >> 6)) * NCP + c), 0xffffffffu << (8 * ((ho >> 4) & 3)));
        atomicAdd(rw + ((1 + (hi >> 6)) * NCP + c), 1u << (8 * ((hi >> 4) & 3)));
        atomicAdd(rw + ((5 + (ho >> 4)) * NCP + c), 0xffffffffu << (8 * ((ho >> 2) & 3)));
        atomicAdd(rw + ((5 + (hi >> 4)) * NCP + c), 1u << (8 * ((hi >> 2) & 3)));
        atomicAdd(rw + ((21 + (ho >> 2)) * NCP + c), 0xffffffffu << (8 * (ho & 3)));
        atomicAdd(rw + ((21 + (hi >> 2)) * NCP + c), 1u << (8 * (hi & 3)));
        pbump_upper(c, ho, -1);
        pbump_upper(c, hi, 1);
        if (vo == vi) return;
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
    };
    constexpr int CH_PF = 2;
    int gxs[CH_PF];
#pragma unroll
    for (int u = 0; u < CH_PF; ++u) gxs[u] = clampi(X0 - r + min(tid + u * T, NCOL - 1), 0, W - 1);
    unsigned pvo[CH_PF], pvi[CH_PF];
    auto prefetch = [&](int yn) {
        const uint16_t *ro = src_row(p, src, clampi(yn - r - 1, 0, H - 1));
        const uint16_t *ri = src_row(p, src, clampi(yn + r, 0, H - 1));
#pragma unroll
        for (int u = 0; u < CH_PF; ++u) {
            pvo[u] = __ldg(ro + gxs[u]);
            pvi[u] = __ldg(ri + gxs[u]);
        }
    };
    if (y0 + 1 < y1) prefetch(y0 + 1);
    // the thread's window: stripe columns tid .. tid+n-1
    const int kp = (tid + 1) >> 1, cs = (tid & 1) ? tid : tid + n - 1, np = (n - 1) >> 1;
    const uint16_t *wcol = scol + tid * n;
    for (int y = y0; y < y1; ++y) {
        if (y > y0) {
            const int yo = clampi(y - r - 1, 0, H - 1), yi = clampi(y + r, 0, H - 1);
            __syncthreads();  // previous row's reads done (also orders the pair init)
            if (yo != yi) {
#pragma unroll
                for (int u = 0; u < CH_PF; ++u) {
                    const int c = tid + u * T;
                    if (c < NCOL) col_step(c, pvo[u], pvi[u]);
                }
                if (NCOL > CH_PF * T) {
                    const uint16_t *ro = src_row(p, src, yo), *ri = src_row(p, src, yi);
                    for (int c = tid + CH_PF * T; c < NCOL; c += T) {
                        const int gx = clampi(X0 - r + c, 0, W - 1);
                        col_step(c, __ldg(ro + gx), __ldg(ri + gx));
                    }
                }
            }
            if (y + 1 < y1) prefetch(y + 1);
        }
        __syncthreads();
        // ---- 1. high byte H and the rank k within it
        uint32_t k = p.rank, w0, w1;
        ch4p_gather<GP>(prs, rec, kp, cs, np, w0, w1);
        const int d3 = ch4_descend(w0, w1, k);
        if (PL >= 2)
            ch4p_gather<GP>(prs + (1 + d3) * NPR, rec + (1 + d3) * NCP, kp, cs, np, w0, w1);
        else
            ch4_gather<G, M>(rec + (1 + d3) * NCP + tid, n, w0, w1);
        const int d2 = ch4_descend(w0, w1, k);
        const int p2 = d3 * 4 + d2;
        if (PL >= 3)
            ch4p_gather<GP>(prs + (5 + p2) * NPR, rec + (5 + p2) * NCP, kp, cs, np, w0, w1);
        else
            ch4_gather<G, M>(rec + (5 + p2) * NCP + tid, n, w0, w1);
        const int d1 = ch4_descend(w0, w1, k);
        const int p3 = p2 * 4 + d1;
        ch4_gather<G, M>(rec + (21 + p3) * NCP + tid, n, w0, w1);
        const int d0 = ch4_descend(w0, w1, k);
        const unsigned hb = (unsigned)(p3 * 4 + d0);
        const uint32_t cH = ((d0 & 2 ? w1 : w0) >> (16 * (d0 & 1))) & 0xffffu;  // count of H
        // ---- 2. the window values with high byte H: one run per column
        const uint32_t *r0 = rec + tid, *r1 = rec + (1 + d3) * NCP + tid;
        const uint32_t *r2 = rec + (5 + p2) * NCP + tid, *r3 = rec + (21 + p3) * NCP + tid;
        const uint32_t m0 = ch16c_below_w(d3), m1 = ch16c_below_w(d2), m2 = ch16c_below_w(d1),
                       m3 = ch16c_below_w(d0);
        const unsigned sh0 = 8 * d0;
        unsigned lo;
        if (cH <= (uint32_t)CMAX) {
            // candidates: the c_H <= CMAX low bytes, stored per thread
            int cnt = 0;
#pragma unroll 4
            for (int j = 0; j < n; ++j) {
                const uint32_t w3 = r3[j];
                const int e0 = (int)__dp4a(r0[j], m0, __dp4a(r1[j], m1, __dp4a(r2[j], m2, __dp4a(w3, m3, 0u))));
                const int ne = (int)((w3 >> sh0) & 0xffu);
                const uint16_t *a = wcol + j * n;
                // run lengths 0, 1, 2 without a branch (addresses stay inside the column)
                const unsigned v0 = a[ne > 0 ? e0 : 0], v1 = a[ne > 1 ? e0 + 1 : 0];
                if (ne > 0) cand[cnt * T + tid] = (uint8_t)v0;
                if (ne > 1) cand[(cnt + 1) * T + tid] = (uint8_t)v1;
                cnt += min(ne, 2);
                if (ne > 2) {  // rare on spread data
                    for (int e = 2; e < ne; ++e) cand[cnt++ * T + tid] = (uint8_t)a[e0 + e];
                }
            }
            // ---- 3. k-th smallest low byte
            if (cnt <= 8) {
                // the usual handful: a 19-comparator sorting network on registers
                uint32_t v[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = i < cnt ? (uint32_t)cand[i * T + tid] : 0x100u;
                auto cx = [&](int i, int j) {
                    const uint32_t lo_ = min(v[i], v[j]), hi_ = max(v[i], v[j]);
                    v[i] = lo_;
                    v[j] = hi_;
                };
                cx(0, 2); cx(1, 3); cx(4, 6); cx(5, 7);
                cx(0, 4); cx(1, 5); cx(2, 6); cx(3, 7);
                cx(0, 1); cx(2, 3); cx(4, 5); cx(6, 7);
                cx(2, 4); cx(3, 5);
                cx(1, 4); cx(3, 6);
                cx(1, 2); cx(3, 4); cx(5, 6);
                lo = v[0];
#pragma unroll
                for (int i = 1; i < 8; ++i) lo = (k == (uint32_t)(i + 1)) ? v[i] : lo;
            } else {
                // high nibble, then low nibble
                uint32_t hn[4] = {0, 0, 0, 0};
                for (int i = 0; i < cnt; ++i) ch16c_count(hn, cand[i * T + tid] >> 4, true);
                const int nh = ch16c_descend16(hn, k);
                uint32_t ln[4] = {0, 0, 0, 0};
                for (int i = 0; i < cnt; ++i) {
                    const unsigned v = cand[i * T + tid];
                    ch16c_count(ln, v & 15u, (int)(v >> 4) == nh);
                }
                lo = (unsigned)(nh * 16 + ch16c_descend16(ln, k));
            }
        } else {
            // a crowded bin (compact data): two counting passes over the runs
            auto runs = [&](auto &&visit) {
                for (int j = 0; j < n; ++j) {
                    const uint32_t w3 = r3[j];
                    const int e0 = (int)__dp4a(r0[j], m0, __dp4a(r1[j], m1, __dp4a(r2[j], m2, __dp4a(w3, m3, 0u))));
                    const int ne = (int)((w3 >> sh0) & 0xffu);
                    const uint16_t *a = wcol + j * n + e0;
                    for (int e = 0; e < ne; ++e) visit(a[e] & 0xffu);
                }
            };
            auto pick = [&](uint32_t &kk) {
                int b = 0;
                for (; b < 15; ++b) {
                    const uint32_t c = sc_get(b);
                    if (c >= kk) break;
                    kk -= c;
                }
                return b;
            };
#pragma unroll
            for (int q = 0; q < 16; ++q) sc_set(q, 0);
            runs([&](unsigned v) { sc_set(v >> 4, sc_get(v >> 4) + 1); });
            const int nh = pick(k);
#pragma unroll
            for (int q = 0; q < 16; ++q) sc_set(q, 0);
            runs([&](unsigned v) {
                if ((int)(v >> 4) == nh) sc_set(v & 15, sc_get(v & 15) + 1);
            });
            lo = (unsigned)(nh * 16 + pick(k));
        }
        const unsigned v = (hb << 8) | lo;
        if (x < W) dst[(int64_t)(y - p.row_begin) * p.dst_pitch + x] = lut ? __ldg(lut + v) : (uint16_t)v;
    }
    if (STREAM) stream_signal(p, y0, y1, X0, X0 + T);
}

}  // namespace mtb
