// kernels_mednet.cuh -- n = 5 and n = 7 medians (r = 2, 3) from sorted
// packed columns with merge sharing between neighbouring outputs.
//
// k_sortnet<n> re-sorts every window's rows and runs a band-selection
// network per output pair (~320 lane-instructions per pixel at n = 7).
// Here the work is factored the way separable median networks share it:
//
//   * PK ring: every input row, once, becomes packed columns
//     PK[m] = (col X-R+m, col X-R+m+1) as u16 pairs (8-bit pixels are
//     zero-extended; 16-bit pixels fit the lanes as they are), kept for the
//     n + 1 rows the next two output rows read.
//   * Phase V (per two output rows): every packed column of the CTA's tile
//     sorts its n - 1 shared rows once (a selection network), then inserts
//     the row above for output row y and the row below for y + 1, and
//     stores both sorted columns (n words each) in shared memory.
//   * Phase H: a thread owns two adjacent output PAIRS (4 pixels).  Pair 0's
//     window is sorted columns C_0..C_{n-1}, pair 1's C_2..C_{n+1}; the
//     shared C_2..C_{n-1} are merged once, each pair merges its two extra
//     columns and takes the median of the two sorted lists as
//     min_i max(A[i-1], S[k-i]).  The straight-line code is generated with
//     dead-code elimination by tools/gen_mednet.py (mednet_gen.cuh):
//     400 min/max per 4 outputs at n = 7, 162 at n = 5.
//
// Exact (min/max of pixel values only); median rank only; replicate
// borders (columns and rows clamp to the image).
#pragma once
#include "common.cuh"
#include "kernels_sortnet.cuh"  // sortnet<M> (odd-even merge sort on registers)
#include "mednet_gen.cuh"

namespace mtb {

constexpr int MN_T = 128;          // threads per CTA
constexpr int MN_TX = 4 * MN_T;    // output columns per CTA (4 per thread)

__host__ __device__ constexpr int mn_npc(int N) { return MN_TX + N - 1; }           // packed columns
__host__ __device__ constexpr int mn_pkstride(int N) { return (mn_npc(N) + 3) & ~3; }
constexpr int MN_SCS = MN_TX + 8;  // sorted-column row stride (phase H reads 12 columns from 4t)
__host__ __device__ constexpr int mn_smem(int N) {
    // PK ring [N+1][stride] + sorted columns [2][N][MN_SCS] (u32, component-major)
    return ((N + 1) * mn_pkstride(N) + 2 * N * MN_SCS) * 4;
}

// o = sorted(a u {x}) for sorted a[0..M-1]
template <int M>
__device__ __forceinline__ void mn_insert(const uint32_t (&a)[M], uint32_t x, uint32_t (&o)[M + 1]) {
    o[0] = __vminu2(a[0], x);
#pragma unroll
    for (int i = 1; i < M; ++i) o[i] = __vmaxu2(a[i - 1], __vminu2(a[i], x));
    o[M] = __vmaxu2(a[M - 1], x);
}

template <int N>
__device__ __forceinline__ void mednet_pairs(const uint32_t (&c)[N + 2][N], uint32_t &o0, uint32_t &o1);
template <>
__device__ __forceinline__ void mednet_pairs<5>(const uint32_t (&c)[7][5], uint32_t &o0, uint32_t &o1) {
    mednet_pairs5(c, o0, o1);
}
template <>
__device__ __forceinline__ void mednet_pairs<7>(const uint32_t (&c)[9][7], uint32_t &o0, uint32_t &o1) {
    mednet_pairs7(c, o0, o1);
}

template <int N, typename P>
__global__ void __launch_bounds__(MN_T) k_mednet(SlabParams p) {
    constexpr int R = N / 2;
    constexpr int NPC = mn_npc(N), PKS = mn_pkstride(N), NR = N + 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t *pk = reinterpret_cast<uint32_t *>(smem_raw);  // [NR][PKS]
    uint32_t *sc = pk + NR * PKS;                            // [2][N][MN_SCS]
    const int tid = threadIdx.x;
    const int W = p.W, H = p.H;
    const int X = blockIdx.x * MN_TX;
    const int Y0 = p.row_begin + blockIdx.y * p.rows_per_cta;
    const int Y1 = min(Y0 + p.rows_per_cta, p.row_end);
    const P *src = static_cast<const P *>(p.src) + blockIdx.z * p.src_img_stride;
    P *dst = static_cast<P *>(p.dst) + blockIdx.z * p.dst_img_stride;
    const P *lut = static_cast<const P *>(p.lut);
    stream_wait_rows(p, Y1 + R);
    // input rows the band reads: Y0-R .. Y1+R-1 (clamped to the image)
    const int ylo = max(Y0 - R, 0), yhi = min(Y1 + R, H) - 1;
    // this thread's packed columns m = tid + MN_T*u (u < MU) of one input row,
    // loaded into registers (issued a step ahead) and stored to the ring later
    constexpr int MU = (NPC + MN_T - 1) / MN_T;
    const bool interior = X - R >= 0 && X - R + NPC <= W - 1;  // no column clamping (CTA-uniform)
    // (raw pixels: combined into packed words only when stored, so the
    // loads stay in flight across the phases in between)
    auto fetch_row = [&](int g, uint32_t (&va)[MU], uint32_t (&vb)[MU]) {
        const P *row = src_row(p, src, clampi(g, ylo, yhi)) + (X - R);
#pragma unroll
        for (int u = 0; u < MU; ++u) {
            const int m = tid + MN_T * u;
            if (m < NPC) {
                if (interior) {
                    va[u] = __ldg(row + m);
                    vb[u] = __ldg(row + m + 1);
                } else {
                    const int c = X - R + m;
                    va[u] = __ldg(row + (clampi(c, 0, W - 1) - (X - R)));
                    vb[u] = __ldg(row + (clampi(c + 1, 0, W - 1) - (X - R)));
                }
            }
        }
    };
    // ring slot of input row g
    auto slot = [&](int g) { return ((g - (Y0 - R)) % NR) * PKS; };
    auto store_row = [&](int g, const uint32_t (&va)[MU], const uint32_t (&vb)[MU]) {
        uint32_t *d = pk + slot(g);
#pragma unroll
        for (int u = 0; u < MU; ++u) {
            const int m = tid + MN_T * u;
            if (m < NPC) d[m] = va[u] | (vb[u] << 16);
        }
    };
    {
        uint32_t va[MU], vb[MU];
        for (int g = Y0 - R; g <= Y0 + R + 1; ++g) {
            fetch_row(g, va, vb);
            store_row(g, va, vb);
        }
    }
    uint32_t pa0[MU], pb0[MU], pa1[MU], pb1[MU];  // input rows y+R+2, y+R+3 in flight
    fetch_row(Y0 + R + 2, pa0, pb0);
    fetch_row(Y0 + R + 3, pa1, pb1);
    for (int y = Y0; y < Y1; y += 2) {
        __syncthreads();  // ring holds rows y-R .. y+R+1; the previous phase H is done with sc
        // ---- phase V: sorted columns for output rows y (sc[0..N)) and y+1 (sc[N..2N))
        int sl[N + 1];
#pragma unroll
        for (int k = 0; k <= N; ++k) sl[k] = slot(y - R + k);
        for (int m = tid; m < NPC; m += MN_T) {
            uint32_t core[N - 1];
#pragma unroll
            for (int k = 0; k < N - 1; ++k) core[k] = pk[sl[k + 1] + m];
            sortnet<N - 1>(core);
            uint32_t c0[N], c1[N];
            mn_insert<N - 1>(core, pk[sl[0] + m], c0);  // + row y-R    -> output row y
            mn_insert<N - 1>(core, pk[sl[N] + m], c1);  // + row y+R+1  -> output row y+1
#pragma unroll
            for (int k = 0; k < N; ++k) {
                sc[k * MN_SCS + m] = c0[k];
                sc[(N + k) * MN_SCS + m] = c1[k];
            }
        }
        __syncthreads();
        // rows y-R, y-R+1 are free: their slots take rows y+R+2, y+R+3, and
        // the loads of the rows after those are issued
        store_row(y + R + 2, pa0, pb0);
        store_row(y + R + 3, pa1, pb1);
        if (y + 2 < Y1) {
            fetch_row(y + R + 4, pa0, pb0);
            fetch_row(y + R + 5, pa1, pb1);
        }
        // ---- phase H: two pairs (4 outputs) per thread and row
        const int x0 = X + 4 * tid;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int yy = y + h;
            if (yy >= Y1) break;
            // sorted columns 4t .. 4t+N+1: per component, three 16-B loads
            // (the warp's 32 lanes read 512 contiguous bytes each)
            uint32_t c[N + 2][N];
#pragma unroll
            for (int k = 0; k < N; ++k) {
                const uint32_t *row = sc + (h * N + k) * MN_SCS + 4 * tid;
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const uint4 u = *reinterpret_cast<const uint4 *>(row + 4 * q);
                    const uint32_t v[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (4 * q + e < N + 2) c[4 * q + e][k] = v[e];
                }
            }
            uint32_t o0, o1;
            mednet_pairs<N>(c, o0, o1);
            uint32_t v[4] = {o0 & 0xffffu, o0 >> 16, o1 & 0xffffu, o1 >> 16};
            if (lut) {
#pragma unroll
                for (int q = 0; q < 4; ++q) v[q] = __ldg(lut + v[q]);
            }
            P *d = dst + (int64_t)(yy - p.row_begin) * p.dst_pitch + x0;
            if (sizeof(P) == 1 && x0 + 4 <= W && (reinterpret_cast<uintptr_t>(d) & 3) == 0) {
                *reinterpret_cast<uint32_t *>(d) = v[0] | (v[1] << 8) | (v[2] << 16) | (v[3] << 24);
            } else if (sizeof(P) == 2 && x0 + 4 <= W && (reinterpret_cast<uintptr_t>(d) & 7) == 0) {
                *reinterpret_cast<uint2 *>(d) = make_uint2(v[0] | (v[1] << 16), v[2] | (v[3] << 16));
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (x0 + q < W) d[q] = (P)v[q];
            }
        }
    }
    stream_signal(p, Y0, Y1, X, X + MN_TX);
}

}  // namespace mtb
