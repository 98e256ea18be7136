// kernels_sortnet.cuh -- median filter for small windows (n = 3, 5, 7) by
// selection networks on packed pairs of pixels.
//
// Two horizontally adjacent outputs are processed together in one 32-bit
// register as two u16 lanes: sm_100a has native VIMNMX.U16x2, so one
// min/max instruction acts on both outputs (8-bit data is zero-extended).
// For the output pair (x, x+1) the window's j-th column pair is
// P_j = (col x-r+j, col x-r+j+1): its low lane belongs to output x and its
// high lane to output x+1, so the pair's whole window is n packed columns.
//
// Per output row (the classic "sort columns, sort rows, keep the band"):
//   1. sort each packed column vertically (n values; two output rows share
//      n-1 of them: sort those once, then insert the extra row);
//   2. sort each row of the column-sorted n x n matrix;
//   3. with rows and columns sorted, element (i,j) has >= (i+1)(j+1)-1
//      values below it and >= (n-i)(n-j)-1 above it, so every element with
//      (i+1)(j+1) > m or (n-i)(n-j) > m (m = (n^2+1)/2) is eliminated --
//      symmetrically -- and the median is the median of the survivors;
//   4. a Batcher odd-even merge network over the survivors; only its middle
//      output is used, so dead-code elimination prunes it to a selection
//      network.
// Exact: only min/max of pixel values.  Default rank (the median) only;
// other ranks use the histogram kernels.
#pragma once
#include "common.cuh"

namespace mtb {

__device__ __forceinline__ void cas2(uint32_t &x, uint32_t &y) {
    const uint32_t lo = __vminu2(x, y);
    y = __vmaxu2(x, y);
    x = lo;
}

// ---- Batcher odd-even merge sort as template recursion (indices are
// compile-time constants, so the arrays stay in registers); comparators
// touching an index >= M (virtual +inf padding) are dropped.
template <int M, int LO, int HI, int R>
struct OEMerge {
    template <class A>
    __device__ __forceinline__ static void run(A &v) {
        constexpr int STEP = 2 * R;
        if constexpr (STEP < HI - LO) {
            OEMerge<M, LO, HI, STEP>::run(v);
            OEMerge<M, LO + R, HI, STEP>::run(v);
#pragma unroll
            for (int i = LO + R; i < HI - R; i += STEP)
                if (i + R < M) cas2(v[i], v[i + R]);
        } else {
            if constexpr (LO + R < M) cas2(v[LO], v[LO + R]);
        }
    }
};

template <int M, int LO, int HI>
struct OESort {
    template <class A>
    __device__ __forceinline__ static void run(A &v) {
        if constexpr (HI - LO >= 1) {
            constexpr int MID = LO + (HI - LO) / 2;
            OESort<M, LO, MID>::run(v);
            OESort<M, MID + 1, HI>::run(v);
            OEMerge<M, LO, HI, 1>::run(v);
        }
    }
};

constexpr int pow2_ceil(int m) {
    int p = 1;
    while (p < m) p <<= 1;
    return p;
}

template <int M>
__device__ __forceinline__ void sortnet(uint32_t (&v)[M]) {
    if constexpr (M > 1) OESort<M, 0, pow2_ceil(M) - 1>::run(v);
}

// survivors of the band elimination for an n x n matrix with sorted rows
// and columns (median rank m = (n*n+1)/2)
template <int N>
struct Band {
    int i[N * N], j[N * N];
    int count;
    constexpr Band() : i(), j(), count(0) {
        const int m = (N * N + 1) / 2;
        for (int r = 0; r < N; ++r)
            for (int c = 0; c < N; ++c)
                if ((r + 1) * (c + 1) <= m && (N - r) * (N - c) <= m) {
                    i[count] = r;
                    j[count] = c;
                    ++count;
                }
    }
};

// median of the packed window given its n sorted packed columns col[0..n-1]
template <int N>
__device__ __forceinline__ uint32_t band_median(const uint32_t (&col)[N][N]) {
    // rows of the column-sorted matrix, each sorted across the n columns
    uint32_t row[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int j = 0; j < N; ++j) row[i][j] = col[j][i];
        sortnet<N>(row[i]);
    }
    constexpr Band<N> band{};
    uint32_t cand[band.count];
#pragma unroll
    for (int t = 0; t < band.count; ++t) cand[t] = row[band.i[t]][band.j[t]];
    sortnet<band.count>(cand);
    return cand[band.count / 2];
}

// Tile: 32 x 4 threads; thread (tx, ty) computes K output pairs (2K columns)
// for RT consecutive rows.  The CTA stages its input tile (with r halo,
// clamped to the global image) in shared memory as u16.
template <int N, int K, int RT, typename P>
__global__ void __launch_bounds__(128) k_sortnet(SlabParams p) {
    constexpr int R = N / 2;
    constexpr int TX = 32 * 2 * K;           // output columns per CTA
    constexpr int TY = 4 * RT;               // output rows per CTA
    constexpr int SW = TX + 2 * R + 2;       // staged width (even, +pad)
    constexpr int SH = TY + 2 * R;
    __shared__ __align__(16) uint16_t tile[SH][SW];

    const int W = p.W, H = p.H;
    const int X0 = blockIdx.x * TX;
    const int Y0 = p.row_begin + blockIdx.y * TY;
    const P *src = static_cast<const P *>(p.src) + blockIdx.z * p.src_img_stride;
    P *dst = static_cast<P *>(p.dst) + blockIdx.z * p.dst_img_stride;
    const P *lut = static_cast<const P *>(p.lut);
    const int tid = threadIdx.x + 32 * threadIdx.y;
    stream_wait_rows(p, Y0 + TY + R);

    // stage rows Y0-R .. Y0+TY+R-1, columns X0-R .. X0+TX+R-1 (clamped)
    for (int idx = tid; idx < SH * SW; idx += 128) {
        const int yy = idx / SW, xx = idx - yy * SW;
        const int gy = clampi(Y0 - R + yy, 0, H - 1);
        const int gx = clampi(X0 - R + xx, 0, W - 1);
        tile[yy][xx] = (uint16_t)__ldg(src_row(p, src, gy) + gx);
    }
    __syncthreads();

    const int lx = threadIdx.x * 2 * K;      // first output column (tile coords)
    const int ly0 = threadIdx.y * RT;
    // packed column j covers staged columns lx + j, lx + j + 1
    auto pair_at = [&](int yy, int j) -> uint32_t {
        const int c = lx + j;
        if ((j & 1) == 0) return *reinterpret_cast<const uint32_t *>(&tile[yy][c]);
        const uint32_t w0 = *reinterpret_cast<const uint32_t *>(&tile[yy][c - 1]);
        const uint32_t w1 = *reinterpret_cast<const uint32_t *>(&tile[yy][c + 1]);
        return __byte_perm(w0, w1, 0x5432);
    };
    constexpr int NC = N + 2 * (K - 1);      // packed columns used by K pairs

#pragma unroll 1
    for (int ry = 0; ry < RT; ry += 2) {
        const int ly = ly0 + ry;              // output rows ly, ly+1 (tile coords)
        // core rows ly-R+1 .. ly+R are shared by the two output rows
        uint32_t core[NC][N - 1];
#pragma unroll
        for (int j = 0; j < NC; ++j) {
#pragma unroll
            for (int k = 0; k < N - 1; ++k) core[j][k] = pair_at(ly + 1 + k, j);
            sortnet<N - 1>(core[j]);
        }
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int gy = Y0 + ly + half;
            // each output row adds one extra row to the core: ly-R or ly+1+R
            const int extra = half ? ly + 2 * R + 1 : ly;
            uint32_t cs[NC][N];
#pragma unroll
            for (int j = 0; j < NC; ++j) {
                uint32_t x = pair_at(extra, j);
#pragma unroll
                for (int k = 0; k < N - 1; ++k) {
                    cs[j][k] = __vminu2(core[j][k], x);
                    x = __vmaxu2(core[j][k], x);
                }
                cs[j][N - 1] = x;
            }
            if (gy >= p.row_end) break;
            P *drow = dst + (int64_t)(gy - p.row_begin) * p.dst_pitch;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                uint32_t col[N][N];
#pragma unroll
                for (int j = 0; j < N; ++j)
#pragma unroll
                    for (int i = 0; i < N; ++i) col[j][i] = cs[2 * k + j][i];
                const uint32_t med = band_median<N>(col);
                const int x = X0 + lx + 2 * k;
                uint32_t v0 = med & 0xffffu, v1 = med >> 16;
                if (lut) {
                    v0 = __ldg(lut + v0);
                    v1 = __ldg(lut + v1);
                }
                if (x < W) drow[x] = (P)v0;
                if (x + 1 < W) drow[x + 1] = (P)v1;
            }
        }
    }
    stream_signal(p, Y0, Y0 + TY, X0, X0 + TX);
}

}  // namespace mtb
