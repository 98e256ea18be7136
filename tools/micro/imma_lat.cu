// IMMA (mma.sync m16n8k32 u8) dependent-issue latency and throughput under the
// access pattern of k_bandmma_u8: accumulator chains fed by shared-memory loads.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma_u8(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// CHAINS independent accumulators, each a dependent chain of DEPTH IMMAs; B from smem when LDS
template <int CHAINS, int DEPTH, bool LDS>
__global__ void k(int iters, long long *out, int *sink) {
    __shared__ __align__(16) unsigned char sm[32 * 1024];
    for (int i = threadIdx.x; i < 32 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = i * 2654435761u;
    __syncthreads();
    const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
    uint32_t a[4] = {0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u};
    const unsigned char *rp = sm + g * 672 + 8 * q + (threadIdx.x >> 5) * 16;
    int tot = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        int acc[CHAINS][4];
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = 0;
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) {
#pragma unroll
            for (int c = 0; c < CHAINS; ++c) {
                uint2 b;
                if (LDS) b = *reinterpret_cast<const uint2 *>(rp + c * 8 * 672 + 32 * d);
                else b = make_uint2(lane + d, c + it);
                mma_u8(acc[c], a, b.x, b.y);
            }
        }
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) tot += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
    if (tot == 0x7fffffff) sink[0] = tot;
}

template <int CHAINS, int DEPTH, bool LDS>
void run(const char *name, int warps) {
    long long *out; int *sink;
    cudaMalloc(&out, 8); cudaMalloc(&sink, 4);
    const int iters = 2000;
    k<CHAINS, DEPTH, LDS><<<148, warps * 32>>>(iters, out, sink);
    k<CHAINS, DEPTH, LDS><<<148, warps * 32>>>(iters, out, sink);
    long long h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("%-34s warps/SM %2d: %7.1f clk per iteration (%d IMMA/warp) -> %.1f clk per IMMA per warp, %.2f clk/IMMA/SMSP\n", name, warps,
           (double)h / iters, CHAINS * DEPTH, (double)h / iters / (CHAINS * DEPTH), (double)h / iters / (CHAINS * DEPTH * (warps / 4.0 < 1 ? 1 : warps / 4.0)));
    cudaFree(out); cudaFree(sink);
}

int main() {
    run<1, 20, false>("1 chain x 20 deep, regs", 1);
    run<1, 20, true>("1 chain x 20 deep, LDS", 1);
    run<4, 5, false>("4 chains x 5 deep, regs", 1);
    run<4, 5, true>("4 chains x 5 deep, LDS", 1);
    run<4, 5, true>("4 chains x 5 deep, LDS", 4);
    run<4, 5, true>("4 chains x 5 deep, LDS", 16);
    run<4, 5, true>("4 chains x 5 deep, LDS", 32);
    run<1, 20, true>("1 chain x 20 deep, LDS", 32);
    run<4, 3, true>("4 chains x 3 deep, LDS", 32);
    run<8, 5, true>("8 chains x 5 deep, LDS", 16);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
