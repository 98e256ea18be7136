// Shared-memory atomicAdd (ATOMS.ADD, result unused) cost per warp instruction on one SM,
// 32 warps: dense / sparse lanes, same plane row / random plane rows (bandmma layout: 272 rows x 672 B).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(int iters, long long *out, const int *rnd) {
    extern __shared__ uint32_t sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < 272 * 168; i += blockDim.x) sm[i] = 0;
    __syncthreads();
    const int NPW = 168;
    unsigned r0 = (unsigned)rnd[tid], r1 = (unsigned)rnd[tid + 1024];
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        int row;
        bool active = true;
        if (MODE == 0) row = (it * 7 + warp) % 272;                       // dense, one plane row per warp
        if (MODE == 1) row = (int)((r0 >> 8) % 272u);                        // dense, random rows per lane
        if (MODE == 2) { row = (it * 7 + warp) % 272; active = (lane & 3) == (it & 3); }   // 25% lanes, same row
        if (MODE == 3) { row = (int)((r0 >> 8) % 272u); active = (lane & 3) == (it & 3); }    // 25% lanes, random rows
        if (MODE == 4) { row = (int)((r0 >> 8) % 272u); active = lane == (it & 31); }         // one lane
        if (active) atomicAdd(sm + row * NPW + (warp * 5 + lane) % 160, 1u << (8 * (r1 & 3)));
        r0 = r0 * 1103515245u + 12345u;
    }
    __syncthreads();
    const long long t1 = clock64();
    if (tid == 0) out[0] = t1 - t0;
    if (sm[tid] == 0xdeadbeef) out[1] = 1;
}

template <int MODE>
void run(const char *name, const int *drnd) {
    long long *out, h;
    cudaMalloc(&out, 16);
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 272 * 672);
    const int iters = 2000;
    k<MODE><<<1, 1024, 272 * 672>>>(iters, out, drnd);
    k<MODE><<<1, 1024, 272 * 672>>>(iters, out, drnd);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("%-34s %6.2f clk per warp-instruction per SM (%s)\n", name, (double)h / (iters * 32.0), cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    int h[2048];
    for (int i = 0; i < 2048; ++i) h[i] = (i * 2654435761u) >> 8;
    int *d; cudaMalloc(&d, sizeof h); cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
    run<0>("dense, one plane row per warp", d);
    run<1>("dense, random plane rows", d);
    run<2>("8 lanes, one plane row", d);
    run<3>("8 lanes, random plane rows", d);
    run<4>("1 lane", d);
    return 0;
}
