// Microbenchmark: mma.sync m16n8k32 u8 x u8 -> s32 throughput on sm_100a, and a
// fragment-layout check (banded 0/1 matrix times u8 counts).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma_u8(int (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int ILP>
__global__ void k_tput(int iters, int *out, uint32_t seed) {
    uint32_t a[4] = {seed, seed + 1, seed + 2, seed + 3};
    uint32_t b[2] = {seed * 3, seed * 5};
    int d[ILP][4];
#pragma unroll
    for (int i = 0; i < ILP; ++i) d[i][0] = d[i][1] = d[i][2] = d[i][3] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) mma_u8(d[i], a, b);
    }
    int s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += d[i][0] + d[i][1] + d[i][2] + d[i][3];
    if (s == 0x12345678) out[0] = s;
}

// layout check: A[m][k] (16x32, row), B[k][n] (32x8, col), D = A*B
__global__ void k_layout(const uint8_t *A, const uint8_t *B, int *D) {
    const int lane = threadIdx.x, g = lane >> 2, q = lane & 3;
    uint32_t a[4], b[2];
    auto pack = [&](const uint8_t *p) { return (uint32_t)p[0] | (uint32_t)p[1] << 8 | (uint32_t)p[2] << 16 | (uint32_t)p[3] << 24; };
    a[0] = pack(A + g * 32 + 4 * q);
    a[1] = pack(A + (g + 8) * 32 + 4 * q);
    a[2] = pack(A + g * 32 + 16 + 4 * q);
    a[3] = pack(A + (g + 8) * 32 + 16 + 4 * q);
    uint8_t t[4];
    for (int i = 0; i < 4; ++i) t[i] = B[(4 * q + i) * 8 + g];
    b[0] = pack(t);
    for (int i = 0; i < 4; ++i) t[i] = B[(16 + 4 * q + i) * 8 + g];
    b[1] = pack(t);
    int d[4] = {0, 0, 0, 0};
    mma_u8(d, a, b);
    D[g * 8 + 2 * q] = d[0];
    D[g * 8 + 2 * q + 1] = d[1];
    D[(g + 8) * 8 + 2 * q] = d[2];
    D[(g + 8) * 8 + 2 * q + 1] = d[3];
}

int main() {
    int *out;
    cudaMalloc(&out, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int dev_clk;
    cudaDeviceGetAttribute(&dev_clk, cudaDevAttrClockRate, 0);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 20000;
    for (int warps = 4; warps <= 32; warps *= 2) {
        for (int pass = 0; pass < 2; ++pass) {
            cudaEventRecord(e0);
            k_tput<8><<<sms, warps * 32>>>(iters, out, 1);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (pass) {
                double mmas = (double)sms * warps * iters * 8;
                double per_clk_sm = mmas / sms / (ms * 1e-3 * dev_clk * 1e3);
                printf("warps/SM %2d ILP 8: %.3f ms, %.3f MMA(m16n8k32 u8)/clk/SM at %d kHz -> %.1f TOPS\n", warps, ms,
                       per_clk_sm, dev_clk, mmas * 16 * 8 * 32 * 2 / (ms * 1e-3) / 1e12);
            }
        }
    }
    // layout
    uint8_t hA[16 * 32], hB[32 * 8];
    for (int i = 0; i < 16 * 32; ++i) hA[i] = (i * 7 + 3) % 5 == 0;
    for (int i = 0; i < 32 * 8; ++i) hB[i] = (uint8_t)((i * 37 + 11) % 251);
    uint8_t *dA, *dB;
    int *dD, hD[16 * 8];
    cudaMalloc(&dA, sizeof hA);
    cudaMalloc(&dB, sizeof hB);
    cudaMalloc(&dD, sizeof hD);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    k_layout<<<1, 32>>>(dA, dB, dD);
    cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < 16; ++m)
        for (int n = 0; n < 8; ++n) {
            int s = 0;
            for (int k = 0; k < 32; ++k) s += hA[m * 32 + k] * hB[k * 8 + n];
            if (s != hD[m * 8 + n]) ++bad;
        }
    printf("layout check: %d mismatches (%s)\n", bad, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
