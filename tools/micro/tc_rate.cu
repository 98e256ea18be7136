// tcgen05.mma kind::i8 (M = 128, K = 32) time per instruction against N, A from tensor memory,
// B from shared memory (K-major, no swizzle), CNT back-to-back accumulating instructions.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr & 0x3ffff) >> 4) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46);
}

template <int N, int CNT>
__global__ void k(long long *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x01010101u;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tmem_base;
    if (warp == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t db = make_desc(smem_u32(sm), 128, 2048);
        const long long t0 = clock64();
#pragma unroll 8
        for (int s = 0; s < CNT; ++s) {
            asm volatile(
                "{\n .reg .pred p, q;\n elect.sync _|q, 0xffffffff;\n setp.ne.b32 p, %4, 0;\n"
                " @q tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n}\n"
                ::"r"(tm), "r"(tm + 400 + 8 * (s & 7)), "l"(db + (uint64_t)(16 * (s & 7))), "r"(idesc), "r"((uint32_t)(s > 0)), "r"(0u) : "memory");
        }
        asm volatile("{\n .reg .pred q;\n elect.sync _|q, 0xffffffff;\n @q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(&bar)) : "memory");
        const long long t1 = clock64();
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.b32 %0, 1, 0, P;\n}\n"
                         : "=r"(done) : "r"(smem_u32(&bar)), "r"(0u) : "memory");
        const long long t2 = clock64();
        if (tid == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

template <int N, int CNT>
void run() {
    long long *out, h[2];
    cudaMalloc(&out, 16);
    cudaFuncSetAttribute(k<N, CNT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k<N, CNT><<<1, 128, 64 * 1024>>>(out);
    k<N, CNT><<<1, 128, 64 * 1024>>>(out);
    cudaDeviceSynchronize();
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("N=%3d: %d instructions issued in %lld clk, done after %lld clk -> %.1f clk each (%s)\n", N, CNT, h[0], h[1],
           (double)h[1] / CNT, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    run<16, 64>(); run<32, 64>(); run<48, 64>(); run<64, 64>(); run<96, 64>(); run<128, 64>(); run<256, 64>();
    run<32, 8>(); run<64, 8>();
    return 0;
}
