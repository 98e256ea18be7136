// (A from TMEM: -DA_TMEM)  Unit check of the tcgen05 int8 path used by k_bandtc_u8: D[128 x N] (s32, TMEM)
// = A[128 x 32] (u8, K-major blocked smem tile) x B[N x 32] (u8, K-major planes in
// the blocked layout), one or more K steps, read back with tcgen05.ld 32x32b.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int M = 128, N = 48, KT = 32, KSTEPS = 3;
constexpr int NPC = 16;                    // column chunks (16 B) per plane group row block: NP = 256 columns
constexpr int NP = NPC * 16;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: 8 rows x 16 B core matrices; LBO = K-direction stride, SBO = MN-direction stride
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3ffff) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
    d |= (uint64_t)1 << 46;  // version = 1 (Blackwell)
    return d;
}

__global__ void k(const uint8_t *A, const uint8_t *B, int *D) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint8_t *sA = sm;                                   // KSTEPS tiles of 128 x 32 blocked: (m/8)*256 + (k/16)*128 + (m%8)*16 + k%16
    uint8_t *sB = sm + KSTEPS * 4096;                   // planes: (p/8)*(NPC*128) + (c/16)*128 + (p%8)*16 + c%16
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < KSTEPS * M * KT; i += blockDim.x) {
        const int s = i / (M * KT), m = (i / KT) % M, kk = i % KT;
        sA[s * 4096 + (m / 8) * 256 + (kk / 16) * 128 + (m % 8) * 16 + kk % 16] = A[i];
    }
    for (int i = tid; i < N * NP; i += blockDim.x) {
        const int p = i / NP, c = i % NP;
        sB[(p / 8) * (NPC * 128) + (c / 16) * 128 + (p % 8) * 16 + c % 16] = B[i];
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tmem_base)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tmem_base;
#ifdef A_TMEM
    // band rows into TMEM: thread m = lane m, K step s at columns 64 + 8 s .. (row bytes k = 4 word + byte)
    for (int s = 0; s < KSTEPS; ++s) {
        uint32_t w[8];
        for (int j = 0; j < 8; ++j) {
            w[j] = 0;
            for (int b = 0; b < 4; ++b) w[j] |= (uint32_t)A[(s * M + tid) * KT + 4 * j + b] << (8 * b);
        }
        const uint32_t ta = tm + ((uint32_t)(32 * warp) << 16) + 64 + 8 * s;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                     ::"r"(ta), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#endif
    if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy smem writes -> async proxy
        // idesc: c_format S32 (2) at [4,6), a/b format u8 (0), K-major both, N >> 3 at [17,23), M >> 4 at [24,29)
        const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const int col0 = 48;  // window columns start here (multiple of 16)
        for (int s = 0; s < KSTEPS; ++s) {
            const uint64_t da = make_desc(smem_u32(sA + s * 4096), 128, 256);
            const uint64_t db = make_desc(smem_u32(sB + ((col0 + 32 * s) / 16) * 128), 128, NPC * 128);
            const uint32_t acc = s > 0;
#ifdef A_TMEM
            (void)da;
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n}\n"
                ::"r"(tm), "r"(tm + 64 + 8 * s), "l"(db), "r"(idesc), "r"(acc), "r"(0u) : "memory");
#else
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n}\n"
                ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(0u) : "memory");
#endif
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    }
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.b32 %0, 1, 0, P;\n}\n"
                     : "=r"(done) : "r"(smem_u32(&bar)), "r"(0u) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // warp w reads TMEM lanes 32w .. 32w+31 (its quadrant), N columns, 16 at a time
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        const uint32_t ta = tm + ((uint32_t)(32 * warp) << 16) + c0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(ta) : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 16; ++j) D[tid * N + c0 + j] = (int)v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm) : "memory");
}

int main() {
    static uint8_t hA[KSTEPS * M * KT], hB[N * NP];
    static int hD[M * N];
    srand(1);
    for (auto &x : hA) x = rand() % 2;
    for (auto &x : hB) x = rand() % 200;
    uint8_t *dA, *dB; int *dD;
    cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, sizeof hD);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    const size_t smem = KSTEPS * 4096 + (size_t)(N / 8) * NPC * 128;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<1, 128, smem>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            int s = 0;
            for (int st = 0; st < KSTEPS; ++st)
                for (int kk = 0; kk < KT; ++kk) s += hA[(st * M + m) * KT + kk] * hB[n * NP + 48 + 32 * st + kk];
            if (s != hD[m * N + n]) { if (bad < 5) printf("mismatch m=%d n=%d got %d want %d\n", m, n, hD[m * N + n], s); ++bad; }
        }
    printf("mismatches: %d of %d\n", bad, M * N);
    return bad != 0;
}
