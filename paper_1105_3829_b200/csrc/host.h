// host.h -- host-side helpers shared by the launcher translation units
// (medtree_b200.cu: dispatch + C ABI; run_colhist.cu, run_ctmf.cu: kernel
// families with many template instantiations, compiled in parallel).
#pragma once
#include <atomic>
#include <cstdint>
#include <string>
#include <type_traits>

#include "../../include/medtree_b200.h"
#include "common.cuh"

namespace mtb {

extern thread_local std::string g_err;
extern thread_local const char *g_kernel;
extern std::atomic<uint64_t> g_launches;

int fail(int code, const std::string &msg);
int sm_count();
int rows_per_cta(const SlabParams &p, int blocks_x, int B, int ctas_per_sm, int waves = 2);
int env_int(const char *name, int dflt);
const char *forced_kernel();
void keep_pool_memory();

// Opt in to the dynamic shared memory a launch needs (static __shared__
// of the kernel counts against the default 48 KB too, so always set it).
template <typename K>
inline int set_smem(K kernel, size_t smem) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(MTB_E_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    return MTB_OK;
}

template <typename K>
inline int launch(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t s, const SlabParams &p,
                  const char *name) {
    if (int rc = set_smem(kernel, smem)) return rc;
    kernel<<<grid, block, smem, s>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(MTB_E_CUDA, std::string(name) + ": " + cudaGetErrorString(e));
    g_kernel = name;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return MTB_OK;
}

// Calls f(std::integral_constant<int, N>{}) for the odd N == n in
// [NLO, NHI] (compile-time window side), f(integral_constant<int, 0>) else.
template <int NLO, int NHI, typename F>
inline int with_fixed_n(int n, F &&f) {
    if constexpr (NLO > NHI) {
        return f(std::integral_constant<int, 0>{});
    } else {
        if (n == NLO) return f(std::integral_constant<int, NLO>{});
        return with_fixed_n<NLO + 2, NHI>(n, f);
    }
}

// largest carry-free group of u8 records whose counts are <= c (G * c <= 255)
constexpr int carry_free_group(int c) { return 8 * c <= 255 ? 8 : (4 * c <= 255 ? 4 : (2 * c <= 255 ? 2 : 1)); }

// kernel families in their own translation units
int run_colhist_u8(SlabParams p, int B, cudaStream_t s);
int run_colhist4_256(SlabParams p, int B, cudaStream_t s);
int run_colhist4p_256(SlabParams p, int B, cudaStream_t s, int pl);
// wk: window-keyed first sweep (pays off on compact data, see kernel)
int run_colhist16_u16(SlabParams p, int B, cudaStream_t s, int wk = 1);
int run_colhist16s_u16(SlabParams p, int B, cudaStream_t s);
int run_colhist16c_u16(SlabParams p, int B, cudaStream_t s);
// 16-bit, widely spread data: high byte by pair records, low byte from per-block candidate lists,
// leftovers by the two-phase kernel (run_lowsel16.cu); device-resident launches, r = 3..63
constexpr int LOWSEL_MIN_R = 3, LOWSEL_MAX_R = 63;
bool lowsel16_applies(const SlabParams &p);
int run_lowsel16_u16(SlabParams p, int B, cudaStream_t s);
// 16-bit, compact and peaked data: one 8-bit pass per tile keyed by a 254-value window around the
// tile's median, leftovers by the two-phase kernel (run_lowsel16.cu); same launches and radii
int run_wk16_u16(SlabParams p, int B, cudaStream_t s);
// compile-time window sides of k_colhist16_u16; 1 (NOT_COVERED) when n is outside the range
int run_colhist16_fixed_a(SlabParams p, int B, cudaStream_t s, int wk);
int run_colhist16_fixed_b(SlabParams p, int B, cudaStream_t s, int wk);
int run_colhist16_fixed_c(SlabParams p, int B, cudaStream_t s, int wk);
int run_ctmf_u8(SlabParams p, int B, cudaStream_t s);
int run_bandmma_u8(SlabParams p, int B, cudaStream_t s);
int run_bandmma_hi16(SlabParams p, int B, cudaStream_t s);
int run_bandtc_u8(SlabParams p, int B, cudaStream_t s);

}  // namespace mtb
