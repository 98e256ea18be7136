// host.h -- host-side helpers shared by the launcher translation units
// (medtree_b200.cu: dispatch + C ABI; run_colhist.cu, run_ctmf.cu: kernel
// families with many template instantiations, compiled in parallel).
#pragma once
#include <atomic>
#include <cstdint>
#include <string>

#include "../../include/medtree_b200.h"
#include "common.cuh"

namespace mtb {

extern thread_local std::string g_err;
extern thread_local const char *g_kernel;
extern std::atomic<uint64_t> g_launches;

int fail(int code, const std::string &msg);
int sm_count();
int rows_per_cta(const SlabParams &p, int blocks_x, int B, int ctas_per_sm);
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

// kernel families in their own translation units
int run_colhist_u8(SlabParams p, int B, cudaStream_t s);
int run_colhist4_256(SlabParams p, int B, cudaStream_t s);
int run_colhist4p_256(SlabParams p, int B, cudaStream_t s, int pl);
// wk: window-keyed first sweep (pays off on compact data, see kernel)
int run_colhist16_u16(SlabParams p, int B, cudaStream_t s, bool wk = true);
int run_colhist16s_u16(SlabParams p, int B, cudaStream_t s);
int run_ctmf_u8(SlabParams p, int B, cudaStream_t s);
int run_lob_u8_32(SlabParams p, int B, cudaStream_t s);

}  // namespace mtb
