// run_bandtc.cu -- launcher of the tcgen05 band-matrix kernel (kernels_bandtc.cuh).
#include <algorithm>

#include "host.h"
#include "kernels_bandtc.cuh"

namespace mtb {

// four 128-pixel tiles fit one SM at every radius; the band tiles (8 columns per k-step) and the
// accumulators (NF columns per tile) fit tensor memory
static_assert(bt_smem(512, 127, 32) <= 227 * 1024 - 256 && bt_smem(512, 127, 64) <= 227 * 1024 - 256, "planes at r = 127");
static_assert(BT_ACOL0 + 8 * bt_nka(127) <= BT_TMEM_COLS && BT_MAXTILES * 64 <= BT_ACOL0, "tensor-memory columns");

template <int NF>
static int run_bandtc_nf(SlabParams p, int B, cudaStream_t s) {
    const int r = p.radius;
    // stripe width: 128-pixel tiles, as many (up to 4) as the planes leave room for
    const size_t smem_max = 227 * 1024 - 256;
    int mt = 1;
    for (int t = 1; t <= BT_MAXTILES; ++t)
        if (bt_smem(BT_M * t, r, NF) <= smem_max) mt = t;
    mt = std::min(mt, std::max(1, env_int("MTB_BT_TILES", mt)));
    const int stripes_max = (p.W + BT_M * mt - 1) / (BT_M * mt);
    // even the tiles out over the stripes the image needs
    const int tiles_total = (p.W + BT_M - 1) / BT_M;
    mt = (tiles_total + stripes_max - 1) / stripes_max;
    const int TW = BT_M * mt;
    const size_t smem = bt_smem(TW, r, NF);
    if (smem > smem_max) return fail(MTB_E_INVAL, "k_bandtc_u8: radius too large for shared memory");
    auto kern = p.in_rows ? k_bandtc_u8<NF, true> : k_bandtc_u8<NF, false>;
    if (int rc = set_smem(kern, smem)) return rc;
    const int bx = (p.W + TW - 1) / TW, rows = p.row_end - p.row_begin;
    // row slabs: one whole round of CTAs (one per SM)
    int64_t slabs = (int64_t)sm_count() * env_int("MTB_BT_WAVES", 1) / ((int64_t)bx * B);
    slabs = std::max<int64_t>(1, std::min<int64_t>(slabs, rows));
    int rpc = (int)((rows + slabs - 1) / slabs);
    rpc = std::max(rpc, std::min(rows, r / 2 + 8));
    p.rows_per_cta = rpc;
    dim3 grid(bx, (rows + rpc - 1) / rpc, B);
    kern<<<grid, 2 * TW, smem, s>>>(p, TW);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(MTB_E_CUDA, std::string("k_bandtc_u8: ") + cudaGetErrorString(e));
    g_kernel = NF == 32 ? "k_bandtc_u8<32>" : "k_bandtc_u8<64>";
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return MTB_OK;
}

// 8-bit, 1 <= r <= 127, any rank.  Four coarse bins per keyed window below
// r = 48 (the median of a smaller window varies more along 128 pixels), two above.
int run_bandtc_u8(SlabParams p, int B, cudaStream_t s) {
    const int nf = env_int("MTB_BT_NF", p.radius >= 48 ? 32 : 64);
    return nf == 32 ? run_bandtc_nf<32>(p, B, s) : run_bandtc_nf<64>(p, B, s);
}

}  // namespace mtb
