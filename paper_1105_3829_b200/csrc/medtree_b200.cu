// medtree_b200.cu -- C ABI (include/medtree_b200.h) and kernel dispatch.
//
// The host side only validates, picks a kernel variant and a grid, and
// launches; there is no CPU compute path and no fallback: a missing device
// or a launch failure is reported as an error.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "host.h"
#include "kernels_vert.cuh"
#include "kernels_sortnet.cuh"
#include "kernels_med3.cuh"
#include "kernels_mednet.cuh"
#include "kernels_select.cuh"
#include <cstdlib>
#if defined(__x86_64__) || defined(_M_X64)
#include <emmintrin.h>
#define MTB_HAVE_SSE2 1
#endif

namespace mtb {

// Spread of the 16-bit value distribution over a strided sample of the source
// rows: out[0] = number of distinct coarse keys, out[1] = the key shift s
// (key = min(v >> s, 255)).  With s = 8 the key is the high byte: a wide
// spread (> SPREAD_WIDE distinct keys: the key of the median changes from
// pixel to pixel) goes to the candidate-bucket path, a compact one to the
// two-phase k_colhist16_u16.  Data whose top bits are empty (10- / 12- /
// 14-bit samples in 16-bit words: compact, or coarsely spread, by its high
// bytes) is looked at again with s = the bits the largest sample needs
// beyond 8: if the keys are then
// widely spread AND flat (no key holds more than 1/64 of the sample, against
// 1/256 on uniformly spread data), the candidate-bucket path takes it with that shift.
// out[2] = 1 when the sample is peaked (see below): compact AND peaked data takes
// the window-key pass instead of the two-phase kernel.
// Every choice is exact; it only decides the speed.
constexpr int SPREAD_SAMPLES = 1 << 14;
constexpr int SPREAD_FLAT_MAX = SPREAD_SAMPLES / 64;

constexpr int SPREAD_THREADS = 1024;

__global__ void __launch_bounds__(SPREAD_THREADS) k_highbyte_spread(const uint16_t *src, int64_t pitch, int rows, int W,
                                                                    int64_t img_stride, int B, int allow_shift, int *out) {
    __shared__ uint16_t smp[SPREAD_SAMPLES];  // the sample, read once
    __shared__ int hist[256];
    __shared__ int vmax, res[2], med[3], inwin;
    const int tid = threadIdx.x;
    // distinct / fullest of the 256 keys min(v >> s, 255) -> res[0], res[1]
    auto keys = [&](int s) {
        if (tid < 256) hist[tid] = 0;
        __syncthreads();
        for (int i = tid; i < SPREAD_SAMPLES; i += SPREAD_THREADS) atomicAdd(hist + min((unsigned)smp[i] >> s, 255u), 1);
        __syncthreads();
        if (tid < 32) {
            int d = 0, m = 0;
            for (int b = tid; b < 256; b += 32) {
                d += hist[b] ? 1 : 0;
                m = max(m, hist[b]);
            }
            d = __reduce_add_sync(0xffffffffu, d);
            m = __reduce_max_sync(0xffffffffu, m);
            if (tid == 0) res[0] = d, res[1] = m;
        }
        __syncthreads();
    };
    if (tid == 0) vmax = 0;
    __syncthreads();
    int mx = 0;
    for (int i = tid; i < SPREAD_SAMPLES; i += SPREAD_THREADS) {
        const int y = (int)(((int64_t)i * 7919) % rows);
        const int x = (int)(((int64_t)i * 104729) % W);
        const int b = B > 1 ? i % B : 0;
        const uint16_t v = src[b * img_stride + (int64_t)y * pitch + x];
        smp[i] = v;
        mx = max(mx, (int)v);
    }
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((tid & 31) == 0) atomicMax(&vmax, mx);
    keys(8);  // (its barriers also order smp and vmax)
    int d = res[0], sh = 8;
    // out[2]: is the sample peaked -- do at least 2 in 5 of its values lie in the 254-value window
    // around its median?  (Then most window medians do, and compact data goes through the
    // window-key pass, run_wk16_u16.)  The median: its high byte from the counts just taken, its
    // low byte from the counts of the low bytes under that high byte.
    if (tid == 0) {
        int acc = 0, h = 0;
        for (; h < 255; ++h) {
            if (acc + hist[h] >= SPREAD_SAMPLES / 2) break;
            acc += hist[h];
        }
        med[0] = h;
        med[1] = acc;
        inwin = 0;
    }
    __syncthreads();
    if (tid < 256) hist[tid] = 0;
    __syncthreads();
    for (int i = tid; i < SPREAD_SAMPLES; i += SPREAD_THREADS)
        if ((smp[i] >> 8) == med[0]) atomicAdd(hist + (smp[i] & 255), 1);
    __syncthreads();
    if (tid == 0) {
        int acc = med[1], l = 0;
        for (; l < 255; ++l) {
            if (acc + hist[l] >= SPREAD_SAMPLES / 2) break;
            acc += hist[l];
        }
        med[2] = med[0] * 256 + l;
    }
    __syncthreads();
    {
        const unsigned lo = (unsigned)max(med[2] - 127, 0);
        int c = 0;
        for (int i = tid; i < SPREAD_SAMPLES; i += SPREAD_THREADS) c += ((unsigned)smp[i] - lo <= 253u) ? 1 : 0;
        c = __reduce_add_sync(0xffffffffu, c);
        if ((tid & 31) == 0) atomicAdd(&inwin, c);
    }
    __syncthreads();
    const int peaked = 5 * inwin >= 2 * SPREAD_SAMPLES ? 1 : 0;
    int s = 0;
    while (s < 8 && (vmax >> s) > 255) ++s;
    if (allow_shift && s < 8) {  // (uniform: all from shared memory)
        __syncthreads();
        keys(s);
        if (res[0] > SPREAD_WIDE && res[1] <= SPREAD_FLAT_MAX) d = res[0], sh = s;
    }
    if (tid == 0) {
        out[0] = d;
        out[1] = sh;
        out[2] = peaked;
    }
}

thread_local std::string g_err;
thread_local const char *g_kernel = "";
std::atomic<uint64_t> g_launches{0};

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev];
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (dev >= 0 && dev < 64) cached[dev] = n;
    return n;
}

// validation.py:19-29 (window), :32-47 (rank); engine.py:252-256 (slab rows)
static int validate(const SlabParams &p, int B) {
    if (!p.src || !p.dst) return fail(MTB_E_INVAL, "null src/dst pointer");
    if (p.H < 1 || p.W < 1) return fail(MTB_E_INVAL, "pixels must be a non-empty 2D array");
    if (B < 1) return fail(MTB_E_INVAL, "batch must be >= 1");
    if (p.radius < 1)
        return fail(MTB_E_INVAL, "window must be an odd integer >= 3, got " +
                                     std::to_string(2 * (int64_t)p.radius + 1));
    const int64_t n = 2 * (int64_t)p.radius + 1;
    const int64_t lim = 2 * (int64_t)(p.W < p.H ? p.W : p.H) + 1;
    if (n > lim)
        return fail(MTB_E_INVAL, "window " + std::to_string(n) + " too large for a " +
                                     std::to_string(p.W) + "x" + std::to_string(p.H) +
                                     " image (limit " + std::to_string(lim) + ")");
    if (n * n > 0xFFFFFFFFll) return fail(MTB_E_INVAL, "window area exceeds 2^32");
    if (p.rank < 1 || (int64_t)p.rank > n * n)
        return fail(MTB_E_INVAL, "rank " + std::to_string(p.rank) + " outside [1, " +
                                     std::to_string(n * n) + "] for window " + std::to_string(n));
    if (p.row_begin < 0 || p.row_end > p.H || p.row_begin > p.row_end)
        return fail(MTB_E_INVAL, "bad output row range");
    if (p.src_pitch < p.W || p.dst_pitch < p.W) return fail(MTB_E_INVAL, "pitch < width");
    if (p.row_begin < p.row_end) {
        const int64_t need0 = p.row_begin - p.radius < 0 ? 0 : p.row_begin - p.radius;
        const int64_t need1 = p.row_end + p.radius > p.H ? p.H : p.row_end + p.radius;
        if (p.src_row0 > need0 || (int64_t)p.src_row0 + p.src_rows < need1)
            return fail(MTB_E_INVAL, "source rows [" + std::to_string(p.src_row0) + ", " +
                                         std::to_string((int64_t)p.src_row0 + p.src_rows) +
                                         ") do not cover the halo [" + std::to_string(need0) +
                                         ", " + std::to_string(need1) + ")");
    }
    return MTB_OK;
}

int rows_per_cta(const SlabParams &p, int blocks_x, int B, int ctas_per_sm, int waves) {
    const int rows = p.row_end - p.row_begin;
    const int64_t target = (int64_t)sm_count() * ctas_per_sm * waves;
    int64_t slabs = (target + (int64_t)blocks_x * B - 1) / ((int64_t)blocks_x * B);
    if (slabs < 1) slabs = 1;
    int rpc = (int)((rows + slabs - 1) / slabs);
    const int n = 2 * p.radius + 1;
    // keep the n^2 window build below ~2x the per-row update work
    int min_rows = n / 2 + 1;
    if (rpc < min_rows) rpc = min_rows;
    if (rpc > rows) rpc = rows;
    return rpc < 1 ? 1 : rpc;
}

int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return (v && *v) ? atoi(v) : dflt;
}

// kernel choice: MTB_KERNEL=vert|ctmf forces a family (testing/tuning)
const char *forced_kernel() {
    const char *v = getenv("MTB_KERNEL");
    return v ? v : "";
}

// keep freed stream-ordered allocations in the device's default pool so the
// per-launch workspace does not go back to the driver at every sync
void keep_pool_memory() {
    static int done[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = 4ull << 30;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[dev] = 1;
}






template <int N, int K, int RT, typename P>
static int run_sortnet_n(SlabParams p, int B, cudaStream_t s, const char *name) {
    constexpr int TX = 32 * 2 * K, TY = 4 * RT;
    const int rows = p.row_end - p.row_begin;
    dim3 grid((p.W + TX - 1) / TX, (rows + TY - 1) / TY, B);
    k_sortnet<N, K, RT, P><<<grid, dim3(32, 4), 0, s>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(MTB_E_CUDA, std::string(name) + ": " + cudaGetErrorString(e));
    g_kernel = name;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return MTB_OK;
}

// 3x3 median of 8-bit frames (k_med3_u8): row bands sized so the grid is
// one wave of resident CTAs
// TMA-staged variant: 16-byte aligned rows, W % 16 == 0; bands sized for
// one wave (the whole frame is requested at launch)
static int run_med3t(SlabParams p, int B, cudaStream_t s) {
    const int rows = p.row_end - p.row_begin;
    const int bx = (p.W + 1023) / 1024;
    const int per_sm = 8;
    const int64_t slots = (int64_t)sm_count() * per_sm;
    int64_t bands = slots / ((int64_t)bx * B);
    if (bands < 1) bands = 1;
    int rt = (int)((rows + bands - 1) / bands);
    rt = std::max(rt, env_int("MTB_MED3_MIN_RT", 8));
    rt = std::min(rt, std::min(rows, 190));  // (rt + 2) rows of 1056 B + barriers <= 200 KB
    p.rows_per_cta = rt;
    const size_t smem = (size_t)(((rt + 2) * 8 + 127) & ~127) + (size_t)(rt + 2) * M3T_SEG;
    dim3 grid(bx, (rows + rt - 1) / rt, B);
    return launch(k_med3t_u8, grid, 128, smem, s, p, "k_med3t_u8");
}

static bool med3t_applies(const SlabParams &p, int B) {
    const auto a16 = [](uintptr_t v) { return (v & 15) == 0; };
    return p.W % 16 == 0 && a16((uintptr_t)p.src) && a16((uintptr_t)p.dst) && a16((uintptr_t)p.src_pitch) &&
           a16((uintptr_t)p.dst_pitch) &&
           (B == 1 || (a16((uintptr_t)p.src_img_stride) && a16((uintptr_t)p.dst_img_stride))) &&
           env_int("MTB_MED3T", 1) != 0;
}

static int run_med3(SlabParams p, int B, cudaStream_t s) {
    if (med3t_applies(p, B)) return run_med3t(p, B, s);
    const int rows = p.row_end - p.row_begin;
    const int bx = (p.W + 1023) / 1024;
    int per_sm = 4;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_med3_u8, 128, 0);
    if (per_sm < 1) per_sm = 1;
    const int64_t slots = (int64_t)sm_count() * per_sm;
    int64_t bands = slots / ((int64_t)bx * B);
    if (bands < 1) bands = 1;
    int rt = (int)((rows + bands - 1) / bands);
    const int min_rt = env_int("MTB_MED3_MIN_RT", 8);
    if (rt < min_rt) rt = min_rt;
    if (rt > rows) rt = rows;
    p.rows_per_cta = rt;
    dim3 grid(bx, (rows + rt - 1) / rt, B);
    return launch(k_med3_u8, grid, 128, 0, s, p, "k_med3_u8");
}

// n = 5, 7 medians from sorted packed columns with merge sharing (k_mednet)
template <int N, typename P>
static int run_mednet(SlabParams p, int B, cudaStream_t s, const char *name) {
    const size_t smem = (size_t)mn_smem(N);
    auto kern = k_mednet<N, P>;
    if (int rc = set_smem(kern, smem)) return rc;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, MN_T, smem);
    if (per_sm < 1) per_sm = 1;
    const int rows = p.row_end - p.row_begin;
    const int bx = (p.W + MN_TX - 1) / MN_TX;
    const int64_t slots = (int64_t)sm_count() * per_sm * 2;
    int64_t bands = slots / ((int64_t)bx * B);
    if (bands < 1) bands = 1;
    int rt = (int)((rows + bands - 1) / bands);
    rt = std::max(rt, env_int("MTB_MN_MIN_RT", 16));
    rt = (rt + 1) & ~1;  // two output rows per step
    if (rt > rows) rt = rows;
    p.rows_per_cta = rt;
    dim3 grid(bx, (rows + rt - 1) / rt, B);
    return launch(kern, grid, MN_T, smem, s, p, name);
}

// small medians: r = 1 (8-bit) -> 3x3 kernels; r = 2, 3 -> sorted packed
// columns with shared merges; r = 1 (16-bit) -> selection network
template <typename P>
static int run_sortnet(SlabParams p, int B, cudaStream_t s) {
    const std::string force = forced_kernel();
    if (p.radius == 2) return run_mednet<5, P>(p, B, s, sizeof(P) == 1 ? "k_mednet<5,u8>" : "k_mednet<5,u16>");
    if (p.radius == 3) return run_mednet<7, P>(p, B, s, sizeof(P) == 1 ? "k_mednet<7,u8>" : "k_mednet<7,u16>");
    if (sizeof(P) == 1 && force != "sortnet" && (int64_t)p.src_rows * p.src_pitch < (1ll << 31))
        return run_med3(p, B, s);
    return run_sortnet_n<3, 4, 8, P>(p, B, s, "k_sortnet<3>");
}

// 16-bit kernel choice by the spread of the value distribution (distinct
// high bytes among 2^14 sampled pixels, k_highbyte_spread): a wide spread
// favours the sorted-column low byte of k_colhist16s_u16 (r <= 16), a
// compact one the window-keyed two-phase k_colhist16_u16.  Both are exact;
// the choice only changes speed.  Host paths that hold the frame on the
// host sample it there (g_spread_hint); device-resident calls sample on the
// device and let the kernels read the result (SlabParams::spread / gate):
// no host synchronisation, stream-ordered scratch, graph-capturable.
static thread_local int g_spread_hint = -1;

static thread_local int g_shift_hint = 8;
static thread_local int g_peaked_hint = 0;

// the same on a host frame: returns the distinct-key count, sets g_shift_hint
static int spread_distinct_host(const uint16_t *src, int64_t pitch, int rows, int W) {
    auto sample = [&](int i) -> unsigned {
        const int y = (int)(((int64_t)i * 7919) % rows);
        const int x = (int)(((int64_t)i * 104729) % W);
        return src[(int64_t)y * pitch + x];
    };
    // (the frame is sampled once: 2^14 scattered host reads are the cost of this probe)
    static thread_local std::vector<uint16_t> all(SPREAD_SAMPLES), tmp(SPREAD_SAMPLES);
    unsigned vmax = 0;
    for (int i = 0; i < SPREAD_SAMPLES; ++i) {
        all[i] = (uint16_t)sample(i);
        vmax = std::max(vmax, (unsigned)all[i]);
    }
    auto keys = [&](int s, int &distinct, int &fullest) {
        int hist[256] = {};
        for (int i = 0; i < SPREAD_SAMPLES; ++i) ++hist[std::min((unsigned)all[i] >> s, 255u)];
        distinct = fullest = 0;
        for (int b = 0; b < 256; ++b) {
            distinct += hist[b] ? 1 : 0;
            fullest = std::max(fullest, hist[b]);
        }
    };
    {  // peaked: at least 2 in 5 sampled values in the 254-value window around the sample's median
        tmp = all;
        std::nth_element(tmp.begin(), tmp.begin() + SPREAD_SAMPLES / 2 - 1, tmp.end());
        const unsigned lo = (unsigned)std::max((int)tmp[SPREAD_SAMPLES / 2 - 1] - 127, 0);
        int in = 0;
        for (uint16_t v : all) in += ((unsigned)v - lo <= 253u) ? 1 : 0;
        g_peaked_hint = 5 * in >= 2 * SPREAD_SAMPLES ? 1 : 0;
    }
    int d8, m8;
    keys(8, d8, m8);
    int s = 0;
    while (s < 8 && (vmax >> s) > 255) ++s;
    g_shift_hint = 8;
    if (s < 8) {
        int ds, ms;
        keys(s, ds, ms);
        if (ds > SPREAD_WIDE && ms <= SPREAD_FLAT_MAX) {
            g_shift_hint = s;
            return ds;
        }
    }
    return d8;
}

static int run_u16_colhist(SlabParams p, int B, cudaStream_t s) {
    const std::string force = forced_kernel();
    if (force == "colhist") return run_colhist16_u16(p, B, s, 1);
    if (force == "colhist16s") return run_colhist16s_u16(p, B, s);
    if (force == "colhist16c") return run_colhist16c_u16(p, B, s);
    if (force == "lowsel") return run_lowsel16_u16(p, B, s);
    if (force == "wk16") return run_wk16_u16(p, B, s);
    // widely spread data: the candidate-list path where it applies (r = 3..63, not the streaming
    // launch; MTB_U16_LIST=0 for comparison), else the candidate-run kernel up to r = 23, else the
    // two-phase kernel without the window-keyed sweep
    const bool list = lowsel16_applies(p) && env_int("MTB_U16_LIST", 1) != 0;
    const bool small_r = p.radius <= env_int("MTB_U16C_MAX_R", 23);
    // compact and peaked data, r >= 40: the window-key pass (same launches as the candidate-bucket
    // path).  Config 4 (8192^2), two-phase kernel / window-key pass + two-phase on the flagged
    // tiles: r = 15 1.97 / 2.35 ms, r = 31 2.91 / 3.33, r = 47 9.75 / 5.78, r = 63 12.0 / 8.86 --
    // below r = 40 the two-phase kernel's window-keyed sweep is the faster form of the same idea
    // (the pass's misses sit along the clamped borders, and redoing those 256-column tiles costs
    // more than it saves).  MTB_U16_WK8=0 / 1: never / from r = 3.
    const int wk8_mode = env_int("MTB_U16_WK8", -1);
    const bool wk8 = lowsel16_applies(p) && (wk8_mode < 0 ? p.radius >= 40 : wk8_mode != 0);
    auto run_wide = [&](const SlabParams &q) {
        return list ? run_lowsel16_u16(q, B, s) : (small_r ? run_colhist16c_u16(q, B, s) : run_colhist16_u16(q, B, s, 0));
    };
    if (g_spread_hint >= 0) {
        if (g_spread_hint <= SPREAD_WIDE) return (wk8 && g_peaked_hint) ? run_wk16_u16(p, B, s) : run_colhist16_u16(p, B, s, 1);
        p.key_down = list ? 8 - g_shift_hint : 0;
        // (a shifted key only helps the candidate-bucket path: the other kernels split at the high byte)
        if (!list && g_shift_hint != 8) return run_colhist16_u16(p, B, s, 1);
        return run_wide(p);
    }
    int *d_spread = nullptr;
    keep_pool_memory();
    if (cudaMallocAsync(reinterpret_cast<void **>(&d_spread), 3 * sizeof(int), s) != cudaSuccess)
        return fail(MTB_E_CUDA, "k_highbyte_spread: scratch allocation failed");
    k_highbyte_spread<<<1, SPREAD_THREADS, 0, s>>>(static_cast<const uint16_t *>(p.src), p.src_pitch, p.src_rows, p.W,
                                        p.src_img_stride, B, list ? 1 : 0, d_spread);
    cudaError_t e = cudaGetLastError();
    int rc = e == cudaSuccess ? MTB_OK : fail(MTB_E_CUDA, std::string("k_highbyte_spread: ") + cudaGetErrorString(e));
    if (!rc) g_launches.fetch_add(1, std::memory_order_relaxed);
    p.spread = d_spread;
    if (!rc) {
        p.gate = GATE_WIDE;  // these launches exit at once unless the data is widely spread
        rc = run_wide(p);
        p.gate = GATE_COMPACT;  // compact data: the window-key pass (where the sample is peaked: spread[2])
        if (!rc) rc = wk8 ? run_wk16_u16(p, B, s) : run_colhist16_u16(p, B, s, 1);  // and the two-phase kernel
        if (!rc)
            g_kernel = list && wk8 ? "k_lowsel_u16|k_colhist4p_u8<u16 window key>|k_colhist16_u16 (device-selected)"
                       : list      ? "k_lowsel_u16|k_colhist16_u16 (device-selected)"
                       : small_r   ? "k_colhist16c_u16|k_colhist16_u16 (device-selected)"
                                   : "k_colhist16_u16 (device-selected)";
    }
    cudaFreeAsync(d_spread, s);
    return rc;
}

// smallest radius sent to k_bandmma_u8 (config 2: 0.51 ms at r = 31 against 0.50 for the pair
// records, 0.47 against 0.71 at r = 40)
constexpr int BANDMMA_MIN_R = 32;
// smallest radius sent to the tcgen05 kernel k_bandtc_u8 (config 2: 0.58 ms against 0.63 for
// k_bandmma_u8 at r = 80, 0.58 against 0.77 at r = 127; 0.59 against 0.54 at r = 72)
constexpr int BANDTC_MIN_R = 76;
// ... and only for launches of at least this many output pixels: its one round of wide CTAs leaves
// SMs idle on small frames (r = 80: 1080p 0.175 ms against 0.133 for k_bandmma_u8, 1024^2 0.165
// against 0.112; 2048^2 0.183 against 0.239 -- tools/small_frames.py)
constexpr int64_t BANDTC_MIN_PIXELS = 3 << 20;

template <typename P>
static int run(SlabParams p, int B, cudaStream_t s) {
    int rc = validate(p, B);
    if (rc) return rc;
    if (p.row_begin == p.row_end) return MTB_OK;
    const int64_t n = 2 * (int64_t)p.radius + 1;
    const bool wide = n * n > 65535;
    const std::string force = forced_kernel();
    // Kernel choice (measured on B200, tools/probe.py):
    //   median, r = 1 (8-bit)                     -> 3x3 kernels (k_med3t / k_med3)
    //   median, r = 2, 3                          -> sorted packed columns + shared merges (k_mednet)
    //   median, r = 1 (16-bit)                    -> selection network (k_sortnet<3>)
    //   8-bit, r < 32 (any rank)                  -> column-histogram gather
    //   8-bit, 32 <= r <= 75                      -> band-matrix products on the tensor cores, mma.sync (k_bandmma_u8)
    //   8-bit, 76 <= r <= 127, >= 3 Mpixel launches  -> the same with tcgen05.mma / tensor memory (k_bandtc_u8)
    //   (CTMF tiles, O(1) in r: MTB_KERNEL=ctmf only -- superseded by k_bandmma_u8)
    //   16-bit, n <= 255                          -> column histograms (two kernels, by value spread)
    //   otherwise (n > 255)                       -> per-column vertical histograms
    // MTB_KERNEL forces a family (tests).
    const bool median = (uint32_t)((n * n + 1) / 2) == p.rank;
    if (median && n <= 7 && (force.empty() || force == "sortnet" || force == "med3" || force == "mednet"))
        return run_sortnet<P>(p, B, s);
    if (sizeof(P) == 1 && n <= 255 && (force == "colhist" || (force.empty() && p.radius < BANDMMA_MIN_R)))
        return run_colhist_u8(p, B, s);
    if (sizeof(P) == 1 && n <= 255 && p.radius >= 1 &&
        (force == "bandtc" || (force.empty() && p.radius >= BANDTC_MIN_R &&
                               (int64_t)(p.row_end - p.row_begin) * p.W * B >= BANDTC_MIN_PIXELS)))
        return run_bandtc_u8(p, B, s);
    if (sizeof(P) == 1 && n <= 255 && p.radius >= 1 && (force == "bandmma" || force.empty()))
        return run_bandmma_u8(p, B, s);
    if (sizeof(P) == 1 && !wide && force == "ctmf") return run_ctmf_u8(p, B, s);
    if (sizeof(P) == 2 && n <= 255 && force != "vert") return run_u16_colhist(p, B, s);
    if (sizeof(P) == 1) {
        constexpr int T = 128;
        const int bx = (p.W + T - 1) / T;
        const size_t smem = (size_t)(16 + 256) * T * (wide ? 4 : 2);
        p.rows_per_cta = rows_per_cta(p, bx, B, wide ? 1 : 3);
        dim3 grid(bx, (p.row_end - p.row_begin + p.rows_per_cta - 1) / p.rows_per_cta, B);
        return wide ? launch(k_vert_u8<uint32_t, T>, grid, T, smem, s, p, "k_vert_u8<u32>")
                    : launch(k_vert_u8<uint16_t, T>, grid, T, smem, s, p, "k_vert_u8<u16>");
    }
    constexpr int T = 64;
    const int bx = (p.W + T - 1) / T;
    const size_t smem = (size_t)2 * (16 + 256) * T * (wide ? 4 : 2);
    p.rows_per_cta = rows_per_cta(p, bx, B, wide ? 1 : 3);
    dim3 grid(bx, (p.row_end - p.row_begin + p.rows_per_cta - 1) / p.rows_per_cta, B);
    return wide ? launch(k_vert_u16<uint32_t, T>, grid, T, smem, s, p, "k_vert_u16<u32>")
                : launch(k_vert_u16<uint16_t, T>, grid, T, smem, s, p, "k_vert_u16<u16>");
}

static SlabParams make_params(const void *src, int64_t src_pitch, int32_t src_row0,
                              int32_t src_rows, void *dst, int64_t dst_pitch, int32_t H,
                              int32_t W, int32_t row_begin, int32_t row_end, int32_t radius,
                              int64_t rank, const void *lut) {
    SlabParams p{};
    p.src = src;
    p.src_pitch = src_pitch;
    p.src_img_stride = 0;
    p.src_row0 = src_row0;
    p.src_rows = src_rows;
    p.dst = dst;
    p.dst_pitch = dst_pitch;
    p.dst_img_stride = 0;
    p.H = H;
    p.W = W;
    p.row_begin = row_begin;
    p.row_end = row_end;
    p.radius = radius;
    p.rank = (rank < 1 || rank > 0xFFFFFFFFll) ? 0u : (uint32_t)rank;
    p.lut = lut;
    return p;
}

}  // namespace mtb

using namespace mtb;

// ---------------------------------------------------------------------------
// Host-buffer path (mtb_filter_host): the frame is cut into row bands; band
// i's source rows go host->device on a copy stream, its filter launch waits
// only for the rows it reads (band + r halo rows), and its result rows go
// device->host on a second copy stream -- so the copies of one band overlap
// the filtering of its neighbours.  Device buffers and streams are kept per
// device between calls (the pool grows, never shrinks).
// Host memcpy workers for pageable frames: the drop-in filter_image gets
// the caller's pageable numpy array, whose copies the driver would stage
// through its own bounce buffer at one host thread's memcpy speed.  The
// host paths instead copy pageable rows into page-locked staging buffers
// with P threads (the calling thread included), so host memcpy, PCIe and
// the kernels overlap band by band (host_pipeline).  Persistent workers,
// one pool per device context; never destroyed (process exit reclaims).
// Staging copy between a pageable frame and a page-locked buffer with
// non-temporal stores: the destination is either read next by the DMA engine
// (from DRAM) or is the caller's result frame, so filling the cache with it
// (and reading the lines first, as plain stores do) only costs memory
// bandwidth -- the host memcpy is the slowest stage of the pageable path.
// MTB_COPY_NT=0: plain memcpy.
static void stage_copy(char *d, const char *s, size_t n) {
#ifdef MTB_HAVE_SSE2
    static const bool nt = env_int("MTB_COPY_NT", 1) != 0;
    if (nt && n >= 4096) {
        const size_t head = (16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15;
        memcpy(d, s, head);
        d += head, s += head, n -= head;
        size_t i = 0;
        for (; i + 64 <= n; i += 64) {
            const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i));
            const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i + 16));
            const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i + 32));
            const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i + 48));
            _mm_stream_si128(reinterpret_cast<__m128i *>(d + i), a);
            _mm_stream_si128(reinterpret_cast<__m128i *>(d + i + 16), b);
            _mm_stream_si128(reinterpret_cast<__m128i *>(d + i + 32), c);
            _mm_stream_si128(reinterpret_cast<__m128i *>(d + i + 48), e);
        }
        _mm_sfence();
        memcpy(d + i, s + i, n - i);
        return;
    }
#endif
    memcpy(d, s, n);
}

struct CopyPool {
    std::mutex mu;
    std::condition_variable cv, cv_done;
    char *d = nullptr;
    const char *s = nullptr;
    size_t n = 0, piece = 0;
    int pieces = 0, done = 0, P = 1;
    std::atomic<int> next{0};
    uint64_t gen = 0;

    void start(int threads) {
        P = std::max(1, threads);
        for (int i = 1; i < P; ++i)
            std::thread([this] {
                uint64_t seen = 0;
                for (;;) {
                    {
                        std::unique_lock<std::mutex> lk(mu);
                        cv.wait(lk, [&] { return gen != seen; });
                        seen = gen;
                    }
                    work();
                }
            }).detach();
    }
    void work() {
        for (;;) {
            const int i = next.fetch_add(1);
            if (i >= pieces) return;
            const size_t o = (size_t)i * piece, l = std::min(piece, n - o);
            stage_copy(d + o, s + o, l);
            std::lock_guard<std::mutex> lk(mu);
            if (++done == pieces) cv_done.notify_all();
        }
    }
    void copy(void *dst, const void *src, size_t len) {
        if (len < (1u << 20) || P <= 1) {
            stage_copy(static_cast<char *>(dst), static_cast<const char *>(src), len);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(mu);
            d = static_cast<char *>(dst);
            s = static_cast<const char *>(src);
            n = len;
            pieces = 2 * P;
            piece = (((len + pieces - 1) / pieces) + 4095) & ~(size_t)4095;
            pieces = (int)((len + piece - 1) / piece);
            done = 0;
            next.store(0);
            ++gen;
        }
        cv.notify_all();
        work();
        std::unique_lock<std::mutex> lk(mu);
        cv_done.wait(lk, [&] { return done == pieces; });
    }
};

struct HostCtx {
    int dev = -1;
    void *dsrc = nullptr, *ddst = nullptr, *dlut = nullptr;
    unsigned int *dflags = nullptr;  // [0] rows arrived, [1..] output pixels per chunk
    unsigned int *hstatus = nullptr, *dstatus = nullptr;  // mapped pinned word: a CTA timed out waiting for rows
    size_t cap = 0;
    void *hin = nullptr, *hout = nullptr;  // page-locked staging for pageable frames
    size_t hcap = 0;
    CopyPool *pool = nullptr;
    cudaStream_t sh = nullptr, sc = nullptr, sd = nullptr;
    static constexpr int KMAX = 16;
    cudaEvent_t eh[KMAX], ec[KMAX], eo[KMAX];
};

static int host_staging(HostCtx *ctx, size_t bytes) {
    if (!ctx->pool) {
        const unsigned hw = std::thread::hardware_concurrency();
        ctx->pool = new CopyPool();
        ctx->pool->start(env_int("MTB_COPY_THREADS", (int)std::min(8u, std::max(1u, hw / 2))));
    }
    if (ctx->hcap >= bytes) return MTB_OK;
    if (ctx->hin) cudaFreeHost(ctx->hin);
    if (ctx->hout) cudaFreeHost(ctx->hout);
    ctx->hin = ctx->hout = nullptr;
    ctx->hcap = 0;
    cudaError_t e = cudaHostAlloc(&ctx->hin, bytes, cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaHostAlloc(&ctx->hout, bytes, cudaHostAllocDefault);
    if (e != cudaSuccess) return fail(MTB_E_CUDA, std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
    ctx->hcap = bytes;
    return MTB_OK;
}

// one context (and one lock) per device: host threads driving different
// GPUs never serialise on each other
static std::mutex g_host_mu[64];
static HostCtx g_host[64];

static int host_ctx(HostCtx *&ctx, std::unique_lock<std::mutex> &lock, size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return fail(MTB_E_CUDA, "device index out of range");
    lock = std::unique_lock<std::mutex>(g_host_mu[dev]);
    ctx = &g_host[dev];
    auto ok = [](cudaError_t e, const char *what) {
        if (e != cudaSuccess) {
            fail(MTB_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
            return false;
        }
        return true;
    };
    if (ctx->dev < 0) {
        if (!ok(cudaStreamCreateWithFlags(&ctx->sh, cudaStreamNonBlocking), "cudaStreamCreate") ||
            !ok(cudaStreamCreateWithFlags(&ctx->sc, cudaStreamNonBlocking), "cudaStreamCreate") ||
            !ok(cudaStreamCreateWithFlags(&ctx->sd, cudaStreamNonBlocking), "cudaStreamCreate") ||
            !ok(cudaMalloc(&ctx->dlut, 65536 * 2), "cudaMalloc") ||
            !ok(cudaMalloc(&ctx->dflags, 64 * sizeof(unsigned int)), "cudaMalloc") ||
            !ok(cudaHostAlloc(&ctx->hstatus, sizeof(unsigned int), cudaHostAllocMapped), "cudaHostAlloc") ||
            !ok(cudaHostGetDevicePointer(&ctx->dstatus, ctx->hstatus, 0), "cudaHostGetDevicePointer"))
            return MTB_E_CUDA;
        for (int i = 0; i < HostCtx::KMAX; ++i)
            if (!ok(cudaEventCreateWithFlags(&ctx->eh[i], cudaEventDisableTiming), "cudaEventCreate") ||
                !ok(cudaEventCreateWithFlags(&ctx->ec[i], cudaEventDisableTiming), "cudaEventCreate") ||
                !ok(cudaEventCreateWithFlags(&ctx->eo[i], cudaEventDisableTiming), "cudaEventCreate"))
                return MTB_E_CUDA;
        ctx->dev = dev;
    }
    if (ctx->cap < bytes) {
        cudaDeviceSynchronize();
        if (ctx->dsrc) cudaFree(ctx->dsrc);
        if (ctx->ddst) cudaFree(ctx->ddst);
        ctx->dsrc = ctx->ddst = nullptr;
        ctx->cap = 0;
        if (!ok(cudaMalloc(&ctx->dsrc, bytes), "cudaMalloc") || !ok(cudaMalloc(&ctx->ddst, bytes), "cudaMalloc"))
            return MTB_E_CUDA;
        ctx->cap = bytes;
    }
    return MTB_OK;
}

// ---- streaming host path: ONE launch over the whole frame while the copies
// run.  Source rows go host->device in chunks on the copy stream, each
// followed by a stream memory write of "rows arrived" (executed by the copy
// engine, after the data); CTAs spin on that counter before reading their
// rows.  Each CTA/tile adds the pixels it finished to its output chunk's
// counter; the device->host stream waits (stream memory wait) for a chunk's
// full count and copies it out.  Copies in, filtering and copies out
// overlap with no per-band relaunch cost.  Chunk copies end on 128-byte
// line boundaries, so no L1 line ever mixes arrived and pending rows.
typedef int (*write32_fn)(cudaStream_t, unsigned long long, unsigned int, unsigned int);

// driver stream memory operations (resolved at run time: no link-time
// libcuda dependency); false when the driver does not provide them
static bool stream_mem_ops(write32_fn &write32, write32_fn &wait32) {
    static write32_fn w = nullptr, t = nullptr;
    static int resolved = 0;
    if (!resolved) {
        void *fw = nullptr, *fwt = nullptr;
        cudaDriverEntryPointQueryResult q1, q2;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fw, cudaEnableDefault, &q1) == cudaSuccess &&
            cudaGetDriverEntryPoint("cuStreamWaitValue32", &fwt, cudaEnableDefault, &q2) == cudaSuccess &&
            q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess && fw && fwt) {
            w = reinterpret_cast<write32_fn>(fw);
            t = reinterpret_cast<write32_fn>(fwt);
            resolved = 1;
        } else {
            cudaGetLastError();
            resolved = -1;
        }
    }
    write32 = w;
    wait32 = t;
    return resolved > 0;
}

// page-locked (or registered) host memory: cudaMemcpyAsync returns at once
static bool host_pinned(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Output rows [A, B) of an H-row host frame: the device copy holds source
// rows [top, bot) = [max(0, A-r), min(H, B+r)) -- the rows the windows
// touch, clamped against the GLOBAL frame (engine.py:252-256) -- and the
// host destination `dst` holds rows [A, B).
struct HostRows {
    const char *src;  // host, global row 0
    char *dst;        // host, global row A
    int bit_depth, H, W, A, B, top, bot, radius;
    int64_t rank;
    const void *lut;
    size_t es, row;
};

static int host_stream(HostCtx *ctx, const HostRows &j) {
    write32_fn write32 = nullptr, wait32 = nullptr;
    if (!stream_mem_ops(write32, wait32)) return 1;  // caller falls back to the banded path
    const int rows = j.B - j.A;
    const size_t row = j.row, total = (size_t)(j.bot - j.top) * row;
    const int K = std::max(1, std::min(4, (j.bot - j.top) / 128));   // input chunks
    const int KO = std::max(1, std::min(8, std::min(63, rows / 128)));  // output chunks
    const int C = (rows + KO - 1) / KO;                                 // rows per output chunk
    const int nout = (rows + C - 1) / C;
    auto ok = [](cudaError_t e, const char *what) {
        return e == cudaSuccess ? MTB_OK : fail(MTB_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    };
    *ctx->hstatus = 0;
    int rc = ok(cudaMemsetAsync(ctx->dflags, 0, (1 + nout) * sizeof(unsigned int), ctx->sh), "memset");
    if (!rc && j.lut)
        rc = ok(cudaMemcpyAsync(ctx->dlut, j.lut, ((size_t)1 << j.bit_depth) * j.es, cudaMemcpyHostToDevice, ctx->sh),
                "H2D lut");
    if (rc) return rc;
    cudaEventRecord(ctx->eh[0], ctx->sh);
    cudaStreamWaitEvent(ctx->sc, ctx->eh[0], 0);
    cudaStreamWaitEvent(ctx->sd, ctx->eh[0], 0);
    // Every chunk copy and its "rows arrived" write (a global row count) is
    // enqueued BEFORE the launch (the source is page-locked, so this
    // returns at once): the kernel's CTAs only ever wait for copy-engine
    // work already in flight, whatever the launch serialisation
    // (CUDA_LAUNCH_BLOCKING, profilers, sanitizers).
    const char *s8 = j.src + (size_t)j.top * row;
    size_t b = 0;
    for (int i = 0; i < K && !rc; ++i) {
        const int R = j.top + (int)((int64_t)(j.bot - j.top) * (i + 1) / K);
        const size_t e = i == K - 1 ? total : std::min(total, ((size_t)(R - j.top) * row + 127) & ~(size_t)127);
        if (e > b) {
            rc = ok(cudaMemcpyAsync(static_cast<char *>(ctx->dsrc) + b, s8 + b, e - b, cudaMemcpyHostToDevice, ctx->sh),
                    "H2D");
            b = e;
        }
        if (!rc && write32(ctx->sh, (unsigned long long)ctx->dflags, (unsigned int)R, 0) != 0)
            rc = fail(MTB_E_CUDA, "cuStreamWriteValue32 failed");
    }
    if (!rc) {
        SlabParams p = make_params(ctx->dsrc, j.W, j.top, j.bot - j.top, ctx->ddst, j.W, j.H, j.W, j.A, j.B,
                                   j.radius, j.rank, j.lut ? ctx->dlut : nullptr);
        p.in_rows = ctx->dflags;
        p.out_px = ctx->dflags + 1;
        p.out_chunk = C;
        p.status = ctx->dstatus;
        rc = j.bit_depth == 8 ? run<uint8_t>(p, 1, ctx->sc) : run<uint16_t>(p, 1, ctx->sc);
    }
    for (int c = 0; c < nout && !rc; ++c) {
        const int a = c * C, e = std::min(rows, a + C);
        if (wait32(ctx->sd, (unsigned long long)(ctx->dflags + 1 + c), (unsigned int)((e - a) * j.W), 0) != 0)
            rc = fail(MTB_E_CUDA, "cuStreamWaitValue32 failed");
        else
            rc = ok(cudaMemcpyAsync(j.dst + (size_t)a * row, static_cast<char *>(ctx->ddst) + (size_t)a * row,
                                    (size_t)(e - a) * row, cudaMemcpyDeviceToHost, ctx->sd), "D2H");
    }
    if (rc) {
        // copy-out waits already enqueued can never be met now: release them
        for (int c = 0; c < nout; ++c)
            write32(ctx->sh, (unsigned long long)(ctx->dflags + 1 + c), 0xFFFFFFFFu, 0);
    }
    const int r1 = ok(cudaStreamSynchronize(ctx->sd), "cudaStreamSynchronize");
    const int r2 = ok(cudaStreamSynchronize(ctx->sc), "cudaStreamSynchronize");
    const int r3 = ok(cudaStreamSynchronize(ctx->sh), "cudaStreamSynchronize");
    if (!rc && *(volatile unsigned int *)ctx->hstatus)
        rc = fail(MTB_E_CUDA, "streaming launch timed out waiting for source rows");
    return rc ? rc : (r1 ? r1 : (r2 ? r2 : r3));
}

static int host_pipeline(const void *src, void *dst, int bit_depth, int H, int W, int A, int B, int radius,
                         int64_t rank, const void *lut) {
    HostRows j;
    j.src = static_cast<const char *>(src);
    j.dst = static_cast<char *>(dst);
    j.bit_depth = bit_depth;
    j.H = H;
    j.W = W;
    j.A = A;
    j.B = B;
    j.top = std::max(0, A - radius);
    j.bot = std::min(H, B + radius);
    j.radius = radius;
    j.rank = rank;
    j.lut = lut;
    j.es = bit_depth == 8 ? 1 : 2;
    j.row = (size_t)W * j.es;
    const size_t row = j.row;
    HostCtx *ctx = nullptr;
    std::unique_lock<std::mutex> lock;
    if (int rc = host_ctx(ctx, lock, (size_t)(j.bot - j.top) * row)) return rc;
    // 16-bit kernel choice from the host copy of the rows this call reads
    struct HintGuard {
        ~HintGuard() { g_spread_hint = -1; }
    } hint_guard;
    if (bit_depth == 16)
        g_spread_hint = spread_distinct_host(reinterpret_cast<const uint16_t *>(j.src + (size_t)j.top * row), W,
                                             j.bot - j.top, W);
    // streaming (one launch, copies overlapped) for compute-heavy radii;
    // row bands below, where the stream-op latencies outweigh the overlap
    // (tools/e2e_probe.py: equal at r = 15, streaming -12% at r = 31, +10%
    // at r <= 3).  Streaming needs a page-locked source (its copies must be
    // enqueued ahead of the launch without blocking); pageable frames take
    // the bands, whose launches never wait on copies.  MTB_HOST_STREAM=0/1
    // forces.
    const int stream_mode = env_int("MTB_HOST_STREAM", -1);
    // (widely spread 16-bit frames take the bands: the candidate-bucket path, several launches
    // over scratch planes, has no streaming form and is 2-5x faster than the kernels that do)
    const bool list16 = bit_depth == 16 && g_spread_hint > SPREAD_WIDE && radius >= LOWSEL_MIN_R &&
                        radius <= LOWSEL_MAX_R && env_int("MTB_U16_LIST", 1) != 0;
    const bool want_stream = (stream_mode < 0 ? radius >= 12 && !list16 : stream_mode != 0) && host_pinned(src);
    if (want_stream) {
        const int rs = host_stream(ctx, j);
        if (rs != 1) return rs;
    }
    // bands: enough rows that per-band launch and halo overheads stay small
    // (measured on config 2, tools/e2e_probe.py: 4 bands of 1024 rows for
    // r <= 31, 2 for r = 63 -- shorter bands re-pay the n-row column build).
    // Pageable frames are staged through page-locked buffers by the copy
    // pool, band by band (more, shorter bands: the host memcpy is the
    // pipeline's slowest stage there).
    const int rows = B - A;
    const bool stage_in = !host_pinned(src), stage_out = !host_pinned(dst);
    const int min_rows = std::max(stage_in || stage_out ? 512 : 1024, 32 * radius);
    int K = env_int("MTB_HOST_BANDS", std::min(stage_in || stage_out ? 12 : 8, std::max(1, rows / min_rows)));
    K = std::max(1, std::min(K, std::min(HostCtx::KMAX, rows)));
    auto cuda_ok = [](cudaError_t e, const char *what) {
        return e == cudaSuccess ? MTB_OK : fail(MTB_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    };
    if ((stage_in || stage_out) && host_staging(ctx, (size_t)(j.bot - j.top) * row) != MTB_OK) return MTB_E_CUDA;
    if (lut) {
        if (int rc = cuda_ok(cudaMemcpyAsync(ctx->dlut, lut, ((size_t)1 << bit_depth) * j.es, cudaMemcpyHostToDevice,
                                             ctx->sh), "H2D lut"))
            return rc;
    }
    char *ds = static_cast<char *>(ctx->dsrc);  // global row top
    char *dd = static_cast<char *>(ctx->ddst);  // global row A
    char *hin = static_cast<char *>(ctx->hin);    // staging: global row top
    char *hout = static_cast<char *>(ctx->hout);  // staging: global row A
    int copied = j.top;  // source rows [top, copied) enqueued host->device
    int rc = MTB_OK;
    auto band = [&](int i, int &a, int &b) {  // global output rows of band i
        a = A + (int)((int64_t)rows * i / K);
        b = A + (int)((int64_t)rows * (i + 1) / K);
    };
    // result rows of band i back to the host (enqueued one band late: with
    // pageable host memory the call blocks until the copy is done, and by
    // then the next band's filter is already queued behind it)
    auto d2h = [&](int i) {
        int a, b;
        band(i, a, b);
        cudaStreamWaitEvent(ctx->sd, ctx->ec[i], 0);
        char *to = stage_out ? hout : j.dst;
        const int r2 = cuda_ok(cudaMemcpyAsync(to + (size_t)(a - A) * row, dd + (size_t)(a - A) * row,
                                               (size_t)(b - a) * row, cudaMemcpyDeviceToHost, ctx->sd), "D2H");
        cudaEventRecord(ctx->eo[i], ctx->sd);
        return r2;
    };
    // a staged band's rows from the staging buffer to the caller's frame
    auto unstage = [&](int i) {
        if (!stage_out) return MTB_OK;
        int a, b;
        band(i, a, b);
        const int r2 = cuda_ok(cudaEventSynchronize(ctx->eo[i]), "cudaEventSynchronize");
        if (!r2) ctx->pool->copy(j.dst + (size_t)(a - A) * row, hout + (size_t)(a - A) * row, (size_t)(b - a) * row);
        return r2;
    };
    int done = 0;
    for (int i = 0; i < K && rc == MTB_OK; ++i) {
        int a, b;
        band(i, a, b);
        const int need = std::min(H, b + radius);
        if (need > copied) {
            const size_t off = (size_t)(copied - j.top) * row, len = (size_t)(need - copied) * row;
            if (stage_in) ctx->pool->copy(hin + off, j.src + (size_t)copied * row, len);
            rc = cuda_ok(cudaMemcpyAsync(ds + off, stage_in ? hin + off : j.src + (size_t)copied * row, len,
                                         cudaMemcpyHostToDevice, ctx->sh), "H2D");
            copied = need;
        }
        if (rc) break;
        cudaEventRecord(ctx->eh[i], ctx->sh);
        cudaStreamWaitEvent(ctx->sc, ctx->eh[i], 0);
        SlabParams p = make_params(ds, W, j.top, j.bot - j.top, dd + (size_t)(a - A) * row, W, H, W, a, b, radius,
                                   rank, lut ? ctx->dlut : nullptr);
        rc = bit_depth == 8 ? run<uint8_t>(p, 1, ctx->sc) : run<uint16_t>(p, 1, ctx->sc);
        if (rc) break;
        cudaEventRecord(ctx->ec[i], ctx->sc);
        if (i >= 1) rc = d2h(i - 1);
        if (!rc && i >= 2) rc = unstage(i - 2);
        done = i;
    }
    if (rc == MTB_OK) rc = d2h(done);
    for (int i = std::max(0, done - 1); i <= done && rc == MTB_OK; ++i) rc = unstage(i);
    const int rs = cuda_ok(cudaStreamSynchronize(ctx->sd), "cudaStreamSynchronize");
    cudaStreamSynchronize(ctx->sc);
    cudaStreamSynchronize(ctx->sh);
    return rc ? rc : rs;
}

// ---- sequence of host frames (mtb_filter_host_frames): whole-frame jobs on
// a ring of NB device buffer pairs.  Job i's host->device copy (copy stream)
// waits only for job i-NB's filter to release its source buffer; its filter
// (compute stream) waits for its copy and for job i-NB's device->host copy
// to release the destination buffer; its device->host copy waits for its
// filter.  So frame i+1 arrives and frame i-1 leaves while frame i is being
// filtered: the copy engines and the SMs stay busy across the sequence.
// NB = one buffer pair per frame of the call, 3 to NBMAX, within a device
// memory budget (round 1 kept 3: the ring's reuse waits then serialised the
// config-2 sweep's six frames behind the copies of the frames 3 back).
struct FramesCtx {
    static constexpr int NBMAX = 8;
    static constexpr int NFLAGS = 64;  // per slot: [0] rows arrived, [1..] output pixels per chunk
    int dev = -1, nb = 0;
    void *dsrc[NBMAX] = {}, *ddst[NBMAX] = {}, *dlut = nullptr;
    unsigned int *dflags = nullptr;  // [NBMAX][NFLAGS]
    unsigned int *hstatus = nullptr, *dstatus = nullptr;  // mapped pinned word: a CTA timed out waiting for rows
    size_t cap = 0;
    cudaStream_t sh = nullptr, sc = nullptr, sd = nullptr;
    cudaEvent_t ein[NBMAX], ek[NBMAX], eout[NBMAX];
};
static FramesCtx g_frames[64];
static std::mutex g_frames_mu[64];

static int frames_ctx(FramesCtx *&ctx, std::unique_lock<std::mutex> &lock, size_t bytes, int want_nb) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return fail(MTB_E_CUDA, "device index out of range");
    lock = std::unique_lock<std::mutex>(g_frames_mu[dev]);
    ctx = &g_frames[dev];
    auto ok = [](cudaError_t e, const char *what) {
        return e == cudaSuccess ? MTB_OK : fail(MTB_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    };
    if (ctx->dev < 0) {
        int rc = ok(cudaStreamCreateWithFlags(&ctx->sh, cudaStreamNonBlocking), "cudaStreamCreate");
        if (!rc) rc = ok(cudaStreamCreateWithFlags(&ctx->sc, cudaStreamNonBlocking), "cudaStreamCreate");
        if (!rc) rc = ok(cudaStreamCreateWithFlags(&ctx->sd, cudaStreamNonBlocking), "cudaStreamCreate");
        if (!rc) rc = ok(cudaMalloc(&ctx->dlut, 65536 * 2), "cudaMalloc");
        if (!rc) rc = ok(cudaMalloc(&ctx->dflags, FramesCtx::NBMAX * FramesCtx::NFLAGS * sizeof(unsigned int)), "cudaMalloc");
        if (!rc) rc = ok(cudaHostAlloc(&ctx->hstatus, sizeof(unsigned int), cudaHostAllocMapped), "cudaHostAlloc");
        if (!rc) rc = ok(cudaHostGetDevicePointer(&ctx->dstatus, ctx->hstatus, 0), "cudaHostGetDevicePointer");
        for (int j = 0; j < FramesCtx::NBMAX && !rc; ++j) {
            rc = ok(cudaEventCreateWithFlags(&ctx->ein[j], cudaEventDisableTiming), "cudaEventCreate");
            if (!rc) rc = ok(cudaEventCreateWithFlags(&ctx->ek[j], cudaEventDisableTiming), "cudaEventCreate");
            if (!rc) rc = ok(cudaEventCreateWithFlags(&ctx->eout[j], cudaEventDisableTiming), "cudaEventCreate");
        }
        if (rc) return rc;
        ctx->dev = dev;
    }
    // buffer pairs: one per frame (3..NBMAX), at most 2 GiB of them
    const size_t budget = 2ull << 30;
    int nb = std::max(3, std::min(FramesCtx::NBMAX, want_nb));
    while (nb > 3 && (size_t)nb * 2 * bytes > budget) --nb;
    if (ctx->cap < bytes) {
        cudaDeviceSynchronize();
        for (int j = 0; j < FramesCtx::NBMAX; ++j) {
            if (ctx->dsrc[j]) cudaFree(ctx->dsrc[j]);
            if (ctx->ddst[j]) cudaFree(ctx->ddst[j]);
            ctx->dsrc[j] = ctx->ddst[j] = nullptr;
        }
        ctx->cap = bytes;
        ctx->nb = 0;
    }
    for (int j = ctx->nb; j < nb; ++j) {
        if (int rc = ok(cudaMalloc(&ctx->dsrc[j], ctx->cap), "cudaMalloc")) return j >= 3 ? (ctx->nb = j, MTB_OK) : rc;
        if (int rc = ok(cudaMalloc(&ctx->ddst[j], ctx->cap), "cudaMalloc")) {
            cudaFree(ctx->dsrc[j]);
            ctx->dsrc[j] = nullptr;
            return j >= 3 ? (ctx->nb = j, MTB_OK) : rc;
        }
        ctx->nb = j + 1;
    }
    return MTB_OK;
}

static int host_frames(const void *const *srcs, void *const *dsts, const int32_t *radii, const int64_t *ranks,
                       int n, int bit_depth, int H, int W, const void *lut, uint32_t flags) {
    const size_t es = bit_depth == 8 ? 1 : 2;
    const size_t bytes = (size_t)H * W * es;
    FramesCtx *ctx = nullptr;
    std::unique_lock<std::mutex> lock;
    if (int rc = frames_ctx(ctx, lock, bytes, n)) return rc;
    auto ok = [](cudaError_t e, const char *what) {
        return e == cudaSuccess ? MTB_OK : fail(MTB_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    };
    (void)flags;
    int rc = MTB_OK;
    *ctx->hstatus = 0;
    if (lut) {
        rc = ok(cudaMemcpyAsync(ctx->dlut, lut, ((size_t)1 << bit_depth) * es, cudaMemcpyHostToDevice, ctx->sc),
                "H2D lut");
    }
    const int NB = std::min(ctx->nb, std::max(3, n));  // buffer pairs this call rotates through
    // Streaming frames: a frame's rows arrive in chunks (CTAs wait on a row
    // counter) and its results leave in chunks (the copy-out stream waits on
    // per-chunk pixel counters), so the frame also overlaps its OWN copies.
    // MTB_FRAMES_STREAM = 4 (default): the first frame of the order only --
    // its copy-in is the one nothing else hides (config-2 sweep, e2e, mean
    // of 6 / 7 runs: 32.5 against 31.8 Gpix/s with whole-frame copies);
    // 1: every frame (31.5: the stream-op latencies cost more than they
    // hide in the middle of the sequence); 2: first and last (32.3, noisier);
    // 3: last only (31.7); 0: none.
    write32_fn write32 = nullptr, wait32 = nullptr;
    const int smode = env_int("MTB_FRAMES_STREAM", 4);
    const bool can_stream = smode != 0 && stream_mem_ops(write32, wait32) && H >= 256;
    const size_t row = (size_t)W * es;
    const int KI = std::max(1, std::min(4, H / 128));
    const int KO = std::max(1, std::min(4, std::min(FramesCtx::NFLAGS - 1, H / 128)));
    const int C = (H + KO - 1) / KO, nout = (H + C - 1) / C;
    // Processing order: heavy and light frames alternate (by radius, the
    // filter cost's proxy at one geometry: largest, smallest, second
    // largest, ...), so a short filter never leaves the SMs idle while the
    // next frame is still arriving, and a long one hides the neighbours'
    // copies.  Results land in dsts[i] whatever the order.  On the
    // config-2 sweep this is within 0.2% of the best of all 720 orders in a
    // copy / filter timeline model (3.16 against 3.52 ms in input order).
    std::vector<int> order(n);
    for (int i = 0; i < n; ++i) order[i] = i;
    {
        std::vector<int> byr(order);
        std::stable_sort(byr.begin(), byr.end(), [&](int a, int b) { return radii[a] > radii[b]; });
        for (int q = 0, lo = 0, hi = n - 1; q < n; ++q) order[q] = (q & 1) ? byr[hi--] : byr[lo++];
        // MTB_FRAMES_PERM="a,b,...": positions in the radius-descending list (tuning)
        if (const char *pe = getenv("MTB_FRAMES_PERM")) {
            std::vector<int> perm;
            for (const char *c = pe; *c;) {
                char *e = nullptr;
                const long v = strtol(c, &e, 10);
                if (e == c) break;
                perm.push_back((int)v);
                c = *e ? e + 1 : e;
            }
            if ((int)perm.size() == n) {
                std::vector<char> seen(n, 0);
                bool okp = true;
                for (int v : perm) okp = okp && v >= 0 && v < n && !seen[v] && (seen[v] = 1);
                if (okp)
                    for (int q = 0; q < n; ++q) order[q] = byr[perm[q]];
            }
        }
    }
    for (int q = 0; q < n && rc == MTB_OK; ++q) {
        const int i = order[q];
        const int j = q % NB;
        if (!srcs[i] || !dsts[i]) {
            rc = fail(MTB_E_INVAL, "null src/dst pointer (frame " + std::to_string(i) + ")");
            break;
        }
        unsigned int *fl = ctx->dflags + j * FramesCtx::NFLAGS;
        // smode 1: every frame streams; 2: the first and last (the copies
        // nothing else hides); 3: the last only
        // (16-bit kernel choice from the host frame; widely spread frames in the candidate-bucket
        // path's radii do not stream -- that path has no streaming form)
        const int hint = bit_depth == 16 ? spread_distinct_host(static_cast<const uint16_t *>(srcs[i]), W, H, W) : -1;
        const bool list16 = hint > SPREAD_WIDE && radii[i] >= LOWSEL_MIN_R && radii[i] <= LOWSEL_MAX_R &&
                            env_int("MTB_U16_LIST", 1) != 0;
        const bool streaming = can_stream && !list16 &&
                               (smode == 1 || (smode == 2 && (q == 0 || q == n - 1)) ||
                                (smode == 3 && q == n - 1) || (smode == 4 && q == 0));
        if (q >= NB) cudaStreamWaitEvent(ctx->sh, ctx->ek[j], 0);  // job i-NB done reading dsrc[j]
        if (streaming) {
            // counters reset before this frame's kernel or copy-out can look
            // at them, and only after job i-NB's copy-out stopped waiting on
            // them (the same slot's counters)
            if (q >= NB) cudaStreamWaitEvent(ctx->sh, ctx->eout[j], 0);
            rc = ok(cudaMemsetAsync(fl, 0, (1 + nout) * sizeof(unsigned int), ctx->sh), "memset");
            if (rc) break;
            cudaEventRecord(ctx->ein[j], ctx->sh);
            const char *s8 = static_cast<const char *>(srcs[i]);
            size_t b = 0;
            for (int q = 0; q < KI && !rc; ++q) {
                const int R = (int)((int64_t)H * (q + 1) / KI);
                const size_t e = q == KI - 1 ? bytes : std::min(bytes, ((size_t)R * row + 127) & ~(size_t)127);
                if (e > b) {
                    rc = ok(cudaMemcpyAsync(static_cast<char *>(ctx->dsrc[j]) + b, s8 + b, e - b,
                                            cudaMemcpyHostToDevice, ctx->sh), "H2D");
                    b = e;
                }
                if (!rc && write32(ctx->sh, (unsigned long long)fl, (unsigned int)R, 0) != 0)
                    rc = fail(MTB_E_CUDA, "cuStreamWriteValue32 failed");
            }
        } else {
            rc = ok(cudaMemcpyAsync(ctx->dsrc[j], srcs[i], bytes, cudaMemcpyHostToDevice, ctx->sh), "H2D");
            if (!rc) cudaEventRecord(ctx->ein[j], ctx->sh);
        }
        if (rc) break;
        cudaStreamWaitEvent(ctx->sc, ctx->ein[j], 0);
        if (q >= NB) cudaStreamWaitEvent(ctx->sc, ctx->eout[j], 0);  // job i-NB's result copied out
        g_spread_hint = hint;
        SlabParams p = make_params(ctx->dsrc[j], W, 0, H, ctx->ddst[j], W, H, W, 0, H, radii[i],
                                   ranks ? ranks[i] : 0, lut ? ctx->dlut : nullptr);
        if (!ranks) {
            const int64_t nn = 2 * (int64_t)radii[i] + 1;
            p.rank = (uint32_t)((nn * nn + 1) / 2);
        }
        if (streaming) {
            p.in_rows = fl;
            p.out_px = fl + 1;
            p.out_chunk = C;
            p.status = ctx->dstatus;
        }
        rc = bit_depth == 8 ? run<uint8_t>(p, 1, ctx->sc) : run<uint16_t>(p, 1, ctx->sc);
        g_spread_hint = -1;
        if (rc) {
            // release CTAs of this or earlier frames that might wait on rows
            if (streaming) write32(ctx->sh, (unsigned long long)fl, (unsigned int)H, 0);
            break;
        }
        cudaEventRecord(ctx->ek[j], ctx->sc);
        char *d8 = static_cast<char *>(dsts[i]);
        if (streaming) {
            cudaStreamWaitEvent(ctx->sd, ctx->ein[j], 0);  // counters reset for this frame
            for (int c = 0; c < nout && !rc; ++c) {
                const int a = c * C, e = std::min(H, a + C);
                if (wait32(ctx->sd, (unsigned long long)(fl + 1 + c), (unsigned int)((e - a) * W), 0) != 0)
                    rc = fail(MTB_E_CUDA, "cuStreamWaitValue32 failed");
                else
                    rc = ok(cudaMemcpyAsync(d8 + (size_t)a * row, static_cast<char *>(ctx->ddst[j]) + (size_t)a * row,
                                            (size_t)(e - a) * row, cudaMemcpyDeviceToHost, ctx->sd), "D2H");
            }
        } else {
            cudaStreamWaitEvent(ctx->sd, ctx->ek[j], 0);
            rc = ok(cudaMemcpyAsync(d8, ctx->ddst[j], bytes, cudaMemcpyDeviceToHost, ctx->sd), "D2H");
        }
        if (rc) break;
        cudaEventRecord(ctx->eout[j], ctx->sd);
    }
    const int r1 = ok(cudaStreamSynchronize(ctx->sd), "cudaStreamSynchronize");
    const int r2 = ok(cudaStreamSynchronize(ctx->sc), "cudaStreamSynchronize");
    const int r3 = ok(cudaStreamSynchronize(ctx->sh), "cudaStreamSynchronize");
    if (!rc && *(volatile unsigned int *)ctx->hstatus)
        rc = fail(MTB_E_CUDA, "streaming launch timed out waiting for source rows");
    return rc ? rc : (r1 ? r1 : (r2 ? r2 : r3));
}

extern "C" {

int mtb_median_u8(const uint8_t *src, int64_t src_pitch, int32_t src_row0, int32_t src_rows,
                  uint8_t *dst, int64_t dst_pitch, int32_t H, int32_t W, int32_t row_begin,
                  int32_t row_end, int32_t radius, int64_t rank, const uint8_t *lut,
                  uint32_t flags, void *stream) {
    (void)flags;
    SlabParams p = make_params(src, src_pitch, src_row0, src_rows, dst, dst_pitch, H, W,
                               row_begin, row_end, radius, rank, lut);
    return run<uint8_t>(p, 1, (cudaStream_t)stream);
}

int mtb_median_u16(const uint16_t *src, int64_t src_pitch, int32_t src_row0, int32_t src_rows,
                   uint16_t *dst, int64_t dst_pitch, int32_t H, int32_t W, int32_t row_begin,
                   int32_t row_end, int32_t radius, int64_t rank, const uint16_t *lut,
                   uint32_t flags, void *stream) {
    (void)flags;
    SlabParams p = make_params(src, src_pitch, src_row0, src_rows, dst, dst_pitch, H, W,
                               row_begin, row_end, radius, rank, lut);
    return run<uint16_t>(p, 1, (cudaStream_t)stream);
}

int mtb_median_batch_u8(const uint8_t *src, int64_t src_image_stride, int64_t src_pitch,
                        uint8_t *dst, int64_t dst_image_stride, int64_t dst_pitch, int32_t B,
                        int32_t H, int32_t W, int32_t radius, int64_t rank, const uint8_t *lut,
                        uint32_t flags, void *stream) {
    (void)flags;
    SlabParams p = make_params(src, src_pitch, 0, H, dst, dst_pitch, H, W, 0, H, radius, rank, lut);
    p.src_img_stride = src_image_stride;
    p.dst_img_stride = dst_image_stride;
    return run<uint8_t>(p, B, (cudaStream_t)stream);
}

int mtb_median_batch_u16(const uint16_t *src, int64_t src_image_stride, int64_t src_pitch,
                         uint16_t *dst, int64_t dst_image_stride, int64_t dst_pitch, int32_t B,
                         int32_t H, int32_t W, int32_t radius, int64_t rank, const uint16_t *lut,
                         uint32_t flags, void *stream) {
    (void)flags;
    SlabParams p = make_params(src, src_pitch, 0, H, dst, dst_pitch, H, W, 0, H, radius, rank, lut);
    p.src_img_stride = src_image_stride;
    p.dst_img_stride = dst_image_stride;
    return run<uint16_t>(p, B, (cudaStream_t)stream);
}

int mtb_filter_host(const void *src, void *dst, int32_t bit_depth, int32_t H, int32_t W,
                    int32_t radius, int64_t rank, const void *lut, uint32_t flags) {
    if (bit_depth != 8 && bit_depth != 16)
        return fail(MTB_E_INVAL, "bit_depth must be 8 or 16, got " + std::to_string(bit_depth));
    if (!src || !dst) return fail(MTB_E_INVAL, "null src/dst pointer");
    if (H < 1 || W < 1) return fail(MTB_E_INVAL, "pixels must be a non-empty 2D array");
    (void)flags;
    return host_pipeline(src, dst, bit_depth, H, W, 0, H, radius, rank, lut);
}

int mtb_filter_host_rows(const void *src, void *dst, int32_t bit_depth, int32_t H, int32_t W, int32_t row_begin,
                         int32_t row_end, int32_t radius, int64_t rank, const void *lut, uint32_t flags,
                         int32_t device) {
    (void)flags;
    if (bit_depth != 8 && bit_depth != 16)
        return fail(MTB_E_INVAL, "bit_depth must be 8 or 16, got " + std::to_string(bit_depth));
    if (!src || !dst) return fail(MTB_E_INVAL, "null src/dst pointer");
    if (H < 1 || W < 1) return fail(MTB_E_INVAL, "pixels must be a non-empty 2D array");
    if (row_begin < 0 || row_end > H || row_begin > row_end) return fail(MTB_E_INVAL, "bad output row range");
    if (row_begin == row_end) return MTB_OK;
    if (device >= 0) {
        cudaError_t e = cudaSetDevice(device);
        if (e != cudaSuccess) return fail(MTB_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    }
    return host_pipeline(src, dst, bit_depth, H, W, row_begin, row_end, radius, rank, lut);
}

int mtb_filter_host_frames(const void *const *srcs, void *const *dsts, const int32_t *radii, const int64_t *ranks,
                           int32_t n_frames, int32_t bit_depth, int32_t H, int32_t W, const void *lut,
                           uint32_t flags) {
    if (bit_depth != 8 && bit_depth != 16)
        return fail(MTB_E_INVAL, "bit_depth must be 8 or 16, got " + std::to_string(bit_depth));
    if (n_frames < 0) return fail(MTB_E_INVAL, "n_frames must be >= 0");
    if (n_frames == 0) return MTB_OK;
    if (!srcs || !dsts || !radii) return fail(MTB_E_INVAL, "null srcs/dsts/radii array");
    if (H < 1 || W < 1) return fail(MTB_E_INVAL, "pixels must be a non-empty 2D array");
    return host_frames(srcs, dsts, radii, ranks, n_frames, bit_depth, H, W, lut, flags);
}

int mtb_rank_bruteforce(const void *src, int64_t src_pitch, void *dst, int64_t dst_pitch, int32_t bit_depth,
                        int32_t H, int32_t W, int32_t radius, int64_t rank, void *stream) {
    if (bit_depth != 8 && bit_depth != 16)
        return fail(MTB_E_INVAL, "bit_depth must be 8 or 16, got " + std::to_string(bit_depth));
    if (!src || !dst) return fail(MTB_E_INVAL, "null src/dst pointer");
    if (H < 1 || W < 1) return fail(MTB_E_INVAL, "pixels must be a non-empty 2D array");
    if (radius < 0) return fail(MTB_E_INVAL, "radius must be >= 0");
    const int64_t n = 2 * (int64_t)radius + 1;
    if (rank < 1 || rank > n * n) return fail(MTB_E_INVAL, "rank must be in [1, n*n]");
    if (src_pitch < W || dst_pitch < W) return fail(MTB_E_INVAL, "pitch must be >= W");
    dim3 block(32, 8), grid((W + 31) / 32, (H + 7) / 8);
    cudaStream_t s = (cudaStream_t)stream;
    if (bit_depth == 8)
        k_select_brute<uint8_t, 8><<<grid, block, 0, s>>>((const uint8_t *)src, src_pitch, (uint8_t *)dst, dst_pitch,
                                                          H, W, radius, (uint32_t)rank);
    else
        k_select_brute<uint16_t, 16><<<grid, block, 0, s>>>((const uint16_t *)src, src_pitch, (uint16_t *)dst,
                                                            dst_pitch, H, W, radius, (uint32_t)rank);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(MTB_E_CUDA, std::string("k_select_brute: ") + cudaGetErrorString(e));
    g_kernel = "k_select_brute";
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return MTB_OK;
}

int mtb_set_device(int32_t device) {
    cudaError_t e = cudaSetDevice(device);
    return e == cudaSuccess ? MTB_OK : fail(MTB_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
}

uint64_t mtb_launch_count(void) { return g_launches.load(); }
const char *mtb_last_kernel(void) { return g_kernel; }
const char *mtb_last_error(void) { return g_err.c_str(); }
int mtb_version(void) { return 2; }

}  // extern "C"
