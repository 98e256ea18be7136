/*
 * medtree_b200.h -- C ABI of the B200 running-median (rank filter) library.
 *
 * Drop-in boundary for the reference's native seam.  The reference
 * (/root/reference/pkg, Python + numba) has no C FFI; its compiled entry
 * points are the numba frame drivers
 *
 *   run_frame_u(img, out, cols, win, lastx, valid, n, d, levels, r, ops,
 *               counting, on_demand)        pkg/src/medtree/_kernels.py:326-351
 *   run_frame_a(img, out, cols, win, lastx, valid, n, r, up, leaf, span,
 *               n_values, precision, max_error, ops, counting, on_demand)
 *                                           pkg/src/medtree/_kernels.py:354-388
 *
 * called from WindowEngine.run (pkg/src/medtree/engine.py:162-184) once per
 * frame or per band (engine.py:243-262).  Like them, these entry points
 * take caller-owned buffers, write `dst` in place and allocate nothing on
 * the hot call.  The reference's scratch arrays (cols/win/lastx/valid/ops)
 * have no counterpart: all per-window state lives in on-chip memory.
 * Reduced precision (max_error) and adaptive topologies enter as an
 * optional value map `lut` (2^bit_depth entries) applied to the exact rank
 * value: the reference's descent returns the lower bound of the first tree
 * node on the path to the exact value whose width is <= max_error
 * (_kernels.py:229-253, 256-289), which is a pure function of that value.
 *
 * Semantics (identical to the reference):
 *   out[y][x] = sorted{ img[clamp(y+j)][clamp(x+i)] : i,j in [-radius,radius] }[rank-1]
 *   (replicate borders: coordinates clamped to the GLOBAL image [0,H)x[0,W)),
 *   then out = lut ? lut[out] : out.
 *
 * Pointers `src`, `dst`, `lut` are DEVICE pointers.  Pitches are in
 * elements.  A call filters output rows [row_begin, row_end) of a global
 * H-row image; `src` holds global rows [src_row0, src_row0 + src_rows),
 * which must cover every clamped row the window touches
 * ([max(0,row_begin-radius), min(H,row_end+radius))).  This is the slab
 * form of the reference's bands (engine.py:252-256): halo rows come from
 * the caller's copy and clamping is against the global edges.
 *
 * Return 0 on success, MTB_E_INVAL for an invalid argument, MTB_E_CUDA for a
 * CUDA launch error; mtb_last_error() returns a thread-local message.
 * Invalid-argument checks mirror pkg/src/medtree/validation.py:19-54.
 */
#ifndef MEDTREE_B200_H
#define MEDTREE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MTB_OK 0
#define MTB_E_INVAL (-1)
#define MTB_E_CUDA (-2)

/* `flags` arguments are reserved: pass 0.  (The reference's adaptive
 * topology only changes results at max_error > 1, where it enters as the
 * value map `lut`; the kernels' data layout does not depend on it --
 * DESIGN.md section 3.7.) */

/* One 8-bit slab.  Replaces run_frame_u/run_frame_a for bit_depth 8. */
int mtb_median_u8(const uint8_t *src, int64_t src_pitch, int32_t src_row0, int32_t src_rows,
                  uint8_t *dst, int64_t dst_pitch,
                  int32_t H, int32_t W, int32_t row_begin, int32_t row_end,
                  int32_t radius, int64_t rank, const uint8_t *lut,
                  uint32_t flags, void *stream);

/* One 16-bit slab.  Replaces run_frame_u/run_frame_a for bit_depth 16. */
int mtb_median_u16(const uint16_t *src, int64_t src_pitch, int32_t src_row0, int32_t src_rows,
                   uint16_t *dst, int64_t dst_pitch,
                   int32_t H, int32_t W, int32_t row_begin, int32_t row_end,
                   int32_t radius, int64_t rank, const uint16_t *lut,
                   uint32_t flags, void *stream);

/* A batch of B independent HxW images (config 5); image b starts at
 * src + b*src_image_stride / dst + b*dst_image_stride (elements). */
int mtb_median_batch_u8(const uint8_t *src, int64_t src_image_stride, int64_t src_pitch,
                        uint8_t *dst, int64_t dst_image_stride, int64_t dst_pitch,
                        int32_t B, int32_t H, int32_t W, int32_t radius, int64_t rank,
                        const uint8_t *lut, uint32_t flags, void *stream);

int mtb_median_batch_u16(const uint16_t *src, int64_t src_image_stride, int64_t src_pitch,
                         uint16_t *dst, int64_t dst_image_stride, int64_t dst_pitch,
                         int32_t B, int32_t H, int32_t W, int32_t radius, int64_t rank,
                         const uint16_t *lut, uint32_t flags, void *stream);

/* Whole-frame convenience on HOST buffers (H2D, filter, D2H on an internal
 * stream; synchronous).  The reference-facing call for callers without a
 * device allocator -- e.g. a ctypes binding replacing
 * WindowEngine.run (engine.py:162-184).  bit_depth is 8 or 16; src/dst point
 * to uint8 or uint16 row-major [H][W]. */
int mtb_filter_host(const void *src, void *dst, int32_t bit_depth, int32_t H, int32_t W,
                    int32_t radius, int64_t rank, const void *lut, uint32_t flags);

/* Output rows [row_begin, row_end) of an H x W HOST frame, on GPU `device`
 * (-1: the calling thread's current device).  `src` is the whole frame
 * (global row 0); only the rows the windows touch,
 * [max(0,row_begin-radius), min(H,row_end+radius)), are read, straight from
 * the host copy -- the reference's band with its n//2 halo rows
 * (engine.py:243-262), clamped against the global frame.  `dst` receives
 * rows [row_begin, row_end) (dst row 0 = global row row_begin).  One host
 * thread per GPU, each with its own slab, filters a frame on several GPUs
 * with no collective.  Synchronous. */
int mtb_filter_host_rows(const void *src, void *dst, int32_t bit_depth, int32_t H, int32_t W,
                         int32_t row_begin, int32_t row_end, int32_t radius, int64_t rank,
                         const void *lut, uint32_t flags, int32_t device);

/* A sequence of n_frames HOST frames of one geometry (e.g. a video, or one
 * frame at several radii), each filtered as by mtb_filter_host, with the
 * copies of neighbouring frames overlapped: frame i+1 goes host->device and
 * frame i-1 device->host while frame i is filtered (a ring of 3 device
 * buffer pairs).  srcs[i] / dsts[i]: host frames [H][W] (page-locked for
 * asynchronous copies); radii[i]: window radius; ranks: per-frame 1-based
 * rank, or NULL for the median.  Synchronous: returns when every result is
 * on the host.  The batched form of the reference's per-image
 * filter_image / WindowEngine.run loop (engine.py:162-184, :209-262). */
int mtb_filter_host_frames(const void *const *srcs, void *const *dsts, const int32_t *radii,
                           const int64_t *ranks, int32_t n_frames, int32_t bit_depth,
                           int32_t H, int32_t W, const void *lut, uint32_t flags);

/* Independent exact selection on DEVICE buffers: per pixel, the bits of the
 * rank-th smallest window value are decided from the top by counting passes
 * over the n x n replicate-clamped window (O(d * n^2) per pixel).  Shares no
 * code with the fast kernels; it is the package's GPU stand-in for the
 * reference's oracle filters (oracles.py:36-66, used by `cli compare` and
 * `bench --oracle`).  bit_depth 8 or 16; src/dst uint8/uint16 [H][pitch]. */
int mtb_rank_bruteforce(const void *src, int64_t src_pitch, void *dst, int64_t dst_pitch,
                        int32_t bit_depth, int32_t H, int32_t W, int32_t radius, int64_t rank,
                        void *stream);

/* Make `device` current for the calling thread in this library's CUDA
 * runtime (the host-buffer entries run on the current device). */
int mtb_set_device(int32_t device);

/* Kernel launches issued by this library since load (evidence counter). */
uint64_t mtb_launch_count(void);

/* Name of the kernel variant the last call on this thread selected. */
const char *mtb_last_kernel(void);

const char *mtb_last_error(void);
int mtb_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MEDTREE_B200_H */
