"""Drop-in ``filter_image``: the reference's call surface on the B200 path.

Mirrors pkg/src/medtree/engine.py:209-262 -- same arguments, same
validation order and ValueErrors, same ``(GrayImage, OpCounters)`` return --
but every output pixel is computed by the sm_100a kernels behind the C ABI
(include/medtree_b200.h).  PyTorch is only the device allocator / stream /
copy engine.  There is no CPU path: without a CUDA device the call raises.

Row slabs.  ``bands=k`` is accepted with the reference's meaning
(horizontal bands with n//2 halo rows, identical output,
engine.py:243-262); the library picks its own row bands for the copy /
filter overlap.  ``devices=[...]`` spreads the frame over several GPUs:
``plan_slabs`` cuts one slab per GPU, and each GPU's host thread sends its
rows plus r halo rows straight from the host copy through
mtb_filter_host_rows and gets its rows back -- no collective
(SURVEY.md section 8(e)).  ``filter_images`` spreads a batch of images
over GPUs (``plan_images``, config 5).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .counters import OpCounters
from .image import GrayImage
from .topology import (
    MODES,
    TreeTopology,
    resolve_topology,
    uniform_topology,
    value_map,
)
from .validation import as_gray_image, check_max_error, check_window, resolve_rank

_torch = None


def _t():
    global _torch
    if _torch is None:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: the B200 rank filter has no CPU fallback")
        _torch = torch
    return _torch


def rank_filter(
    src,
    radius: int,
    rank: int | None = None,
    *,
    out=None,
    lut=None,
    rows: tuple[int, int] | None = None,
    src_row0: int = 0,
    height: int | None = None,
    stream=None,
):
    """Device-resident rank filter (no host copies).

    ``src``: CUDA tensor uint8/uint16, shape (H, W) or (B, H, W).  For a
    2-D slab, ``src`` holds global rows [src_row0, src_row0+src.shape[0]) of
    an image with ``height`` rows and ``rows=(a, b)`` selects the output
    rows; ``out`` then has b-a rows.  ``out`` (optional) must be a CUDA
    tensor on src's device with src's dtype and contiguous rows.  ``lut``:
    optional CUDA tensor with 2^bit_depth entries applied to the exact rank
    value.  Runs on ``stream`` (default: the current stream of src's
    device).  Returns ``out``.
    """
    torch = _t()
    if src.device.type != "cuda":
        raise ValueError("src must be a CUDA tensor")
    if src.dtype == torch.uint8:
        bits = 8
    elif src.dtype == torch.uint16:
        bits = 16
    else:
        raise ValueError(f"src dtype must be uint8 or uint16, got {src.dtype}")
    if src.stride(-1) != 1:
        raise ValueError("src rows must be contiguous")
    if src.dim() not in (2, 3):
        raise ValueError("src must be 2-D (H, W) or 3-D (B, H, W)")
    n = 2 * int(radius) + 1
    if rank is None:
        rank = (n * n + 1) // 2
    if out is not None:
        if out.device != src.device or out.dtype != src.dtype:
            raise ValueError(f"out must be a {src.dtype} tensor on {src.device}, "
                             f"got {out.dtype} on {out.device}")
        if out.dim() != src.dim() or out.stride(-1) != 1:
            raise ValueError("out must have src's rank and contiguous rows")
    lib = _lib.load()
    lut_ptr = None
    if lut is not None:
        if lut.device != src.device or lut.dtype != src.dtype or lut.numel() != (1 << bits):
            raise ValueError("lut must be a CUDA tensor of 2^bit_depth entries, src dtype")
        lut_ptr = lut.data_ptr()
    with torch.cuda.device(src.device):
        _lib.check(lib.mtb_set_device(src.device.index))
        sh = (stream if stream is not None else torch.cuda.current_stream(src.device)).cuda_stream
        if src.dim() == 3:
            B, H, W = src.shape
            if out is None:
                out = torch.empty((B, H, W), dtype=src.dtype, device=src.device)
            elif tuple(out.shape) != (B, H, W):
                raise ValueError(f"out must have shape {(B, H, W)}, got {tuple(out.shape)}")
            fn = lib.mtb_median_batch_u8 if bits == 8 else lib.mtb_median_batch_u16
            rc = fn(src.data_ptr(), src.stride(0), src.stride(1), out.data_ptr(), out.stride(0),
                    out.stride(1), B, H, W, int(radius), int(rank), lut_ptr, 0, sh)
            _lib.check(rc)
            return out
        src_rows, W = src.shape
        H = src_rows if height is None else int(height)
        a, b = (0, H) if rows is None else (int(rows[0]), int(rows[1]))
        if out is None:
            out = torch.empty((max(0, b - a), W), dtype=src.dtype, device=src.device)
        if out.shape[0] < b - a or out.shape[1] != W:
            raise ValueError(f"out must be ({b - a}, {W}) with contiguous rows, got {tuple(out.shape)}")
        fn = lib.mtb_median_u8 if bits == 8 else lib.mtb_median_u16
        rc = fn(src.data_ptr(), src.stride(0), int(src_row0), int(src_rows), out.data_ptr(),
                out.stride(0), H, W, a, b, int(radius), int(rank), lut_ptr, 0, sh)
        _lib.check(rc)
    return out


# ---------------------------------------------------------------- planners

class Slab(tuple):
    """Output rows [a, b) of a frame and the source rows [top, bot) their
    windows read: the reference's band with n//2 halo rows
    (engine.py:243-262), clamped against the global frame."""

    __slots__ = ()

    def __new__(cls, a, b, top, bot):
        return tuple.__new__(cls, (a, b, top, bot))

    a = property(lambda s: s[0])
    b = property(lambda s: s[1])
    top = property(lambda s: s[2])
    bot = property(lambda s: s[3])


def plan_slabs(H: int, parts: int, radius: int) -> list[Slab]:
    """Cut H rows into ``parts`` row slabs with their halo source rows.
    Edges follow engine.py:248 (numpy.linspace(0, H, parts+1, dtype=int));
    empty slabs are dropped."""
    edges = np.linspace(0, H, int(parts) + 1, dtype=int)
    return [Slab(int(a), int(b), max(0, int(a) - radius), min(H, int(b) + radius))
            for a, b in zip(edges[:-1], edges[1:]) if a != b]


def plan_images(count: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous, balanced runs of images [i0, i1) per part (config 5:
    the batch over GPUs); parts beyond ``count`` get none."""
    edges = np.linspace(0, count, int(parts) + 1, dtype=int)
    return [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:])]


def _band_edges(H: int, bands: int) -> list[tuple[int, int]]:
    """engine.py:248: numpy.linspace(0, H, bands+1, dtype=int) edges."""
    return [(s.a, s.b) for s in plan_slabs(H, bands, 0)]


def _device_index(d) -> int:
    if isinstance(d, int):
        return d
    torch = _t()
    d = torch.device(d)
    if d.type != "cuda":
        raise ValueError(f"devices must be CUDA devices, got {d}")
    return torch.cuda.current_device() if d.index is None else d.index


def _devices(devices) -> list[int]:
    torch = _t()
    if devices is None:
        return [torch.cuda.current_device()]
    devs = [_device_index(d) for d in devices]
    if not devs:
        raise ValueError("devices must not be empty")
    return devs


def _on_devices(jobs):
    """Run ``fn(device)`` for each (device, fn) on its own host thread (the
    ctypes calls release the GIL), re-raising the first error."""
    if len(jobs) == 1:
        dev, fn = jobs[0]
        return [fn(dev)]
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        futs = [ex.submit(fn, dev) for dev, fn in jobs]
        return [f.result() for f in futs]


def _check_lut(lut, dtype, bits):
    if lut is None:
        return None
    lut = np.ascontiguousarray(lut, dtype=dtype)
    if lut.ndim != 1 or lut.size != 1 << bits:
        raise ValueError(f"lut must have 2^{bits} = {1 << bits} entries, got {lut.size}")
    return lut


def _run(px: np.ndarray, bits: int, radius: int, rank: int, lut: np.ndarray | None,
         devices) -> np.ndarray:
    devs = _devices(devices)
    if len(devs) == 1:
        # one device: the library's host-buffer entry, which pipelines row
        # bands or streams the frame (copy in / filter / copy out overlap)
        return filter_host_buffer(px, radius, rank, lut=lut, device=devs[0])
    # several GPUs: one row slab per device, halo rows read straight from the
    # host frame by each device's own host thread -- no collective
    H, W = px.shape
    src = np.ascontiguousarray(px)
    out = np.empty_like(src)
    lut = _check_lut(lut, src.dtype, bits)
    lut_ptr = lut.ctypes.data if lut is not None else None
    lib = _lib.load()
    slabs = plan_slabs(H, min(len(devs), H), radius)

    def job(slab):
        def fn(dev):
            rc = lib.mtb_filter_host_rows(
                src.ctypes.data, out[slab.a:slab.b].ctypes.data, bits, H, W, slab.a, slab.b,
                int(radius), int(rank), lut_ptr, 0, dev)
            _lib.check(rc)
        return fn

    _on_devices([(dev, job(sl)) for sl, dev in zip(slabs, devs)])
    return out


def filter_image(
    image,
    n: int,
    *,
    rank=None,
    percentile=None,
    max_error: int = 1,
    mode: str = "uniform",
    profile=None,
    topology: TreeTopology | None = None,
    counting: bool = True,
    bands: int = 1,
    devices=None,
) -> tuple[GrayImage, OpCounters]:
    """Rank-filter a full frame on the GPU (engine.py:209-262 semantics).

    Returns the output image and an OpCounters whose tallies are zero (the
    CPU-tree tallies have no GPU counterpart) and whose ``pixels`` is the
    number of output pixels.  ``counting`` is accepted for compatibility.
    ``devices``: optional list of CUDA devices to spread row slabs over
    (one slab per device, halos read from the host frame, no collective).
    """
    image = as_gray_image(image)
    n = check_window(n, image.width, image.height)
    rank = resolve_rank(n, rank, percentile)
    need_map = False
    if topology is None:
        if mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {mode!r}")
        if mode == "adaptive":
            if profile is not None and profile.weights.size != 1 << image.bit_depth:
                raise ValueError(
                    f"profile length {profile.weights.size} does not match "
                    f"{image.bit_depth}-bit data"
                )
            # the adaptive tree only changes results at max_error > 1
            need_map = int(max_error) > 1
        else:
            topology = uniform_topology(image.bit_depth)
    bands = int(bands)
    if bands < 1:
        raise ValueError(f"bands must be >= 1, got {bands}")
    bands = min(bands, image.height)
    max_error = check_max_error(max_error)
    if need_map:
        topology = resolve_topology(image, n, mode, profile)
    if topology is not None and topology.bit_depth != image.bit_depth:
        raise ValueError(f"topology is {topology.bit_depth}-bit, image is {image.bit_depth}-bit")
    lut = value_map(topology, max_error) if topology is not None else None
    # `bands` does not change results (engine.py:243-262); the library picks
    # its own row bands / streaming for the copy-filter overlap
    out = _run(image.pixels, image.bit_depth, n // 2, rank, lut, devices)
    return GrayImage(out, image.bit_depth), OpCounters(pixels=image.width * image.height)


def median_filter(image, radius: int, bit_depth: int | None = None, adaptive: bool = False,
                  rank=None, devices=None) -> np.ndarray:
    """North-star convenience: radius r (window n = 2r+1), bit depth,
    adaptive flag; returns the filtered array (same dtype)."""
    img = as_gray_image(image, bit_depth) if isinstance(image, GrayImage) else GrayImage(
        np.asarray(image), bit_depth)
    out, _ = filter_image(img, 2 * int(radius) + 1, rank=rank,
                          mode="adaptive" if adaptive else "uniform", devices=devices)
    return out.pixels


def filter_host_buffer(src: np.ndarray, radius: int, rank: int | None = None,
                       lut: np.ndarray | None = None, out: np.ndarray | None = None,
                       device=None) -> np.ndarray:
    """Whole-frame call through the C ABI's HOST-buffer entry
    (mtb_filter_host): what a ctypes binding in the reference would use.
    The library pipelines row bands (copy in / filter / copy out overlap);
    a page-locked ``src`` (e.g. a numpy view of a pinned torch tensor) also
    enables the single streaming launch for r >= 12.  ``out``: optional
    C-contiguous destination of src's shape and dtype.  ``device``: CUDA
    device (default: the current one)."""
    src = np.ascontiguousarray(src)
    if src.dtype not in (np.uint8, np.uint16):
        raise ValueError("src must be uint8 or uint16")
    bits = 8 if src.dtype == np.uint8 else 16
    if src.ndim != 2:
        raise ValueError("src must be a 2-D array")
    H, W = src.shape
    n = 2 * int(radius) + 1
    if rank is None:
        rank = (n * n + 1) // 2
    if out is None:
        dst = np.empty_like(src)
    else:
        if out.shape != src.shape or out.dtype != src.dtype or not out.flags.c_contiguous:
            raise ValueError("out must be C-contiguous with src's shape and dtype")
        dst = out
    lut = _check_lut(lut, src.dtype, bits)
    lut_ptr = lut.ctypes.data if lut is not None else None
    dev = _devices(None if device is None else [device])[0]
    rc = _lib.load().mtb_filter_host_rows(
        src.ctypes.data_as(ctypes.c_void_p), dst.ctypes.data_as(ctypes.c_void_p), bits, H, W, 0, H,
        int(radius), int(rank), lut_ptr, 0, dev)
    _lib.check(rc)
    return dst


def filter_host_frames(srcs, radii, ranks=None, lut: np.ndarray | None = None,
                       outs=None, device=None) -> list:
    """A sequence of host frames of one shape and dtype through the C ABI's
    multi-frame HOST entry (mtb_filter_host_frames): frame i+1's copy in and
    frame i-1's copy out overlap frame i's filtering.  ``radii``: one radius
    per frame (or one int for all); ``ranks``: per-frame 1-based ranks or
    None (medians); ``outs``: optional C-contiguous destinations.  Page-locked
    frames (numpy views of pinned torch tensors) make the copies
    asynchronous.  ``device``: CUDA device (default: the current one).
    Returns the list of filtered frames."""
    srcs = [np.ascontiguousarray(s) for s in srcs]
    if not srcs:
        return []
    s0 = srcs[0]
    if s0.dtype not in (np.uint8, np.uint16) or s0.ndim != 2:
        raise ValueError("frames must be 2-D uint8 or uint16 arrays")
    if any(s.shape != s0.shape or s.dtype != s0.dtype for s in srcs):
        raise ValueError("all frames must share one shape and dtype")
    n = len(srcs)
    radii = [int(radii)] * n if np.isscalar(radii) else [int(r) for r in radii]
    if len(radii) != n:
        raise ValueError("one radius per frame")
    for r in radii:
        if r < 1:
            raise ValueError(f"window must be an odd integer >= 3, got {2 * r + 1}")
    if outs is None:
        outs = [np.empty_like(s0) for _ in range(n)]
    elif len(outs) != n or any(o.shape != s0.shape or o.dtype != s0.dtype or not o.flags.c_contiguous
                                for o in outs):
        raise ValueError("outs must be C-contiguous frames of the inputs' shape and dtype")
    H, W = s0.shape
    bits = 8 if s0.dtype == np.uint8 else 16
    P = ctypes.c_void_p * n
    src_arr = P(*[s.ctypes.data for s in srcs])
    dst_arr = P(*[o.ctypes.data for o in outs])
    rad_arr = (ctypes.c_int32 * n)(*radii)
    rank_arr = None
    if ranks is not None:
        if len(ranks) != n:
            raise ValueError("one rank per frame")
        rank_arr = (ctypes.c_int64 * n)(*[int(k) for k in ranks])
    lut = _check_lut(lut, s0.dtype, bits)
    lut_ptr = lut.ctypes.data if lut is not None else None
    lib = _lib.load()
    dev = _devices(None if device is None else [device])[0]
    _lib.check(lib.mtb_set_device(dev))
    rc = lib.mtb_filter_host_frames(
        ctypes.cast(src_arr, ctypes.c_void_p), ctypes.cast(dst_arr, ctypes.c_void_p),
        ctypes.cast(rad_arr, ctypes.c_void_p),
        ctypes.cast(rank_arr, ctypes.c_void_p) if rank_arr is not None else None,
        n, bits, H, W, lut_ptr, 0)
    _lib.check(rc)
    return outs


def filter_images(images, n: int, *, rank=None, percentile=None, max_error: int = 1,
                  mode: str = "uniform", devices=None, outs=None) -> list:
    """A batch of same-shape images (config 5), each filtered exactly as
    ``filter_image(image, n, ...)`` would: the reference's per-image loop
    (engine.py:209-262) as one call.  The images are split into contiguous
    runs, one per device (``plan_images``); each device's host thread sends
    its run through the frame-sequence entry (mtb_filter_host_frames: image
    i+1's copy in and image i-1's copy out overlap image i's filter).
    Returns the list of output pixel arrays."""
    imgs = [as_gray_image(im) for im in images]
    if not imgs:
        return []
    g0 = imgs[0]
    if any(g.pixels.shape != g0.pixels.shape or g.bit_depth != g0.bit_depth for g in imgs):
        raise ValueError("all images must share one shape and bit depth")
    n = check_window(n, g0.width, g0.height)
    rank = resolve_rank(n, rank, percentile)
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}, got {mode!r}")
    max_error = check_max_error(max_error)
    if outs is None:
        outs = [np.empty_like(g.pixels) for g in imgs]
    devs = _devices(devices)
    runs = plan_images(len(imgs), len(devs))
    per_image_map = mode == "adaptive" and max_error > 1  # topology depends on each image
    lut = None if per_image_map else value_map(uniform_topology(g0.bit_depth), max_error)

    def job(i0, i1):
        def fn(dev):
            if i0 == i1:
                return
            if per_image_map:
                for i in range(i0, i1):
                    t = resolve_topology(imgs[i], n, mode, None)
                    filter_host_buffer(imgs[i].pixels, n // 2, rank, lut=value_map(t, max_error),
                                       out=outs[i], device=dev)
                return
            filter_host_frames([g.pixels for g in imgs[i0:i1]], n // 2, ranks=[rank] * (i1 - i0),
                               lut=lut, outs=outs[i0:i1], device=dev)
        return fn

    _on_devices([(dev, job(i0, i1)) for (i0, i1), dev in zip(runs, devs)])
    return outs
