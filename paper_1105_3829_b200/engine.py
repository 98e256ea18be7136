"""Drop-in ``filter_image``: the reference's call surface on the B200 path.

Mirrors pkg/src/medtree/engine.py:209-262 -- same arguments, same
validation order and ValueErrors, same ``(GrayImage, OpCounters)`` return --
but every output pixel is computed by the sm_100a kernels behind the C ABI
(include/medtree_b200.h).  PyTorch is only the device allocator / stream /
copy engine.  There is no CPU path: without a CUDA device the call raises.

Row slabs.  ``bands=k`` keeps the reference's meaning (horizontal bands
with n//2 halo rows, identical output, engine.py:243-262); on the GPU a band
is one launch over rows [a,b) of the device-resident frame.  ``devices=[...]``
additionally spreads the bands over several GPUs: each GPU receives its
rows plus r halo rows straight from the host copy and returns its rows --
no collective is involved.
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


def _tdtype(bit_depth: int):
    torch = _t()
    return torch.uint8 if bit_depth == 8 else torch.uint16


def _stream_handle(stream) -> int:
    torch = _t()
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def rank_filter(
    src,
    radius: int,
    rank: int | None = None,
    *,
    out=None,
    lut=None,
    adaptive: bool = False,
    rows: tuple[int, int] | None = None,
    src_row0: int = 0,
    height: int | None = None,
    stream=None,
):
    """Device-resident rank filter (no host copies).

    ``src``: CUDA tensor uint8/uint16, shape (H, W) or (B, H, W).  For a
    2-D slab, ``src`` holds global rows [src_row0, src_row0+src.shape[0]) of
    an image with ``height`` rows and ``rows=(a, b)`` selects the output
    rows; ``out`` then has b-a rows.  ``lut``: optional CUDA tensor with
    2^bit_depth entries applied to the exact rank value.
    Returns ``out``.
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
    n = 2 * int(radius) + 1
    if rank is None:
        rank = (n * n + 1) // 2
    flags = _lib.FLAG_ADAPTIVE if adaptive else 0
    lib = _lib.load()
    sh = _stream_handle(stream)
    lut_ptr = None
    if lut is not None:
        if lut.device != src.device or lut.dtype != src.dtype or lut.numel() != (1 << bits):
            raise ValueError("lut must be a CUDA tensor of 2^bit_depth entries, src dtype")
        lut_ptr = lut.data_ptr()
    if src.dim() == 3:
        B, H, W = src.shape
        if out is None:
            out = torch.empty((B, H, W), dtype=src.dtype, device=src.device)
        fn = lib.mtb_median_batch_u8 if bits == 8 else lib.mtb_median_batch_u16
        rc = fn(src.data_ptr(), src.stride(0), src.stride(1), out.data_ptr(), out.stride(0),
                out.stride(1), B, H, W, int(radius), int(rank), lut_ptr, flags, sh)
        _lib.check(rc)
        return out
    if src.dim() != 2:
        raise ValueError("src must be 2-D (H, W) or 3-D (B, H, W)")
    src_rows, W = src.shape
    H = src_rows if height is None else int(height)
    a, b = (0, H) if rows is None else (int(rows[0]), int(rows[1]))
    if out is None:
        out = torch.empty((b - a, W), dtype=src.dtype, device=src.device)
    if out.stride(-1) != 1 or out.shape[0] < b - a or out.shape[1] != W:
        raise ValueError("out must be (rows, W) with contiguous rows")
    fn = lib.mtb_median_u8 if bits == 8 else lib.mtb_median_u16
    rc = fn(src.data_ptr(), src.stride(0), int(src_row0), int(src_rows), out.data_ptr(),
            out.stride(0), H, W, a, b, int(radius), int(rank), lut_ptr, flags, sh)
    _lib.check(rc)
    return out


def _band_edges(H: int, bands: int) -> list[tuple[int, int]]:
    """engine.py:248: numpy.linspace(0, H, bands+1, dtype=int) edges."""
    edges = np.linspace(0, H, bands + 1, dtype=int)
    return [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if a != b]


def _run(px: np.ndarray, bits: int, radius: int, rank: int, lut: np.ndarray | None,
         bands: int, devices, adaptive: bool) -> np.ndarray:
    torch = _t()
    H, W = px.shape
    tdt = _tdtype(bits)
    host = torch.from_numpy(np.ascontiguousarray(px))
    if devices is None:
        devices = [torch.cuda.current_device()]
    devices = [torch.device("cuda", d) if isinstance(d, int) else torch.device(d) for d in devices]
    if len(devices) == 1:
        # one device: the library's host-buffer entry, which pipelines row
        # bands (copy in / filter / copy out overlap); `bands` does not change
        # results and the library picks its own band count
        with torch.cuda.device(devices[0]):
            return filter_host_buffer(px, radius, rank, lut=lut, adaptive=adaptive)
    # several GPUs: one slab per device (each may still be cut into bands)
    pinned = host.pin_memory()
    result = torch.empty((H, W), dtype=tdt).pin_memory()
    slabs = _band_edges(H, min(len(devices), H))
    pending = []
    for (a, b), dev in zip(slabs, devices):
        with torch.cuda.device(dev):
            s = torch.cuda.Stream(dev)
            with torch.cuda.stream(s):
                top, bot = max(0, a - radius), min(H, b + radius)
                src = torch.empty((bot - top, W), dtype=tdt, device=dev)
                src.copy_(pinned[top:bot], non_blocking=True)
                dlut = torch.from_numpy(lut).to(dev, non_blocking=True) if lut is not None else None
                out = torch.empty((b - a, W), dtype=tdt, device=dev)
                sub = _band_edges(b - a, max(1, min(bands, b - a)))
                for sa, sb in sub:
                    rank_filter(src, radius, rank, out=out[sa:sb], lut=dlut, adaptive=adaptive,
                                rows=(a + sa, a + sb), src_row0=top, height=H, stream=s)
                result[a:b].copy_(out, non_blocking=True)
                pending.append((s, src, out, dlut))
    for s, *_ in pending:
        s.synchronize()
    return result.numpy()


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
    ``devices``: optional list of CUDA devices to spread row slabs over.
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
    out = _run(image.pixels, image.bit_depth, n // 2, rank, lut, bands, devices,
               adaptive=(mode == "adaptive"))
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
                       lut: np.ndarray | None = None, adaptive: bool = False,
                       out: np.ndarray | None = None) -> np.ndarray:
    """Whole-frame call through the C ABI's HOST-buffer entry
    (mtb_filter_host): what a ctypes binding in the reference would use.
    The library pipelines row bands (copy in / filter / copy out overlap);
    page-locked ``src`` / ``out`` buffers (e.g. numpy views of pinned torch
    tensors) make the copies asynchronous.  ``out``: optional C-contiguous
    destination of src's shape and dtype."""
    src = np.ascontiguousarray(src)
    bits = 8 if src.dtype == np.uint8 else 16
    if src.dtype not in (np.uint8, np.uint16):
        raise ValueError("src must be uint8 or uint16")
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
    lut_ptr = None
    if lut is not None:
        lut = np.ascontiguousarray(lut, dtype=src.dtype)
        lut_ptr = lut.ctypes.data
    rc = _lib.load().mtb_filter_host(
        src.ctypes.data_as(ctypes.c_void_p), dst.ctypes.data_as(ctypes.c_void_p), bits, H, W,
        int(radius), int(rank), lut_ptr, _lib.FLAG_ADAPTIVE if adaptive else 0)
    _lib.check(rc)
    return dst


def filter_host_frames(srcs, radii, ranks=None, lut: np.ndarray | None = None,
                       outs=None) -> list:
    """A sequence of host frames of one shape and dtype through the C ABI's
    multi-frame HOST entry (mtb_filter_host_frames): frame i+1's copy in and
    frame i-1's copy out overlap frame i's filtering.  ``radii``: one radius
    per frame (or one int for all); ``ranks``: per-frame 1-based ranks or
    None (medians); ``outs``: optional C-contiguous destinations.  Page-locked
    frames (numpy views of pinned torch tensors) make the copies
    asynchronous.  Returns the list of filtered frames."""
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
    lut_ptr = None
    if lut is not None:
        lut = np.ascontiguousarray(lut, dtype=s0.dtype)
        lut_ptr = lut.ctypes.data
    rc = _lib.load().mtb_filter_host_frames(
        ctypes.cast(src_arr, ctypes.c_void_p), ctypes.cast(dst_arr, ctypes.c_void_p),
        ctypes.cast(rad_arr, ctypes.c_void_p),
        ctypes.cast(rank_arr, ctypes.c_void_p) if rank_arr is not None else None,
        n, bits, H, W, lut_ptr, 0)
    _lib.check(rc)
    return outs
