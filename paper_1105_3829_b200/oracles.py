"""Independent reference filters (the reference's oracles.py:36-66 surface).

The reference ships three CPU ground-truth filters (full sort, quickselect,
sliding histogram) for its `compare` command and tests.  This package has no
CPU compute path, so every kind runs the GPU brute-force selection
(`mtb_rank_bruteforce`: per pixel, the value's bits decided from the top by
counting passes over the n x n window) -- an algorithm that shares nothing
with the fast kernels.  `huang_filter` also returns the reference's
histogram-update addition count, which is a closed form of the geometry
(2n per horizontal step, n^2 per row start; _kernels.py:403-446).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .image import GrayImage
from .validation import as_gray_image, check_window, resolve_rank

ORACLE_KINDS = ("full_sort", "quickselect", "huang_histogram")


def _bruteforce(image: GrayImage, n: int, rank: int) -> GrayImage:
    from .engine import _t

    torch = _t()
    px = np.ascontiguousarray(image.pixels)
    H, W = px.shape
    src = torch.from_numpy(px).cuda()
    dst = torch.empty_like(src)
    rc = _lib.load().mtb_rank_bruteforce(src.data_ptr(), W, dst.data_ptr(), W, image.bit_depth, H, W,
                                         n // 2, int(rank), torch.cuda.current_stream().cuda_stream)
    _lib.check(rc)
    return GrayImage(dst.cpu().numpy(), image.bit_depth)


def oracle_median_filter(image, n: int, rank=None, kind: str = "full_sort") -> GrayImage:
    """Rank-filter with the independent selection (any of the reference's
    oracle kinds; they are exact, so they agree)."""
    image = as_gray_image(image)
    n = check_window(n, image.width, image.height)
    rank = resolve_rank(n, rank)
    if kind not in ORACLE_KINDS:
        raise ValueError(f"oracle kind must be one of {ORACLE_KINDS}, got {kind!r}")
    return _bruteforce(image, n, rank)


def huang_adds(height: int, width: int, n: int) -> int:
    """Histogram-update additions of the sliding-histogram filter."""
    return height * (n * n + (width - 1) * 2 * n)


def huang_filter(image, n: int, rank=None) -> tuple[GrayImage, int]:
    """(filtered image, histogram-update additions) like the reference's
    sliding-histogram oracle."""
    image = as_gray_image(image)
    n = check_window(n, image.width, image.height)
    rank = resolve_rank(n, rank)
    return _bruteforce(image, n, rank), huang_adds(image.height, image.width, n)
