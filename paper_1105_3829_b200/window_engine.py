"""Stepwise engine API (the reference's WindowEngine, engine.py:36-184) as a
host emulation over the GPU path.

`step()` yields `(value, error_bound)` per output pixel in scan order --
the lower bound and width of the interval where the reference's descent
stops, both pure functions of the exact rank value (topology.
descent_intervals) -- and raises StopIteration past the last pixel.  The
exact frame is computed on the GPU at the first step; `run()` is the
whole-frame call, only before the first `step()`.  `counters` reports the
`counting=False` view (zero tallies, `pixels` = pixels emitted).
"""

from __future__ import annotations

import numpy as np

from .counters import OpCounters
from .engine import filter_host_buffer
from .topology import TreeTopology, descent_intervals
from .validation import as_gray_image, check_max_error, check_window, resolve_rank


class WindowEngine:
    def __init__(self, image, n: int, topology: TreeTopology, rank=None, max_error: int = 1,
                 on_demand: bool = True, counting: bool = True):
        image = as_gray_image(image)
        if topology.bit_depth != image.bit_depth:
            raise ValueError(f"topology is {topology.bit_depth}-bit, image is {image.bit_depth}-bit")
        self.image = image
        self.n = check_window(n, image.width, image.height)
        self.topology = topology
        self.rank = resolve_rank(self.n, rank)
        self.max_error = check_max_error(max_error)
        self.on_demand = bool(on_demand)  # window update policy: no effect on results
        self.counting = bool(counting)
        self._pos = 0
        self._stepping = False
        self._exact = None
        self._lo = self._width = None

    @property
    def position(self) -> tuple[int, int]:
        """(x, y) of the next output pixel."""
        return self._pos % self.image.width, self._pos // self.image.width

    @property
    def counters(self) -> OpCounters:
        return OpCounters(pixels=self._pos)

    def __iter__(self):
        return self

    def __next__(self):
        return self.step()

    def _frame(self) -> np.ndarray:
        if self._exact is None:
            self._exact = filter_host_buffer(self.image.pixels, self.n // 2, self.rank).ravel()
            self._lo, self._width = descent_intervals(self.topology, self.max_error)
        return self._exact

    def step(self) -> tuple[int, int]:
        W, H = self.image.width, self.image.height
        if self._pos >= W * H:
            raise StopIteration
        self._stepping = True
        v = int(self._frame()[self._pos])
        self._pos += 1
        return int(self._lo[v]), int(self._width[v])

    def run(self) -> np.ndarray:
        """Whole frame (values as `step()` would emit them)."""
        if self._stepping or self._pos:
            raise RuntimeError("run() requires a fresh engine (step() already used)")
        exact = self._frame().reshape(self.image.height, self.image.width)
        self._pos = self.image.width * self.image.height
        return self._lo[exact].astype(self.image.pixels.dtype)
