"""Tree topologies and the value maps they induce on the GPU path.

The reference descends an interval tree per output pixel and returns the
lower bound of the node where it stops (uniform: after `levels` bisection
steps, pkg/src/medtree/_kernels.py:229-253; adaptive: when a node is no
wider than max_error or is a leaf, :256-289).  That descent always follows
the path to the exact rank value v, so its output is a pure function of v.
The GPU kernels compute v exactly and apply that function as a lookup
table (``value_map``); at max_error=1 with unit leaves the map is the
identity and no table is used.

The adaptive builder restates pkg/src/medtree/topology.py:112-264 (profile,
weighted-median splits, flat preorder layout) so that mode="adaptive" with
max_error > 1 is reproduced exactly.  It only runs on the host, once per
call, and only when the value map is not the identity.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .image import GrayImage


class TreeTopology:
    """Split structure over [0, 2^bit_depth) (topology.py:57-102)."""

    def __init__(self, bit_depth, mode, leaf_precision=1, lo=None, up=None, leaf=None, span=None):
        self.bit_depth = int(bit_depth)
        self.mode = mode
        self.leaf_precision = int(leaf_precision)
        self.n_values = 1 << self.bit_depth
        self.lo, self.up, self.leaf, self.span = lo, up, leaf, span
        self.slots = self.n_values if mode == "uniform" else len(up)

    def __repr__(self) -> str:
        return f"TreeTopology(d={self.bit_depth}, {self.mode}, slots={self.slots})"


def uniform_topology(bit_depth: int) -> TreeTopology:
    """topology.py:105-109."""
    if not 1 <= int(bit_depth) <= 16:
        raise ValueError(f"bit_depth must be in 1..16, got {bit_depth}")
    return TreeTopology(bit_depth, "uniform")


@dataclass
class FrequencyProfile:
    """topology.py:112-141."""

    weights: np.ndarray
    source: str = "source-histogram"

    def __post_init__(self):
        w = np.asarray(self.weights, dtype=np.float64)
        if w.ndim != 1:
            raise ValueError("profile weights must be one-dimensional")
        if w.size & (w.size - 1) or w.size < 2:
            raise ValueError(f"profile length must be a power of two, got {w.size}")
        if not np.isfinite(w).all():
            raise ValueError("profile weights must be finite")
        if (w < 0).any():
            raise ValueError("profile weights must be non-negative")
        self.weights = w

    @property
    def bit_depth(self) -> int:
        return int(self.weights.size).bit_length() - 1

    @property
    def total(self) -> float:
        return float(self.weights.sum())

    @property
    def is_degenerate(self) -> bool:
        return self.total <= 0.0


def source_histogram(image: GrayImage) -> FrequencyProfile:
    """topology.py:144-147."""
    counts = np.bincount(image.pixels.ravel(), minlength=1 << image.bit_depth)
    return FrequencyProfile(counts.astype(np.float64), "source-histogram")


def box_mean(image: GrayImage, n: int) -> np.ndarray:
    """topology.py:150-162: float64 running box mean, replicate borders,
    via a summed-area table over the edge-padded image."""
    if n < 1 or n % 2 == 0:
        raise ValueError(f"window must be odd and positive, got {n}")
    h, w = image.pixels.shape
    if n > 2 * min(h, w) + 1:
        raise ValueError(f"window {n} larger than twice the image extent {h}x{w}")
    pad = np.pad(image.pixels.astype(np.float64), n // 2, mode="edge")
    sat = np.zeros((h + n, w + n))
    np.cumsum(pad, axis=0, out=pad)
    np.cumsum(pad, axis=1, out=sat[1:, 1:])
    total = sat[n:, n:] - sat[:-n, n:] - sat[n:, :-n] + sat[:-n, :-n]
    return total / float(n * n)


def estimate_median_profile(image: GrayImage, n: int) -> FrequencyProfile:
    """topology.py:165-171."""
    means = np.clip(np.rint(box_mean(image, n)).astype(np.int64), 0, (1 << image.bit_depth) - 1)
    counts = np.bincount(means.ravel(), minlength=1 << image.bit_depth)
    return FrequencyProfile(counts.astype(np.float64), "median-estimate")


def mix_profiles(source: FrequencyProfile, median: FrequencyProfile) -> FrequencyProfile:
    """topology.py:174-190: 1:1 mix by mass; empty inputs contribute nothing."""
    if source.weights.size != median.weights.size:
        raise ValueError(
            f"profile length mismatch: {source.weights.size} vs {median.weights.size}"
        )
    mixed = np.zeros_like(source.weights)
    for prof in (source, median):
        if not prof.is_degenerate:
            mixed += prof.weights / prof.total
    return FrequencyProfile(mixed, "mixed")


def _weighted_median_split(cum: np.ndarray, a: int, b: int) -> int:
    """topology.py:193-211: split [a,b) at the profile's half-mass point;
    of the two bracketing integer positions the better balanced wins, then
    the one nearer the midpoint, then the smaller; zero mass bisects."""
    mass = cum[b] - cum[a]
    if mass <= 0.0:
        return a + (b - a) // 2
    half = cum[a] + mass / 2.0
    s = min(int(np.searchsorted(cum[a + 1:b], half, side="left")) + a + 1, b - 1)
    if s == a + 1:
        return s
    mid = 0.5 * (a + b)
    best = None
    for cand in (s - 1, s):
        key = (abs(2.0 * (cum[cand] - cum[a]) - mass), abs(cand - mid), cand)
        if best is None or key < best[0]:
            best = (key, cand)
    return best[1]


def build_adaptive_topology(profile: FrequencyProfile, leaf_precision: int = 1) -> TreeTopology:
    """topology.py:214-264: explicit (left) nodes in flat preorder -- each
    node, then its left subtree, then the subtree under its implicit right
    sibling; span[k] = size of slot k's explicit subtree."""
    if leaf_precision < 1:
        raise ValueError(f"leaf_precision must be >= 1, got {leaf_precision}")
    nv = profile.weights.size
    cum = np.concatenate(([0.0], np.cumsum(profile.weights)))
    lo, up, leaf, span = [0], [nv], [0], [0]
    todo = [(0, 0, nv)]  # (kind, a, b); kind 1 = close slot a
    while todo:
        kind, a, b = todo.pop()
        if kind == 1:
            span[a] = len(up) - a
            continue
        if b - a <= leaf_precision:
            continue
        s = _weighted_median_split(cum, a, b)
        k = len(up)
        lo.append(a)
        up.append(s)
        leaf.append(1 if s - a <= leaf_precision else 0)
        span.append(0)
        todo += [(0, s, b), (1, k, 0), (0, a, s)]
    span[0] = len(up)
    return TreeTopology(
        nv.bit_length() - 1, "adaptive", leaf_precision,
        lo=np.asarray(lo, dtype=np.int64), up=np.asarray(up, dtype=np.int64),
        leaf=np.asarray(leaf, dtype=np.uint8), span=np.asarray(span, dtype=np.int64),
    )


MODES = ("uniform", "adaptive", "unconditional")


def resolve_topology(image: GrayImage, n: int, mode: str, profile=None) -> TreeTopology:
    """engine.py:187-206."""
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}, got {mode!r}")
    if mode != "adaptive":
        return uniform_topology(image.bit_depth)
    if profile is None:
        profile = mix_profiles(source_histogram(image), estimate_median_profile(image, n))
    if profile.weights.size != 1 << image.bit_depth:
        raise ValueError(
            f"profile length {profile.weights.size} does not match {image.bit_depth}-bit data"
        )
    if profile.is_degenerate:
        return uniform_topology(image.bit_depth)
    return build_adaptive_topology(profile)


def uniform_levels(bit_depth: int, max_error: int) -> int:
    """engine.py:32-35."""
    levels = bit_depth - (int(max_error).bit_length() - 1)
    return max(0, min(bit_depth, levels))


def descent_intervals(topology: TreeTopology, max_error: int) -> tuple[np.ndarray, np.ndarray]:
    """(lo, width) of the interval where the reference's rank descent stops,
    for every exact rank value v (int64 arrays of 2^d entries).  Uniform:
    lo = v & ~(w-1), width w = 2^(d-levels) (_kernels.py:229-253).  Adaptive:
    the first node on v's root-to-leaf path no wider than max_error, or
    whose child is a leaf, or whose right part is within the leaf precision
    (_kernels.py:256-289)."""
    d = topology.bit_depth
    nv = 1 << d
    v = np.arange(nv, dtype=np.int64)
    if topology.mode == "uniform":
        w = 1 << (d - uniform_levels(d, max_error))
        return v & ~(w - 1), np.full(nv, w, dtype=np.int64)
    up, leaf, span = topology.up, topology.leaf.astype(bool), topology.span
    prec = topology.leaf_precision
    lo = np.zeros(nv, dtype=np.int64)
    hi = np.full(nv, nv, dtype=np.int64)
    pos = np.ones(nv, dtype=np.int64)
    live = hi - lo > max_error
    while live.any():
        idx = np.nonzero(live)[0]
        p = pos[idx]
        s = up[p]
        go_left = v[idx] < s
        li, ri = idx[go_left], idx[~go_left]
        hi[li] = s[go_left]
        stop_l = leaf[p[go_left]]
        pos[li] = p[go_left] + 1
        lo[ri] = s[~go_left]
        stop_r = hi[ri] - lo[ri] <= prec
        pos[ri] = p[~go_left] + span[p[~go_left]]
        live[li[stop_l]] = False
        live[ri[stop_r]] = False
        still = np.nonzero(live)[0]
        live[still] = hi[still] - lo[still] > max_error
    return lo, hi - lo


def value_map(topology: TreeTopology, max_error: int) -> np.ndarray | None:
    """Output value as a function of the exact rank value (the lower bound
    of descent_intervals), or None for the identity."""
    lo, _ = descent_intervals(topology, max_error)
    if np.array_equal(lo, np.arange(lo.size, dtype=np.int64)):
        return None
    return lo.astype(np.uint8 if topology.bit_depth <= 8 else np.uint16)
