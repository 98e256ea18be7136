"""Seeded synthetic inputs for the five BASELINE.json configs.

The reference publishes no datasets for this path,
so these generators ARE the workloads: shapes, value distributions and seeds
follow SURVEY.md section 8(d).  Every generator takes a size override so the
tests can draw smaller images from the same distribution.
"""

from __future__ import annotations

import numpy as np


def cfg1_uniform_u8(h: int = 512, w: int = 512, seed: int = 0) -> np.ndarray:
    """Config 1: i.i.d. uniform [0,255] u8 (512x512, seed 0)."""
    return np.random.default_rng(seed).integers(0, 256, (h, w), dtype=np.uint8)


def cfg2_blur_sp_u8(h: int = 4096, w: int = 4096, seed: int = 1,
                    sigma: float = 8.0, impulse: float = 0.05) -> np.ndarray:
    """Config 2: Gaussian-blurred white noise (sigma 8 px) rescaled to
    [0,255], plus 5% salt-and-pepper impulses."""
    from scipy.ndimage import gaussian_filter

    rng = np.random.default_rng(seed)
    f = gaussian_filter(rng.standard_normal((h, w)), sigma)
    lo, hi = float(f.min()), float(f.max())
    px = np.rint(255.0 * (f - lo) / max(hi - lo, 1e-300)).astype(np.uint8)
    m = rng.random((h, w)) < impulse
    px[m] = np.where(rng.random(int(m.sum())) < 0.5, 0, 255).astype(np.uint8)
    return px


def cfg3_uniform_u16(h: int = 4096, w: int = 4096, seed: int = 2) -> np.ndarray:
    """Config 3: i.i.d. uniform [0,65535] u16."""
    return np.random.default_rng(seed).integers(0, 65536, (h, w)).astype(np.uint16)


def cfg4_three_gauss_u16(h: int = 8192, w: int = 8192, seed: int = 3) -> np.ndarray:
    """Config 4: compact-histogram u16, per-pixel mixture of 3 Gaussians
    (weights .6/.3/.1, means 800/1500/4000, sigma 60/120/200), clipped."""
    rng = np.random.default_rng(seed)
    comp = rng.choice(3, size=(h, w), p=[0.6, 0.3, 0.1])
    means = np.array([800.0, 1500.0, 4000.0])
    sig = np.array([60.0, 120.0, 200.0])
    v = rng.normal(means[comp], sig[comp])
    return np.clip(np.rint(v), 0, 65535).astype(np.uint16)


def cfg5_batch_u8(count: int = 64, h: int = 2048, w: int = 2048) -> np.ndarray:
    """Config 5: batch of u8 images; first half uniform, second half as
    config 2, image i seeded with 100+i."""
    out = np.empty((count, h, w), dtype=np.uint8)
    half = count // 2
    for i in range(count):
        if i < half:
            out[i] = cfg1_uniform_u8(h, w, seed=100 + i)
        else:
            out[i] = cfg2_blur_sp_u8(h, w, seed=100 + i)
    return out


CONFIG_RADII = {
    1: (5,),
    2: (1, 3, 7, 15, 31, 63),
    3: (3, 7, 15, 31),
    4: (15, 31),
    5: (7, 25),
}
