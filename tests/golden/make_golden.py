"""Generate the golden fixtures from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src and
records, for seeded inputs:

* ``small_cases.npz``   -- inputs AND outputs of small cases covering the
  reference's own exactness matrix (tests/test_engine.py:25-99,
  tests/test_acceptance.py:46-93): 8/16-bit, windows 3..51, ranks,
  percentiles, all three modes, reduced precision, degenerate shapes.
* ``digests.json``      -- SHA-256 of reference outputs for config-shaped
  inputs too large to commit (regenerated from ``workloads.py`` at test time).
* ``topologies.npz``    -- adaptive topology arrays built by the reference
  (topology.py:214-264) for a few images, to pin the restated builder.

Nothing at GPU-test time reads /root/reference; only these files travel.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import medtree  # noqa: E402  (the reference)
from medtree.engine import resolve_topology  # noqa: E402

import workloads  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def small_cases():
    rng = np.random.default_rng(20261020)
    cases = []
    # (bit_depth, n, mode, h, w, rank-or-None, percentile, max_error, flavor)
    for d in (8, 16):
        for n in (3, 5, 11, 25, 51):
            for mode in ("uniform", "adaptive", "unconditional"):
                lo = max(6, n // 2)
                cap = 20 if (mode == "unconditional" and d == 16) else 40
                h = int(rng.integers(lo, max(lo + 1, cap)))
                w = int(rng.integers(lo, max(lo + 1, cap)))
                cases.append((d, n, mode, h, w, None, None, 1, "uniform_noise"))
    for rank in (1, 5, 9):
        cases.append((8, 3, "uniform", 16, 14, rank, None, 1, "uniform_noise"))
    cases.append((8, 3, "uniform", 12, 15, None, 1.0 / 9.0, 1, "uniform_noise"))
    cases.append((8, 3, "uniform", 12, 15, None, 1.0, 1, "uniform_noise"))
    cases.append((16, 7, "uniform", 21, 17, None, 0.1, 1, "normal_noise"))
    cases.append((8, 9, "uniform", 30, 22, 80, None, 1, "two_mode"))
    for shape in ((1, 40), (40, 1), (2, 19), (19, 2), (1, 1), (3, 3)):
        cases.append((8, 3, "uniform", shape[0], shape[1], None, None, 1, "uniform_noise"))
    cases.append((16, 3, "uniform", 1, 33, None, None, 1, "uniform_noise"))
    # windows larger than the image (n up to 2*min(H,W)+1, validation.py:24)
    cases.append((8, 9, "uniform", 4, 7, None, None, 1, "uniform_noise"))
    cases.append((16, 13, "uniform", 6, 9, None, None, 1, "uniform_noise"))
    cases.append((8, 41, "uniform", 20, 31, None, None, 1, "normal_noise"))
    # reduced precision, uniform and adaptive
    for me in (2, 3, 16, 20, 1000):
        cases.append((16, 5, "uniform", 24, 24, None, None, me, "uniform_noise"))
    for me in (2, 16):
        cases.append((8, 5, "uniform", 24, 24, None, None, me, "normal_noise"))
        cases.append((8, 5, "adaptive", 24, 24, None, None, me, "two_mode"))
        cases.append((16, 7, "adaptive", 24, 24, None, None, me, "two_mode"))
    # a few larger frames
    cases.append((8, 51, "uniform", 96, 80, None, None, 1, "uniform_noise"))
    cases.append((16, 25, "adaptive", 64, 64, None, None, 1, "two_mode"))
    cases.append((16, 31, "uniform", 70, 66, None, None, 1, "uniform_noise"))

    inputs, outputs, meta = {}, {}, []
    for i, (d, n, mode, h, w, rank, pct, me, flavor) in enumerate(cases):
        if flavor == "uniform_noise":
            px = rng.integers(0, 1 << d, size=(h, w)).astype(np.uint8 if d == 8 else np.uint16)
            img = medtree.GrayImage(px, d)
        else:
            img = medtree.gen_image(flavor, w, h, d, seed=int(rng.integers(2**31)))
        out, _ = medtree.filter_image(
            img, n, rank=rank, percentile=pct, max_error=me, mode=mode, counting=False
        )
        inputs[f"in{i}"] = img.pixels
        outputs[f"out{i}"] = out.pixels
        meta.append(dict(idx=i, bit_depth=d, n=n, mode=mode, rank=rank,
                         percentile=pct, max_error=me, flavor=flavor))
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **inputs, **outputs)
    with open(os.path.join(HERE, "small_cases.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(f"small cases: {len(cases)}")


def digests():
    rec = {}

    def run(name, px, n, mode="uniform", bands=1):
        out, _ = medtree.filter_image(px, n, mode=mode, counting=False, bands=bands)
        rec[name] = dict(input=sha(px), output=sha(out.pixels), n=n, mode=mode,
                         first=[int(v) for v in out.pixels.ravel()[:8]])
        print(name, rec[name]["output"][:16])

    px1 = workloads.cfg1_uniform_u8()
    run("cfg1_512_r5", px1, 11)
    px2 = workloads.cfg2_blur_sp_u8(512, 512)
    for r in (1, 3, 7, 15, 31, 63):
        run(f"cfg2_512_r{r}", px2, 2 * r + 1, bands=8)
    px3 = workloads.cfg3_uniform_u16(192, 160)
    for r in (3, 7, 15, 31):
        run(f"cfg3_192x160_r{r}", px3, 2 * r + 1, bands=8)
    px4 = workloads.cfg4_three_gauss_u16(160, 192)
    for r in (15, 31):
        run(f"cfg4_160x192_r{r}_adaptive", px4, 2 * r + 1, mode="adaptive", bands=8)
    b5 = workloads.cfg5_batch_u8(4, 256, 256)
    for i in range(4):
        for r in (7, 25):
            run(f"cfg5_256_img{i}_r{r}", b5[i], 2 * r + 1, bands=4)
    with open(os.path.join(HERE, "digests.json"), "w") as fh:
        json.dump(rec, fh, indent=1, sort_keys=True)


def topologies():
    arrs = {}
    imgs = [
        ("two_mode8", medtree.gen_image("two_mode", 48, 40, 8, seed=5), 5),
        ("normal8", medtree.gen_image("normal_noise", 40, 48, 8, seed=6), 11),
        ("two_mode16", medtree.gen_image("two_mode", 32, 32, 16, seed=12), 5),
        ("cfg4_16", medtree.GrayImage(workloads.cfg4_three_gauss_u16(64, 64), 16), 31),
    ]
    for name, img, n in imgs:
        t = resolve_topology(img, n, "adaptive")
        arrs[f"{name}_px"] = img.pixels
        arrs[f"{name}_n"] = np.array(n)
        arrs[f"{name}_up"] = t.up
        arrs[f"{name}_leaf"] = t.leaf
        arrs[f"{name}_span"] = t.span
        arrs[f"{name}_lo"] = t.lo
    np.savez_compressed(os.path.join(HERE, "topologies.npz"), **arrs)


if __name__ == "__main__":
    small_cases()
    topologies()
    digests()
