"""Full-size SHA-256 digests of the REFERENCE's own outputs for BASELINE
configs 2-5 (the exactness bar of pkg/tests/test_acceptance.py:46-93,
applied at the sizes the configs name).

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_fullsize_digests.py [--jobs 8]

Each frame is cut into row bands with n//2 halo rows, exactly the
reference's own band scheme (pkg/src/medtree/engine.py:243-262): band
[a, b) is the rows [a-top, b-top) of ``filter_image`` run on source rows
[top, bottom) = [max(0, a-h2), min(H, b+h2)), so clamping only ever happens
at the global edges and the stitched frame is byte-identical to one
engine over the whole frame.  The bands run in a fork-based process pool
(the numba kernels hold the GIL).  Config 4 is adaptive: its topology is
resolved ONCE on the full frame (engine.py:186-206) and passed to every
band, as ``filter_image(..., bands=k)`` does.

Writes ``fullsize_digests.json``: per config and radius the input and
output SHA-256 (config 5: one digest per image plus the digest of the
stacked batch).  The GPU tests regenerate the inputs from ``workloads.py``
(checking the input digest first) and hash the full GPU frames against
these.  Nothing at GPU-test time reads /root/reference.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import workloads  # noqa: E402

_FRAMES: dict = {}
_TOPO: dict = {}


# beyond BASELINE's sweep: the radii of the tcgen05 kernel (k_bandtc_u8, r >= 76) on the config-2 frame
EXTRA_RADII_CFG2 = (80, 127)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _band(task):
    """One band of one frame through the reference's public filter_image."""
    import medtree

    key, n, a, b, mode = task
    px = _FRAMES[key]
    H = px.shape[0]
    h2 = n // 2
    top, bottom = max(0, a - h2), min(H, b + h2)
    topo = _TOPO.get((key, n))
    out, _ = medtree.filter_image(px[top:bottom], n, mode=mode, topology=topo, counting=False)
    return task, out.pixels[a - top:b - top].copy()


def _edges(H, k):
    e = np.linspace(0, H, k + 1, dtype=int)
    return [(int(a), int(b)) for a, b in zip(e[:-1], e[1:]) if a != b]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=os.cpu_count())
    ap.add_argument("--only", default="", help="comma list of cfg2,cfg3,cfg4,cfg5")
    args = ap.parse_args()
    only = set(filter(None, args.only.split(",")))
    path = os.path.join(HERE, "fullsize_digests.json")
    rec = {}
    if os.path.exists(path):
        with open(path) as fh:
            rec = json.load(fh)

    import medtree
    from medtree.engine import resolve_topology

    jobs = []  # (name, key, n, mode, bands)
    if not only or "cfg2" in only:
        _FRAMES["cfg2"] = workloads.cfg2_blur_sp_u8()
        for r in workloads.CONFIG_RADII[2] + EXTRA_RADII_CFG2:
            jobs.append((f"cfg2_4096_r{r}", "cfg2", 2 * r + 1, "uniform", 32))
    if not only or "cfg3" in only:
        _FRAMES["cfg3"] = workloads.cfg3_uniform_u16()
        for r in workloads.CONFIG_RADII[3]:
            jobs.append((f"cfg3_4096_r{r}", "cfg3", 2 * r + 1, "uniform", 32))
    if not only or "cfg4" in only:
        _FRAMES["cfg4"] = workloads.cfg4_three_gauss_u16()
        for r in workloads.CONFIG_RADII[4]:
            n = 2 * r + 1
            t0 = time.time()
            _TOPO[("cfg4", n)] = resolve_topology(medtree.GrayImage(_FRAMES["cfg4"], 16), n, "adaptive")
            print(f"cfg4 topology n={n}: {time.time() - t0:.1f}s", flush=True)
            jobs.append((f"cfg4_8192_r{r}_adaptive", "cfg4", n, "adaptive", 32))
    if not only or "cfg5" in only:
        batch = workloads.cfg5_batch_u8()
        for i in range(batch.shape[0]):
            _FRAMES[f"cfg5_{i}"] = batch[i]
        for r in workloads.CONFIG_RADII[5]:
            for i in range(batch.shape[0]):
                jobs.append((f"cfg5_2048_img{i}_r{r}", f"cfg5_{i}", 2 * r + 1, "uniform", 1))

    tasks, owner = [], {}
    outs = {}
    for name, key, n, mode, k in jobs:
        H = _FRAMES[key].shape[0]
        outs[name] = np.empty_like(_FRAMES[key])
        for a, b in _edges(H, k):
            t = (key, n, a, b, mode)
            tasks.append(t)
            owner[t] = name
    t0 = time.time()
    ctx = mp.get_context("fork")
    with ctx.Pool(args.jobs) as pool:
        done = 0
        for task, band in pool.imap_unordered(_band, tasks):
            _, _, a, b, _ = task
            outs[owner[task]][a:b] = band
            done += 1
            if done % 32 == 0:
                print(f"{done}/{len(tasks)} bands, {time.time() - t0:.0f}s", flush=True)
    for name, key, n, mode, _ in jobs:
        rec[name] = dict(input=sha(_FRAMES[key]), output=sha(outs[name]), n=n, mode=mode,
                         shape=list(_FRAMES[key].shape), dtype=str(_FRAMES[key].dtype),
                         first=[int(v) for v in outs[name].ravel()[:8]])
        print(name, rec[name]["output"][:16], flush=True)
    for r in workloads.CONFIG_RADII[5]:
        names = [f"cfg5_2048_img{i}_r{r}" for i in range(64)]
        if all(nm in outs for nm in names):
            stack = np.stack([outs[nm] for nm in names])
            inp = np.stack([_FRAMES[f"cfg5_{i}"] for i in range(64)])
            rec[f"cfg5_batch_r{r}"] = dict(input=sha(inp), output=sha(stack),
                                          n=2 * r + 1, mode="uniform", shape=list(stack.shape),
                                          dtype="uint8")
    rec["_generator"] = ("tests/golden/make_fullsize_digests.py: reference medtree.filter_image "
                         "(counting=False) in row bands with n//2 halos (engine.py:243-262)")
    with open(path, "w") as fh:
        json.dump(rec, fh, indent=1, sort_keys=True)
    print(f"done in {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
