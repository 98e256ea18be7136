#!/usr/bin/env python
"""Benchmark: output Mpixel/s of the 2D running median (BASELINE.json metric).

Workload (N=1): BASELINE config 2 -- a 4096x4096 uint8 frame (Gaussian-
blurred noise + 5% salt-and-pepper, workloads.cfg2_blur_sp_u8) filtered at
every radius of the sweep r in {1,3,7,15,31,63}.  One step = the frame at
all six radii.  ``value`` = output pixels of all radii / device time of the
step, inputs resident in HBM, L2 flushed (256 MiB write) before every
launch.  ``per_radius`` gives the curve the metric is quoted as.

N>1 (torchrun, one rank per GPU): weak scaling -- rank k filters rows
[k*4096, (k+1)*4096) of a frame made of N stacked copies, with its radius
halo rows taken from the host copy; no collective on the data path (NCCL
only for the barrier and the max-over-ranks of the timings).

Configs 4 and 5 (``sharded_configs``, every N): config 4 row-sharded and
config 5 image-sharded over the ranks with the product's own planners
(plan_slabs / plan_images), strong scaling.

``--impl reference``: the reference algorithm on the host cores (the C
restatement in oracle/, all threads, band-parallel like engine.py:243-262)
over the same sample as the GPU arm's ``cpu_baseline`` (the whole frame
when a sweep fits the budget), plus the unmodified numba reference from
baseline/_ref on that sample; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

RADII = workloads.CONFIG_RADII[2]
H = W = 4096
METRIC = "output Mpixel/s vs radius (8-bit, config 2 sweep r=1..63)"
UNIT = "Mpixel/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML
    in-process every ~2 ms (a timed region of a few tens of ms still gets
    many samples under load), else nvidia-smi -lms 50."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        cvd = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [x.strip() for x in cvd.split(",") if x.strip()]
        self.index = int(ids[index]) if index < len(ids) and ids[index].isdigit() else index
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()
        self.lines: list[str] = []

    def _nvml_loop(self):
        p, h = self.nvml
        bits = [("hw_slowdown", getattr(p, "nvmlClocksEventReasonHwSlowdown", 0x8)),
                ("hw_thermal_slowdown", getattr(p, "nvmlClocksEventReasonHwThermalSlowdown", 0x40)),
                ("sw_thermal_slowdown", getattr(p, "nvmlClocksEventReasonSwThermalSlowdown", 0x20)),
                ("sw_power_cap", getattr(p, "nvmlClocksEventReasonSwPowerCap", 0x4))]
        mx = p.nvmlDeviceGetMaxClockInfo(h, p.NVML_CLOCK_SM)
        while not self.stop.is_set():
            try:
                sm = p.nvmlDeviceGetClockInfo(h, p.NVML_CLOCK_SM)
                rs = p.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                break
            flags = ["Active" if rs & b else "Not Active" for _, b in bits]
            self.lines.append(", ".join([str(sm), str(mx), hex(rs)] + flags))
            time.sleep(0.002)

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index))
            self._t = threading.Thread(target=self._nvml_loop, daemon=True)
            self._t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.nvml is not None:
            self.stop.set()
            self._t.join(timeout=2)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self._t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def _traffic_from_profiles():
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except Exception:
        return {}


# ------------------------------------------------------------ CPU legs

def _cpu_rows(px, r, rows, threads):
    from oracle import oracle as O

    n = 2 * r + 1
    t0 = time.perf_counter()
    O.iot_rows(px, n, 0, rows, threads=threads, bands=threads)
    return time.perf_counter() - t0


def _port_rows(px, threads, budget_s):
    """Rows of the sweep sample: the whole frame when one sweep over it fits
    the budget, else the largest band that does (every thread still gets
    >= 2*63 rows so halo re-reads stay below 2x)."""
    probe = max(threads * 64, 256)
    t = sum(_cpu_rows(px, r, probe, threads) for r in RADII)
    rows = int(min(H, probe * budget_s / max(t, 1e-3)))
    rows = max(min(H, threads * 4 * max(RADII)), rows)
    return rows - rows % threads if rows < H else H


def port_sweep(px, threads, rows):
    """One config-2 sweep (all radii) over rows [0, rows) with the C port."""
    return sum(_cpu_rows(px, r, rows, threads) for r in RADII)


def _numba_band(task):
    import medtree  # the reference package (baseline/_ref)

    r, a, b = task
    px = _NUMBA_FRAME
    h2 = r
    top, bot = max(0, a - h2), min(px.shape[0], b + h2)
    medtree.filter_image(px[top:bot], 2 * r + 1, counting=False)
    return b - a


_NUMBA_FRAME = None


def numba_reference(px, rows, procs):
    """The UNMODIFIED reference (medtree.filter_image, numba, installed in
    baseline/_ref) on the same sample as the port: rows [0, rows) of the
    config-2 frame at every radius, one band per process (fork pool; the
    numba kernels hold the GIL), bands with n//2 halos exactly as
    engine.py:243-262.  Returns None when the reference is not installed."""
    global _NUMBA_FRAME
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "medtree")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/mtb_numba_cache")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import multiprocessing as mp

    import medtree

    medtree.filter_image(px[:64, :64], 3, counting=False)  # JIT once, before the fork
    _NUMBA_FRAME = px
    edges = np.linspace(0, rows, procs + 1, dtype=int)
    tasks = [(r, int(a), int(b)) for r in RADII for a, b in zip(edges[:-1], edges[1:]) if a < b]
    with mp.get_context("fork").Pool(procs) as pool:
        pool.map(_numba_band, [(1, 0, 8)] * procs)  # warm every worker
        t0 = time.perf_counter()
        done = sum(pool.map(_numba_band, tasks, chunksize=1))
        t = time.perf_counter() - t0
    return {"value": round(done * W / t / 1e6, 3), "unit": UNIT, "cores": procs, "kind": "reference",
            "sample": f"rows [0,{rows}) x {W} of the config-2 frame at r={list(RADII)}: unmodified reference "
                      f"medtree.filter_image(counting=False) from baseline/_ref (numba), {procs} processes, "
                      f"one band each with n//2 halo rows (engine.py:243-262)"}


def cpu_baseline(px, budget_s: float = 4.0):
    """Reference algorithm (oracle C port) on all host cores over the same
    sample as the reference arm, plus the unmodified numba reference on that
    sample beside it."""
    from oracle import oracle as O

    O.build()
    threads = O.cpu_count()
    rows = _port_rows(px, threads, budget_s)
    t = port_sweep(px, threads, rows)
    value = len(RADII) * rows * W / t / 1e6
    out = {"value": round(value, 3), "unit": UNIT, "cores": threads, "kind": "port",
           "sample": f"rows [0,{rows}) x {W} of the config-2 frame at r={list(RADII)} (one sweep), "
                     f"oracle/medtree_oracle.c (IOT restatement), {threads} band threads"}
    try:
        nb = numba_reference(px, rows, threads)
    except Exception as e:  # reported, never fatal
        nb = {"unavailable": f"{type(e).__name__}: {e}"}
    if nb is not None:
        out["numba_reference"] = nb
    return out


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    from oracle import oracle as O

    O.build()
    px = workloads.cfg2_blur_sp_u8(H, W)
    threads = O.cpu_count()
    rows = _port_rows(px, threads, args.cpu_budget)
    for _ in range(max(args.warmup, 0)):
        for r in RADII:
            _cpu_rows(px, r, threads * 8, threads)
    times = [port_sweep(px, threads, rows) for _ in range(args.steps)]
    t = statistics.median(times)
    value = len(RADII) * rows * W / t / 1e6
    cb = {"value": round(value, 3), "unit": UNIT, "cores": threads, "kind": "port",
          "sample": f"rows [0,{rows}) x {W} of the config-2 frame per radius (the same sample as the GPU "
                    f"arm's cpu_baseline), oracle C port, {threads} threads, median of {args.steps} sweeps"}
    try:
        nb = numba_reference(px, rows, threads)
    except Exception as e:
        nb = {"unavailable": f"{type(e).__name__}: {e}"}
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3 * H / rows, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic (workloads.cfg2_blur_sp_u8, seed 1)",
        "config": {"workload": "config2_4096x4096_u8_radius_sweep", "radii": list(RADII),
                   "frame": [H, W], "rows_per_step": rows, "same_config": rows == H},
        "cpu_baseline": cb,
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if nb is not None:
        line["reference_numba"] = nb
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------ GPU arm

ISSUE_RATE_PER_SM_CLK = 4  # warp-instructions issued per SM per clock (4 schedulers)


def _issue_profile():
    """ncu-derived per-kernel instruction counts (profiles/ncu_issue.json,
    written by tools/ncu_issue.py from `ncu --metrics` captures of each
    radius' launch)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_issue.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


IMMA_PER_SM_CLK = 1.79  # measured: tools/micro/imma_lat.cu, profiles/r2_micro_imma.txt


def _tensor_share(r, npx, ms, sm_mhz, nsm):
    """Tensor-core work of one k_bandmma_u8 launch: one product of 4 n-tiles x
    NK k-tiles (mma.sync m16n8k32 u8, 8192 MACs x 2 ops) per 16 output pixels,
    against the measured IMMA issue rate."""
    nk = (16 + 2 * r + 31) // 32
    imma = npx / 16 * 4 * nk
    bound_ms = imma / (nsm * IMMA_PER_SM_CLK * (sm_mhz or 1965.0) * 1e6) * 1e3
    return {"imma_per_launch": int(imma), "int8_tops": round(imma * 16 * 8 * 32 * 2 / (ms * 1e-3) / 1e12, 1),
            "imma_bound_ms": round(bound_ms, 4), "frac": round(bound_ms / ms, 4)}


def _issue_ceiling(key, npx, ms, sm_mhz, nsm):
    """The second ceiling: the kernel's warp-instructions per
    output pixel (ncu) against the chip's issue rate.  issue_bound_ms = the
    time the launch would take at one warp-instruction per scheduler per
    clock; frac = issue_bound_ms / measured ms."""
    rec = _issue_profile().get(key)
    if not rec or not sm_mhz:
        return None
    wipp = rec["warp_inst"] / rec["pixels"]
    bound_ms = npx * wipp / (nsm * ISSUE_RATE_PER_SM_CLK * sm_mhz * 1e6) * 1e3
    return {"warp_inst_per_px": round(wipp, 2), "issue_bound_ms": round(bound_ms, 4),
            "frac": round(bound_ms / ms, 4), "ncu_issue_active": rec.get("issue_active_pct"),
            "kernel": rec.get("kernel")}


def _events(torch, fn, flush, reps):
    """Median event time (ms) of `fn` over `reps` launches, L2 flushed
    before each (the flush is outside the events)."""
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    return statistics.median([a.elapsed_time(b) for a, b in ts])


def run_ours(args):
    import torch

    import paper_1105_3829_b200 as mtb
    from paper_1105_3829_b200 import _lib

    ws, rank, local = _dist()
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    backend = os.environ.get("MTB_BENCH_BACKEND", "nccl")  # gloo: CPU-side smoke of the N>1 logic
    red_dev = dev if backend == "nccl" else torch.device("cpu")
    if ws > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        pg = dist

    def max_over_ranks(vals):
        if not pg:
            return vals
        t = torch.tensor(vals, device=red_dev, dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        return [float(v) for v in t]

    base = workloads.cfg2_blur_sp_u8(H, W)
    # weak scaling: rank k owns rows [k*H, (k+1)*H) of N stacked copies
    Hg = H * ws
    a, b = rank * H, (rank + 1) * H
    rmax = max(RADII)
    top, bot = max(0, a - rmax), min(Hg, b + rmax)
    slab_host = base[np.arange(top, bot) % H]
    src = torch.from_numpy(np.ascontiguousarray(slab_host)).to(dev)
    out = torch.empty((H, W), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def launch(r):
        mtb.rank_filter(src, r, out=out, rows=(a, b), src_row0=top, height=Hg)

    # correctness guard: the whole frame of every radius against the
    # reference's own full-frame digests (the oracle is not run here)
    if ws == 1 and not args.no_check:
        from tests import golden_data as G

        for r in RADII:
            launch(r)
            if G.sha(out.cpu().numpy()) != G.fullsize_digests()[f"cfg2_4096_r{r}"]["output"]:
                print(json.dumps({"error": f"parity check failed at r={r}"}))
                return 1

    for _ in range(args.warmup):
        for r in RADII:
            launch(r)
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    kernels = {}
    for r in RADII:
        launch(r)
        kernels[r] = _lib.last_kernel()
    torch.cuda.synchronize()
    evs = {r: [] for r in RADII}
    launches0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if pg:
            pg.barrier()
        for _ in range(args.steps):
            for r in RADII:
                flush.fill_(1)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                launch(r)
                e1.record()
                evs[r].append((e0, e1))
        torch.cuda.synchronize()
        if pg:
            pg.barrier()
    launches = _lib.launch_count() - launches0
    ms_r = {r: sum(e0.elapsed_time(e1) for e0, e1 in evs[r]) / args.steps for r in RADII}
    ms_step = sum(ms_r.values())
    red = max_over_ranks([ms_step] + [ms_r[r] for r in RADII])
    ms_step, ms_r = red[0], {r: red[i + 1] for i, r in enumerate(RADII)}
    px_step = len(RADII) * H * W * ws
    value = px_step / (ms_step * 1e-3) / 1e6
    clocks = clk.summary()
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count

    # e2e: the C-ABI host-buffer entries on page-locked host frames; every
    # step copies each radius' input frame host->device and its result
    # device->host inside the timed region.  Headline: the six radii as one
    # frame sequence (mtb_filter_host_frames: frame i+1's copy in and frame
    # i-1's copy out overlap frame i's filtering); beside it the six
    # single-frame calls (mtb_filter_host, each synchronous) on pinned
    # frames, and the drop-in filter_image on the caller's pageable numpy
    # frame (what a reference caller passes).
    e2e = None
    if not args.no_e2e:
        hsrc = torch.empty((H, W), dtype=torch.uint8).pin_memory().numpy()
        hsrc[...] = base
        houts = [torch.empty((H, W), dtype=torch.uint8).pin_memory().numpy() for _ in RADII]

        def timed(step_fn, steps=None):
            for _ in range(max(1, args.warmup // 2)):
                step_fn()
            torch.cuda.synchronize()
            if pg:
                pg.barrier()
            e2e_steps = steps or max(1, min(args.steps, 5))
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                step_fn()
            torch.cuda.synchronize()
            dt = max_over_ranks([(time.perf_counter() - t0) / e2e_steps])[0]
            return round(len(RADII) * H * W * ws / dt / 1e6, 3)

        v_frames = timed(lambda: mtb.filter_host_frames([hsrc] * len(RADII), list(RADII), outs=houts))
        if ws == 1 and not args.no_check:
            from tests import golden_data as G

            for o, r in zip(houts, RADII):
                if G.sha(o) != G.fullsize_digests()[f"cfg2_4096_r{r}"]["output"]:
                    print(json.dumps({"error": f"e2e parity check failed at r={r}"}))
                    return 1

        def single_calls():
            for r, o in zip(RADII, houts):
                mtb.filter_host_buffer(hsrc, r, out=o)

        v_single = timed(single_calls)
        page_src = np.ascontiguousarray(base)

        def dropin_calls():
            for r in RADII:
                mtb.filter_image(page_src, 2 * r + 1)

        v_page = timed(dropin_calls, steps=2)
        e2e = {"value": v_frames, "unit": UNIT,
               "h2d_bytes_per_step": len(RADII) * H * W, "d2h_bytes_per_step": len(RADII) * H * W,
               "api": "paper_1105_3829_b200.filter_host_frames -> mtb_filter_host_frames (C ABI, six pinned "
                      "host frames per step, one per radius; copies of neighbouring frames overlapped with "
                      "filtering, one device buffer pair per frame)",
               "single_frame_calls": {"value": v_single, "api": "filter_host_buffer -> mtb_filter_host_rows per "
                                      "radius on pinned frames (synchronous; row bands for r < 12, streaming "
                                      "launch for r >= 12)"},
               "dropin_pageable": {"value": v_page, "api": "filter_image(numpy frame, n) per radius: the "
                                   "reference's call on a pageable array (row bands, driver-staged copies)"}}

    sharded = None if args.no_extra else sharded_configs(mtb, torch, flush, ws, rank, max_over_ranks, args)

    if rank != 0:
        if pg:
            pg.destroy_process_group()
        return 0
    peak, peak_kind = _peaks()
    dom = max(RADII, key=lambda r: ms_r[r])
    alg_bytes = 2 * H * W  # 1 B read + 1 B write per output pixel
    achieved = alg_bytes / (ms_r[dom] * 1e-3) / 1e9
    traffic = _traffic_from_profiles().get(f"cfg2_r{dom}")
    per_radius = {}
    for r in RADII:
        per_radius[str(r)] = {"ms": round(ms_r[r], 4), "kernel": kernels[r],
                              "mpix_s": round(H * W / (ms_r[r] * 1e-3) / 1e6, 1),
                              "hbm_frac": round(alg_bytes / (ms_r[r] * 1e-3) / 1e9 / peak, 5),
                              "issue": _issue_ceiling(f"cfg2_r{r}", H * W, ms_r[r], clocks.get("sm_mhz"), nsm)}
    for r in RADII:  # the tensor-core share of the band-matrix kernel (k_bandmma_u8)
        if kernels[r].startswith("k_bandmma"):
            per_radius[str(r)]["tensor"] = _tensor_share(r, H * W, ms_r[r], clocks.get("sm_mhz"), nsm)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (workloads.cfg2_blur_sp_u8, seed 1)",
        "config": {"workload": "config2_4096x4096_u8_radius_sweep", "radii": list(RADII),
                   "frame": [H, W], "l2": "flushed (256 MiB write) before every launch",
                   "parallelism": f"row slabs x{ws}, no collective"},
        "per_radius": per_radius,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 5), "traffic": traffic,
                     "kernel": f"{kernels[dom]} r={dom}",
                     "algorithmic_bytes_per_launch": alg_bytes, "peak_kind": peak_kind,
                     "issue": per_radius[str(dom)]["issue"]},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if e2e:
        line["e2e"] = e2e
    if sharded:
        line["sharded_configs"] = sharded
    if ws == 1 and not args.no_extra:
        line["other_configs"] = other_configs(mtb, torch, flush, clocks.get("sm_mhz"), nsm)
    if ws == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(base, args.cpu_budget)
    print(json.dumps(line))
    if pg:
        pg.destroy_process_group()
    return 0


def sharded_configs(mtb, torch, flush, ws, rank, max_over_ranks, args, reps: int = 20):
    """Configs 4 and 5 split over the N ranks exactly as the product splits
    them (plan_slabs / plan_images): config 4 row-sharded (rank k filters
    slab k of the 8192^2 frame, halo rows from the host copy), config 5
    image-sharded (rank k filters its run of the 64 images).  Strong
    scaling: the total work is fixed.  Device time per radius = median of
    `reps` event-timed launches (L2 flushed), max over ranks; e2e = the host
    entries (mtb_filter_host_rows / mtb_filter_host_frames) on pinned host
    buffers, wall clock, max over ranks."""
    res = {}
    dev = torch.cuda.current_device()
    # config 4
    px4 = workloads.cfg4_three_gauss_u16()
    H4, W4 = px4.shape
    sl = mtb.plan_slabs(H4, ws, max(workloads.CONFIG_RADII[4]))[rank]
    pin4 = torch.from_numpy(px4).pin_memory()
    src4 = pin4[sl.top:sl.bot].to(dev)
    out4 = torch.empty((sl.b - sl.a, W4), dtype=torch.uint16, device=dev)
    hout4 = torch.empty((sl.b - sl.a, W4), dtype=torch.uint16).pin_memory().numpy()
    entry = {}
    for r in workloads.CONFIG_RADII[4]:
        s = mtb.plan_slabs(H4, ws, r)[rank]
        s4 = src4[s.top - sl.top:s.bot - sl.top]
        fn = lambda: mtb.rank_filter(s4, r, out=out4, rows=(s.a, s.b), src_row0=s.top, height=H4)  # noqa: E731
        fn()
        ms = max_over_ranks([_events(torch, fn, flush, reps)])[0]
        lib = mtb._lib.load()
        pin_np = pin4.numpy()

        def host_rows():
            n = 2 * r + 1
            mtb._lib.check(lib.mtb_filter_host_rows(pin_np.ctypes.data, hout4.ctypes.data, 16, H4, W4, s.a, s.b,
                                                    r, (n * n + 1) // 2, None, 0, dev))
        host_rows()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            host_rows()
        e2e_s = max_over_ranks([(time.perf_counter() - t0) / 3])[0]
        entry[str(r)] = {"ms": round(ms, 4), "mpix_s": round(H4 * W4 / (ms * 1e-3) / 1e6, 1),
                         "e2e_mpix_s": round(H4 * W4 / e2e_s / 1e6, 1), "kernel": mtb._lib.last_kernel(),
                         "rows_per_rank": s.b - s.a}
    res["config4_8192x8192_u16_adaptive_row_sharded"] = entry
    del src4, out4, pin4
    # config 5
    b5 = workloads.cfg5_batch_u8()
    B = b5.shape[0]
    i0, i1 = mtb.plan_images(B, ws)[rank]
    entry = {}
    if i1 > i0:
        pin5 = torch.from_numpy(b5[i0:i1]).pin_memory()
        src5 = pin5.to(dev)
        out5 = torch.empty_like(src5)
        hout5 = [torch.empty(b5.shape[1:], dtype=torch.uint8).pin_memory().numpy() for _ in range(i1 - i0)]
        frames = [pin5[i].numpy() for i in range(i1 - i0)]
    for r in workloads.CONFIG_RADII[5]:
        if i1 > i0:
            fn = lambda: mtb.rank_filter(src5, r, out=out5)  # noqa: E731
            fn()
            ms_l = _events(torch, fn, flush, max(3, reps // 4))
            mtb.filter_host_frames(frames, r, outs=hout5)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            mtb.filter_host_frames(frames, r, outs=hout5)
            e2e_l = time.perf_counter() - t0
        else:
            ms_l, e2e_l = 0.0, 0.0
        ms, e2e_s = max_over_ranks([ms_l, e2e_l])
        npx = b5.size
        entry[str(r)] = {"ms": round(ms, 4), "mpix_s": round(npx / (ms * 1e-3) / 1e6, 1),
                         "e2e_mpix_s": round(npx / e2e_s / 1e6, 1), "kernel": mtb._lib.last_kernel(),
                         "images_per_rank": i1 - i0}
    res["config5_64x2048x2048_u8_batch_image_sharded"] = entry
    res["_note"] = ("strong scaling (fixed total work) over the ranks; device ms = median of event-timed "
                    "launches with L2 flushed, max over ranks; e2e through the host entries on pinned buffers")
    return res


def other_configs(mtb, torch, flush, sm_mhz, nsm, reps: int = 20):
    """Configs 1 and 3, device-resident, L2 flushed, median of `reps`
    event-timed launches (informational: the headline `value` is config 2).
    Mpix/s per radius, HBM-roofline fraction (2 B/px for u8, 4 B/px for
    u16) and the issue ceiling."""
    from paper_1105_3829_b200 import _lib

    peak, _ = _peaks()
    res = {}
    specs = [
        ("config1_512x512_u8", "cfg1", lambda: workloads.cfg1_uniform_u8(), workloads.CONFIG_RADII[1], 2),
        ("config3_4096x4096_u16", "cfg3", lambda: workloads.cfg3_uniform_u16(), workloads.CONFIG_RADII[3], 4),
    ]
    for name, key, gen, radii, bpp in specs:
        px = gen()
        src = torch.from_numpy(px).cuda()
        out = torch.empty_like(src)
        npx = px.size
        entry = {}
        for r in radii:
            fn = lambda: mtb.rank_filter(src, r, out=out)  # noqa: E731
            fn()
            ms = _events(torch, fn, flush, reps)
            entry[str(r)] = {"ms": round(ms, 4), "mpix_s": round(npx / (ms * 1e-3) / 1e6, 1),
                             "hbm_frac": round(bpp * npx / (ms * 1e-3) / 1e9 / peak, 5),
                             "kernel": _lib.last_kernel(),
                             "issue": _issue_ceiling(f"{key}_r{r}", npx, ms, sm_mhz, nsm)}
        res[name] = entry
        del src, out
        torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip configs 1,3,4,5")
    ap.add_argument("--cpu-budget", type=float, default=8.0, help="seconds per port sweep (sample size)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
