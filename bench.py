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

``--impl reference``: the reference algorithm on the host cores (the C
restatement in oracle/, all threads, band-parallel like engine.py:243-262),
on a bounded band of the same frame; rank 0 only.
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


def cpu_baseline(px, budget_s: float = 12.0):
    """Reference algorithm (oracle C port) on all host cores, bounded sample:
    the first `rows` full-width rows of the frame at every radius."""
    from oracle import oracle as O

    O.build()
    threads = O.cpu_count()
    probe_rows = max(threads * 4, 32)
    t = sum(_cpu_rows(px, r, probe_rows, threads) for r in RADII)
    rows = int(min(H, max(probe_rows, probe_rows * budget_s / max(t, 1e-3))))
    rows = max(threads, rows - rows % threads)
    t = sum(_cpu_rows(px, r, rows, threads) for r in RADII)
    value = len(RADII) * rows * W / t / 1e6
    return {"value": round(value, 3), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"rows [0,{rows}) x {W} cols of the config-2 frame at r={list(RADII)}, "
                      f"oracle/medtree_oracle.c (IOT restatement), {threads} band threads"}


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    from oracle import oracle as O

    O.build()
    px = workloads.cfg2_blur_sp_u8(H, W)
    threads = O.cpu_count()
    rows = min(H, max(threads * 32, 64))
    for _ in range(max(args.warmup, 0)):
        for r in RADII:
            _cpu_rows(px, r, threads * 2, threads)
    times = []
    for _ in range(args.steps):
        times.append(sum(_cpu_rows(px, r, rows, threads) for r in RADII))
    t = sum(times) / len(times)
    value = len(RADII) * rows * W / t / 1e6
    cb = {"value": round(value, 3), "unit": UNIT, "cores": threads, "kind": "port",
          "sample": f"rows [0,{rows}) x {W} of the config-2 frame per radius, "
                    f"oracle C port, {threads} threads"}
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": "config2_4096x4096_u8_sweep_sample", "radii": list(RADII),
                   "rows_per_step": rows},
        "cpu_baseline": cb,
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------ GPU arm

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

    # correctness guard on a sample band (oracle is the checker, not measured)
    ref_rows = {}
    if rank == 0 and not args.no_check:
        from oracle import oracle as O

        for r in RADII:
            launch(r)
            got = out[:16].cpu().numpy()
            ref = ref_rows[r] = O.iot_rows(base, 2 * r + 1, 0, 16)
            if not np.array_equal(got, ref):
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
    if pg:
        t = torch.tensor([ms_step] + [ms_r[r] for r in RADII], device=red_dev, dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms_step = float(t[0])
        ms_r = {r: float(t[i + 1]) for i, r in enumerate(RADII)}
    px_step = len(RADII) * H * W * ws
    value = px_step / (ms_step * 1e-3) / 1e6

    # e2e: the C-ABI host-buffer entries on page-locked host frames; every
    # step copies each radius' input frame host->device and its result
    # device->host inside the timed region.  Headline: the six radii as one
    # frame sequence (mtb_filter_host_frames: frame i+1's copy in and frame
    # i-1's copy out overlap frame i's filtering); beside it the six
    # single-frame calls (mtb_filter_host, each synchronous).
    e2e = None
    if not args.no_e2e:
        hsrc = torch.empty((H, W), dtype=torch.uint8).pin_memory().numpy()
        hsrc[...] = base
        houts = [torch.empty((H, W), dtype=torch.uint8).pin_memory().numpy() for _ in RADII]

        def timed(step_fn):
            for _ in range(max(1, args.warmup // 2)):
                step_fn()
            torch.cuda.synchronize()
            if pg:
                pg.barrier()
            e2e_steps = max(1, min(args.steps, 5))
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                step_fn()
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / e2e_steps
            if pg:
                tt = torch.tensor([dt], device=red_dev, dtype=torch.float64)
                pg.all_reduce(tt, op=pg.ReduceOp.MAX)
                dt = float(tt[0])
            return round(len(RADII) * H * W * ws / dt / 1e6, 3)

        v_frames = timed(lambda: mtb.filter_host_frames([hsrc] * len(RADII), list(RADII), outs=houts))
        for o, r in zip(houts, RADII):
            if r in ref_rows and not np.array_equal(o[:16], ref_rows[r]):
                print(json.dumps({"error": f"e2e parity check failed at r={r}"}))
                return 1

        def single_calls():
            for r, o in zip(RADII, houts):
                mtb.filter_host_buffer(hsrc, r, out=o)

        v_single = timed(single_calls)
        e2e = {"value": v_frames, "unit": UNIT,
               "h2d_bytes_per_step": len(RADII) * H * W, "d2h_bytes_per_step": len(RADII) * H * W,
               "api": "paper_1105_3829_b200.filter_host_frames -> mtb_filter_host_frames (C ABI, six pinned "
                      "host frames per step, one per radius; copies of neighbouring frames overlapped with "
                      "filtering on a ring of 3 device buffer pairs)",
               "single_frame_calls": {"value": v_single, "api": "filter_host_buffer -> mtb_filter_host per "
                                      "radius (synchronous; row bands for r < 12, streaming launch for r >= 12)"}}

    if rank != 0:
        if pg:
            pg.destroy_process_group()
        return 0
    peak, peak_kind = _peaks()
    dom = max(RADII, key=lambda r: ms_r[r])
    alg_bytes = 2 * H * W  # 1 B read + 1 B write per output pixel
    achieved = alg_bytes / (ms_r[dom] * 1e-3) / 1e9
    traffic = _traffic_from_profiles().get(f"cfg2_r{dom}")
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (workloads.cfg2_blur_sp_u8, seed 1)",
        "config": {"workload": "config2_4096x4096_u8_radius_sweep", "radii": list(RADII),
                   "frame": [H, W], "l2": "flushed (256 MiB write) before every launch",
                   "parallelism": f"row slabs x{ws}, no collective"},
        "per_radius": {str(r): {"ms": round(ms_r[r], 4), "kernel": kernels[r],
                                "mpix_s": round(H * W / (ms_r[r] * 1e-3) / 1e6, 1),
                                "hbm_frac": round(alg_bytes / (ms_r[r] * 1e-3) / 1e9 / peak, 5)}
                       for r in RADII},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 5), "traffic": traffic,
                     "kernel": f"{kernels[dom]} r={dom}",
                     "algorithmic_bytes_per_launch": alg_bytes, "peak_kind": peak_kind},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if e2e:
        line["e2e"] = e2e
    if ws == 1 and not args.no_extra:
        line["other_configs"] = other_configs(mtb, torch, flush)
    if ws == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(base, args.cpu_budget)
    print(json.dumps(line))
    if pg:
        pg.destroy_process_group()
    return 0


def other_configs(mtb, torch, flush, reps: int = 2):
    """The other BASELINE configs, device-resident, L2 flushed, event-timed
    (informational: the headline `value` is config 2).  Mpix/s per radius and
    HBM-roofline fraction (2 B/px for u8, 4 B/px for u16)."""
    from paper_1105_3829_b200 import _lib

    peak, _ = _peaks()
    res = {}

    def timed(src, r, out, **kw):
        mtb.rank_filter(src, r, out=out, **kw)
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            mtb.rank_filter(src, r, out=out, **kw)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return min(ts)

    specs = [
        ("config1_512x512_u8", lambda: workloads.cfg1_uniform_u8(), workloads.CONFIG_RADII[1], 2),
        ("config3_4096x4096_u16", lambda: workloads.cfg3_uniform_u16(), workloads.CONFIG_RADII[3], 4),
        ("config4_8192x8192_u16_adaptive", lambda: workloads.cfg4_three_gauss_u16(),
         workloads.CONFIG_RADII[4], 4),
        ("config5_64x2048x2048_u8_batch", lambda: workloads.cfg5_batch_u8(), workloads.CONFIG_RADII[5], 2),
    ]
    for name, gen, radii, bpp in specs:
        px = gen()
        src = torch.from_numpy(px).cuda()
        out = torch.empty_like(src)
        npx = px.size
        entry = {}
        for r in radii:
            ms = timed(src, r, out, adaptive=("adaptive" in name))
            entry[str(r)] = {"ms": round(ms, 4), "mpix_s": round(npx / (ms * 1e-3) / 1e6, 1),
                             "hbm_frac": round(bpp * npx / (ms * 1e-3) / 1e9 / peak, 5),
                             "kernel": _lib.last_kernel()}
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
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
