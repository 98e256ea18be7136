"""Instruction counts per output pixel of every benchmarked launch (the
second ceiling of SURVEY 8(d): issue slots, next to the HBM roofline).

On the GPU box (one ncu pass over every case; the plain run first):

    python tools/ncu_issue.py run > gpurun_out/issue_plain.log 2>&1 &&
    ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum,sm__cycles_elapsed.avg,\
smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_ \
        --csv --log-file gpurun_out/issue.csv python tools/ncu_issue.py run

Here:

    python tools/ncu_issue.py parse gpurun_out/issue.csv gpurun_out/ncu_issue_manifest.json \
        > profiles/ncu_issue.json

``run`` warms each case with one call and measures the second; it writes
the number of library launches of each call to the manifest, so ``parse``
can assign the ncu rows (in launch order) to cases.  bench.py reads
profiles/ncu_issue.json: warp_inst / pixels per case, and the issue-bound
time at the measured SM clock.
"""

from __future__ import annotations

import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def cases():
    import workloads

    out = [("cfg1", 5, lambda: workloads.cfg1_uniform_u8())]
    out += [("cfg2", r, workloads.cfg2_blur_sp_u8) for r in workloads.CONFIG_RADII[2]]
    out += [("cfg3", r, workloads.cfg3_uniform_u16) for r in workloads.CONFIG_RADII[3]]
    out += [("cfg4", r, workloads.cfg4_three_gauss_u16) for r in workloads.CONFIG_RADII[4]]
    out += [("cfg5", r, workloads.cfg5_batch_u8) for r in workloads.CONFIG_RADII[5]]
    return out


def run():
    import torch

    import paper_1105_3829_b200 as mtb
    from paper_1105_3829_b200 import _lib

    torch.cuda.set_device(0)
    manifest = []
    frames = {}
    for key, r, gen in cases():
        if key not in frames:
            frames.clear()
            frames[key] = torch.from_numpy(gen()).cuda()
        src = frames[key]
        out = torch.empty_like(src)
        counts = []
        for _ in range(2):
            c0 = _lib.launch_count()
            mtb.rank_filter(src, r, out=out)
            torch.cuda.synchronize()
            counts.append(_lib.launch_count() - c0)
        manifest.append({"case": f"{key}_r{r}", "warm": counts[0], "measured": counts[1],
                         "pixels": int(src.numel()), "kernel": _lib.last_kernel()})
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "ncu_issue_manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
    print("ok", len(manifest))


def parse(csv_path, manifest_path):
    with open(manifest_path) as fh:
        manifest = json.load(fh)
    rows = {}
    order = []
    with open(csv_path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for rec in csv.DictReader(lines):
        kid = int(rec["ID"])
        if kid not in rows:
            rows[kid] = {"name": rec["Kernel Name"]}
            order.append(kid)
        val = rec["Metric Value"].replace(",", "")
        try:
            rows[kid][rec["Metric Name"]] = float(val)
        except ValueError:
            pass
    launches = [rows[k] for k in order]
    res = {"_note": ("ncu --metrics sm__inst_executed.sum (warp instructions), sm__cycles_elapsed.avg, "
                     "smsp__issue_active.avg.pct_of_peak_sustained_active, gpu__time_duration.sum per launch of "
                     "the measured call of each case (tools/ncu_issue.py); warp_inst sums every library launch "
                     "of the call (spread probe, gated launches, CTMF pre-pass included)")}
    i = 0
    for m in manifest:
        i += m["warm"]
        mine = launches[i:i + m["measured"]]
        i += m["measured"]
        inst = sum(x.get("sm__inst_executed.sum", 0.0) for x in mine)
        top = max(mine, key=lambda x: x.get("gpu__time_duration.sum", 0.0))
        res[m["case"]] = {
            "kernel": m["kernel"], "pixels": m["pixels"], "warp_inst": inst,
            "warp_inst_per_px": round(inst / m["pixels"], 3),
            "issue_active_pct": top.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "ncu_ns": sum(x.get("gpu__time_duration.sum", 0.0) for x in mine),
            "launches": [x["name"].split("(")[0] for x in mine],
        }
    if i != len(launches):
        res["_warning"] = f"{len(launches)} ncu rows, manifest accounts for {i}"
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    else:
        parse(sys.argv[2], sys.argv[3])
