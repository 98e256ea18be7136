"""Ad-hoc GPU probe: per-radius timing of each kernel family + sampled parity.

usage: python tools/probe.py [--cfg 2|3|5] [--radii 1,3,...] [--kernels vert,ctmf]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
import paper_1105_3829_b200 as mtb  # noqa: E402
from paper_1105_3829_b200 import _lib  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--radii", default="")
    ap.add_argument("--kernels", default="vert,ctmf")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--env", default="", help="extra env k=v;k=v applied per run")
    a = ap.parse_args()
    if a.cfg == 2:
        px = workloads.cfg2_blur_sp_u8()
    elif a.cfg == 1:
        px = workloads.cfg1_uniform_u8(4096, 4096)
    elif a.cfg == 3:
        px = workloads.cfg3_uniform_u16()
    elif a.cfg == 5:
        px = workloads.cfg5_batch_u8(1, 2048, 2048)[0]
    elif a.cfg == 4:
        px = workloads.cfg4_three_gauss_u16()
    radii = [int(x) for x in a.radii.split(",")] if a.radii else list(workloads.CONFIG_RADII[a.cfg])
    for kv in filter(None, a.env.split(";")):
        k, v = kv.split("=")
        os.environ[k] = v
    src = torch.from_numpy(px).cuda()
    out = torch.empty_like(src)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    H, W = px.shape
    res = {}
    for kern in a.kernels.split(","):
        os.environ["MTB_KERNEL"] = kern
        for r in radii:
            mtb.rank_filter(src, r, out=out)
            torch.cuda.synchronize()
            ts = []
            for _ in range(a.reps):
                flush.fill_(1)
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record()
                mtb.rank_filter(src, r, out=out)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = sorted(ts)[len(ts) // 2]
            got = out.cpu().numpy()
            ok = True
            for y0 in (0, H // 2 - 5, H - 12):
                ref = O.iot_rows(px, 2 * r + 1, y0, y0 + 12)
                ok &= bool(np.array_equal(got[y0:y0 + 12], ref))
            res[f"{kern}_r{r}"] = dict(ms=round(ms, 4), gpix_s=round(H * W / ms / 1e6, 2), ok=ok,
                                      kernel=_lib.last_kernel())
            print(kern, r, res[f"{kern}_r{r}"], flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
