"""Parity of a forced kernel family against the CPU oracle on small ragged frames.
usage: python tools/check_family.py [kernel] [radii]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1105_3829_b200 as mtb  # noqa: E402
from paper_1105_3829_b200 import _lib  # noqa: E402
from oracle import oracle as O  # noqa: E402

kern = sys.argv[1] if len(sys.argv) > 1 else "bandmma"
radii = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4, 7, 8, 9, 15, 24, 25, 31, 40, 41, 63, 72, 73, 100, 127]
os.environ["MTB_KERNEL"] = kern
rng = np.random.default_rng(5)
bad = 0
for (H, W) in ((97, 333), (40, 1500), (300, 64)):
    noise = rng.integers(0, 256, (H, W), dtype=np.uint8)
    smooth = (np.add.outer(np.arange(H), np.arange(W)) // 3 % 256).astype(np.uint8)
    smooth[rng.random((H, W)) < 0.05] = 255
    for name, px in (("noise", noise), ("ramp", smooth)):
        src = torch.from_numpy(px).cuda()
        for r in radii:
            n = 2 * r + 1
            if n > 2 * min(H, W) + 1:
                continue
            for rank in (None, 1, n * n, max(1, n * n // 3)):
                out = mtb.rank_filter(src, r, rank=rank) if rank else mtb.rank_filter(src, r)
                torch.cuda.synchronize()
                ref = O.iot_filter(px, n, rank=rank) if rank else O.iot_filter(px, n)
                got = out.cpu().numpy()
                if not np.array_equal(got, ref):
                    bad += 1
                    d = np.argwhere(got != ref)
                    print(f"MISMATCH {name} {H}x{W} r={r} rank={rank}: {len(d)} px, first {d[0]} got {got[tuple(d[0])]} ref {ref[tuple(d[0])]} kernel {_lib.last_kernel()}")
        print(name, H, W, "done; kernel", _lib.last_kernel(), flush=True)
print("bad =", bad)
sys.exit(1 if bad else 0)
