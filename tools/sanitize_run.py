"""Small run exercising every kernel family (for compute-sanitizer)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1105_3829_b200 as mtb  # noqa: E402
from oracle import oracle as O  # noqa: E402

rng = np.random.default_rng(3)
px8 = rng.integers(0, 256, (90, 300), dtype=np.uint8)
px16 = rng.integers(0, 65536, (70, 90)).astype(np.uint16)
bad = 0
# 3x3 kernels (TMA-staged for W % 16 == 0) and the merge networks at tile-edge widths
for W in (16, 1040, 1043):
    for bits, dt in ((8, np.uint8), (16, np.uint16)):
        im = rng.integers(0, 1 << bits, (37, W)).astype(dt)
        for r in (1, 2, 3):
            out = mtb.rank_filter(torch.from_numpy(im).cuda(), r).cpu().numpy()
            bad += int(not np.array_equal(out, O.iot_filter(im, 2 * r + 1)))
# CTMF with up-front snapshots in both register budgets
for ctb in ("1", "1000"):
    os.environ["MTB_CT_CTB4_R"] = ctb
    os.environ["MTB_KERNEL"] = "ctmf"
    out = mtb.rank_filter(torch.from_numpy(px8).cuda(), 40).cpu().numpy()
    bad += int(not np.array_equal(out, O.iot_filter(px8, 81)))
os.environ.pop("MTB_CT_CTB4_R", None)
for fam in ("sortnet", "vert", "vert2", "ctmf", "lob", ""):
    os.environ["MTB_KERNEL"] = fam
    for r in (1, 2, 3, 5, 20, 40):
        out = mtb.rank_filter(torch.from_numpy(px8).cuda(), r).cpu().numpy()
        bad += int(not np.array_equal(out, O.iot_filter(px8, 2 * r + 1)))
        out16 = mtb.rank_filter(torch.from_numpy(px16).cuda(), min(r, 34)).cpu().numpy()
        bad += int(not np.array_equal(out16, O.iot_filter(px16, 2 * min(r, 34) + 1)))
    b = torch.from_numpy(np.stack([px8[:60, :80]] * 3)).cuda()
    mtb.rank_filter(b, 4)
torch.cuda.synchronize()
print("mismatches:", bad)
sys.exit(1 if bad else 0)
