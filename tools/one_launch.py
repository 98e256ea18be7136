"""Run one rank-filter launch (for ncu): python tools/one_launch.py CFG R [KERNEL]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
import paper_1105_3829_b200 as mtb  # noqa: E402

cfg, r = int(sys.argv[1]), int(sys.argv[2])
if len(sys.argv) > 3 and sys.argv[3]:
    os.environ["MTB_KERNEL"] = sys.argv[3]
px = {1: lambda: workloads.cfg1_uniform_u8(4096, 4096), 2: workloads.cfg2_blur_sp_u8,
      3: workloads.cfg3_uniform_u16, 4: workloads.cfg4_three_gauss_u16}[cfg]()
src = torch.from_numpy(px).cuda()
out = torch.empty_like(src)
for _ in range(2):
    mtb.rank_filter(src, r, out=out)
torch.cuda.synchronize()
print("ok")
