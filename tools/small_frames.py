import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import workloads, paper_1105_3829_b200 as mtb
from paper_1105_3829_b200 import _lib
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for (H, W) in ((512, 512), (1024, 1024), (2048, 2048), (1080, 1920)):
    px = workloads.cfg2_blur_sp_u8(H, W)
    src = torch.from_numpy(px).cuda(); out = torch.empty_like(src)
    for r in (32, 40, 63, 80, 100):
        if r > min(H, W): continue
        row = []
        for kern in ("", "colhist", "ctmf", "bandmma", "bandtc"):
            os.environ["MTB_KERNEL"] = kern
            mtb.rank_filter(src, r, out=out); torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                flush.fill_(1)
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record(); mtb.rank_filter(src, r, out=out); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            row.append(f"{kern or 'default'}={sorted(ts)[2]:.3f}")
        print(H, W, r, " ".join(row), flush=True)
