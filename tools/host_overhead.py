import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1105_3829_b200 as mtb
for H in (64, 1024, 4096):
    src = torch.empty((H, 4096), dtype=torch.uint8).pin_memory().numpy(); src[...] = 7
    dst = torch.empty((H, 4096), dtype=torch.uint8).pin_memory().numpy()
    for r in (1, 15):
        for _ in range(3): mtb.filter_host_buffer(src, r, out=dst)
        t = time.perf_counter()
        for _ in range(20): mtb.filter_host_buffer(src, r, out=dst)
        print(H, r, f"{(time.perf_counter()-t)/20*1e3:.3f} ms")
