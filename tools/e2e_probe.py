"""Host-path breakdown: pinned copy bandwidth and mtb_filter_host per radius."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads, paper_1105_3829_b200 as mtb

H = W = 4096
base = workloads.cfg2_blur_sp_u8(H, W)
hs = torch.empty((H, W), dtype=torch.uint8).pin_memory()
hs.numpy()[...] = base
hd = torch.empty((H, W), dtype=torch.uint8).pin_memory()
d = torch.empty((H, W), dtype=torch.uint8, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(hs, non_blocking=True)), ("d2h", lambda: hd.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20): fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 20
    print(name, f"{dt*1e3:.3f} ms  {H*W/dt/1e9:.1f} GB/s")
s2 = torch.cuda.Stream()
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(20):
    d.copy_(hs, non_blocking=True)
    with torch.cuda.stream(s2): hd.copy_(d, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 20
print("bidir", f"{dt*1e3:.3f} ms")
for bands in (None, "1", "2", "4", "8", "16"):
    if bands: os.environ["MTB_HOST_BANDS"] = bands
    else: os.environ.pop("MTB_HOST_BANDS", None)
    row = []
    for r in (1, 3, 7, 15, 31, 63):
        mtb.filter_host_buffer(hs.numpy(), r, out=hd.numpy())
        t = time.perf_counter()
        for _ in range(5): mtb.filter_host_buffer(hs.numpy(), r, out=hd.numpy())
        row.append((time.perf_counter() - t) / 5 * 1e3)
    print("bands", bands, " ".join(f"{x:.2f}" for x in row), f"sum {sum(row):.2f} ms")
