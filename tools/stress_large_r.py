"""Random shapes / radii 32..127 / ranks / image kinds through the default 8-bit dispatch (k_bandmma_u8,
k_bandtc_u8) against the CPU oracle."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1105_3829_b200 as mtb
from paper_1105_3829_b200 import _lib
from oracle import oracle as O
rng = np.random.default_rng(123)
bad = 0
seen = {}
for it in range(70):
    r = int(rng.integers(32, 128))
    lo = r
    H = int(rng.integers(lo, lo + 200)); W = int(rng.integers(lo, lo + 1400))
    if it % 7 == 0: W = 4096 + int(rng.integers(-3, 4)); H = max(lo, 40)
    kind = it % 4
    if kind == 0: px = rng.integers(0, 256, (H, W), dtype=np.uint8)
    elif kind == 1: px = ((np.arange(H)[:, None] * 3 + np.arange(W)[None, :] * 2) % 256).astype(np.uint8)
    elif kind == 2:
        px = rng.integers(0, 4, (H, W), dtype=np.uint8) * 85
    else:
        px = np.clip(rng.normal(200, 60, (H, W)), 0, 255).astype(np.uint8)
    n = 2 * r + 1
    rank = [None, 1, n * n, int(rng.integers(1, n * n + 1))][it % 4]
    dev = torch.from_numpy(px).cuda()
    out = (mtb.rank_filter(dev, r, rank=rank) if rank else mtb.rank_filter(dev, r)).cpu().numpy()
    k = _lib.last_kernel(); seen[k] = seen.get(k, 0) + 1
    ref = O.iot_filter(px, n, rank=rank) if rank else O.iot_filter(px, n)
    if not np.array_equal(out, ref):
        bad += 1
        print("MISMATCH", it, r, H, W, kind, rank, k, int((out != ref).sum()))
print("bad =", bad, seen)
