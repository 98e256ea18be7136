"""Random shapes / radii 3..63 / ranks / slabs / image kinds through the default 16-bit dispatch
(device-selected: candidate-bucket path on spread data, two-phase kernel on compact data) and through
the forced candidate-bucket path (MTB_KERNEL=lowsel) against the CPU oracle."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1105_3829_b200 as mtb
from paper_1105_3829_b200 import _lib
from oracle import oracle as O
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 321)
N = int(sys.argv[2]) if len(sys.argv) > 2 else 160
bad = 0
seen = {}
for it in range(N):
    r = int(rng.integers(3, 64))
    lo = max(1, (2 * r + 1) // 2)
    H = int(rng.integers(lo, lo + 150)); W = int(rng.integers(lo, lo + 500))
    kind = it % 8
    if kind == 0: px = rng.integers(0, 65536, (H, W))
    elif kind == 1: px = (np.arange(H)[:, None] * 301 + np.arange(W)[None, :] * 77) % 65536           # ramps
    elif kind == 2: px = rng.integers(0, 4, (H, W)) * 21845                                           # four values
    elif kind == 3: px = np.clip(rng.normal(40000, 6000, (H, W)), 0, 65535)                           # wide bell
    elif kind == 4:                                                                                   # noise with a saturated and a constant region
        px = rng.integers(0, 65536, (H, W)); px[: H // 2, W // 3:] = 65535; px[H // 2:, : W // 5] = 1234
    elif kind == 5: px = rng.integers(0, 1024, (H, W)) * 64                                           # 10 bits in 16
    elif kind == 6: px = np.where(rng.random((H, W)) < 0.5, rng.integers(0, 65536, (H, W)), 30000 + rng.integers(0, 200, (H, W)))
    else: px = np.full((H, W), int(rng.integers(0, 65536)))                                           # constant
    px = px.astype(np.uint16)
    n = 2 * r + 1
    rank = [None, 1, n * n, int(rng.integers(1, n * n + 1))][it % 4]
    a = int(rng.integers(0, H)); b = int(rng.integers(a + 1, H + 1))
    rows = (a, b) if it % 3 == 0 else None
    if it % 2: os.environ["MTB_KERNEL"] = "lowsel"
    else: os.environ.pop("MTB_KERNEL", None)
    os.environ["MTB_LS_PH"] = "4" if it % 5 == 0 else "8"
    dev = torch.from_numpy(px).cuda()
    kw = {}
    if rank: kw["rank"] = rank
    if rows: kw["rows"] = rows
    out = mtb.rank_filter(dev, r, **kw).cpu().numpy()
    k = _lib.last_kernel(); seen[k] = seen.get(k, 0) + 1
    ref = O.iot_filter(px, n, rank=rank) if rank else O.iot_filter(px, n)
    if rows: ref = ref[a:b]
    if not np.array_equal(out, ref):
        bad += 1
        print("MISMATCH", it, r, H, W, kind, rank, rows, k, int((out != ref).sum()), flush=True)
print("bad =", bad, seen)
sys.exit(1 if bad else 0)
