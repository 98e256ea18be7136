"""The window-key pass of compact 16-bit data (k_colhist4p_u8<..., uint16_t, 1>, MTB_KERNEL=wk16) against the
CPU oracle on ragged frames of compact, drifting, spread and mixed data, every rank position; then
config-4 timings against the two-phase kernel.  usage: python tools/check_wk16.py [radii] [--time]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
import paper_1105_3829_b200 as mtb  # noqa: E402
from paper_1105_3829_b200 import _lib  # noqa: E402
from oracle import oracle as O  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
radii = [int(x) for x in args[0].split(",")] if args else [3, 4, 7, 15, 16, 17, 24, 31, 40, 63]
rng = np.random.default_rng(12)
bad = 0


def frames(H, W):
    compact = (30000 + rng.normal(0, 60, (H, W))).clip(0, 65535).astype(np.uint16)
    drift = (np.add.outer(np.arange(H) * 3, np.arange(W) * 2) + rng.normal(0, 40, (H, W)) + 500).clip(0, 65535).astype(np.uint16)
    noise = rng.integers(0, 65536, (H, W)).astype(np.uint16)
    mixed = compact.copy()
    mixed[:, W // 2:] = noise[:, W // 2:]
    low = rng.integers(0, 90, (H, W)).astype(np.uint16)          # window clamped at 0
    high = (65535 - rng.integers(0, 90, (H, W))).astype(np.uint16)  # ... and at the top
    cfg4 = workloads.cfg4_three_gauss_u16(H, W)
    return (("compact", compact), ("drift", drift), ("noise", noise), ("mixed", mixed), ("low", low), ("high", high), ("cfg4", cfg4))


os.environ["MTB_KERNEL"] = "wk16"
for (H, W) in ((97, 333), (40, 700), (300, 64), (131, 257)):
    for name, px in frames(H, W):
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
                    print(f"MISMATCH {name} {H}x{W} r={r} rank={rank}: {len(d)} px, first {d[0]} got {got[tuple(d[0])]} ref {ref[tuple(d[0])]} kernel {_lib.last_kernel()}", flush=True)
    print(H, W, "done; kernel", _lib.last_kernel(), "bad", bad, flush=True)
os.environ.pop("MTB_KERNEL")
print("bad =", bad, flush=True)

if "--time" in sys.argv:
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    drift = (np.add.outer(np.arange(4096) * 2, np.arange(4096)) // 4 + np.random.default_rng(3).normal(0, 40, (4096, 4096)) + 500).clip(0, 65535).astype(np.uint16)
    for cfg, px in (("4 (8192^2)", workloads.cfg4_three_gauss_u16()), ("drift (4096^2)", drift)):
        src = torch.from_numpy(px).cuda()
        out = torch.empty_like(src)
        for r in (4, 7, 15, 31, 47, 63):
            row = []
            for label, env in (("old", {"MTB_U16_WK8": "0"}), ("wk8", {}), ("waves2", {"MTB_WK16_WAVES": "2"}), ("waves8", {"MTB_WK16_WAVES": "8"})):
                for k in ("MTB_U16_WK8", "MTB_WK16_WAVES"):
                    os.environ.pop(k, None)
                os.environ.update(env)
                mtb.rank_filter(src, r, out=out)
                torch.cuda.synchronize()
                ts = []
                for _ in range(5):
                    flush.fill_(1)
                    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                    e0.record()
                    mtb.rank_filter(src, r, out=out)
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
                row.append(f"{label}={sorted(ts)[2]:.3f}")
                if label == "old":
                    ref = out.clone()
                elif not torch.equal(ref, out):
                    row.append("DIFFERS")
                    bad += 1
            print("cfg", cfg, "r", r, " ".join(row), "|", _lib.last_kernel(), flush=True)
sys.exit(1 if bad else 0)
