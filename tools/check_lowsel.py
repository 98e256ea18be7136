"""The 16-bit candidate-list path (k_lowsel_u16, MTB_KERNEL=lowsel) against the CPU oracle on
ragged frames of spread, compact and mixed data (mixed: blocks overflow their lists and go to the
two-phase kernel), every rank position, slabs and a batch; then config-3 timings against the
kernels it replaces.  usage: python tools/check_lowsel.py [radii] [--time]"""
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
radii = [int(x) for x in args[0].split(",")] if args else [3, 4, 7, 12, 15, 16, 17, 24, 31, 40, 63]
rng = np.random.default_rng(11)
bad = 0


def frames(H, W):
    noise = rng.integers(0, 65536, (H, W)).astype(np.uint16)
    compact = (30000 + rng.normal(0, 300, (H, W))).clip(0, 65535).astype(np.uint16)
    mixed = noise.copy()
    mixed[:, W // 3: 2 * W // 3] = compact[:, W // 3: 2 * W // 3]
    mixed[H // 2:, : W // 4] = 65535
    twelve = (rng.integers(0, 4096, (H, W)) * 16).astype(np.uint16)
    return (("noise", noise), ("compact", compact), ("mixed", mixed), ("twelve", twelve))


for ph in ("4", "8", "16m"):
    os.environ["MTB_LS_PH"] = ph.rstrip("m")
    os.environ["MTB_LS_HI"] = "mma" if ph.endswith("m") else ""
    os.environ["MTB_KERNEL"] = "lowsel"
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
                        print(f"MISMATCH PH={ph} {name} {H}x{W} r={r} rank={rank}: {len(d)} px, first {d[0]} got {got[tuple(d[0])]} ref {ref[tuple(d[0])]} kernel {_lib.last_kernel()}", flush=True)
        print("PH", ph, H, W, "done; kernel", _lib.last_kernel(), "bad", bad, flush=True)
os.environ.pop("MTB_LS_PH")
os.environ.pop("MTB_LS_HI")
# default dispatch (device-selected), a batch
os.environ.pop("MTB_KERNEL")
stack = np.stack([f for _, f in frames(120, 200)])
got = mtb.rank_filter(torch.from_numpy(stack).cuda(), 9).cpu().numpy()
for i in range(stack.shape[0]):
    if not np.array_equal(got[i], O.iot_filter(stack[i], 19)):
        bad += 1
        print("MISMATCH batch image", i)
print("batch done; kernel", _lib.last_kernel())
print("bad =", bad, flush=True)

if "--time" in sys.argv:
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    twelve = np.random.default_rng(5).integers(0, 4096, (4096, 4096)).astype(np.uint16)
    for cfg, px in ((3, workloads.cfg3_uniform_u16()), (12, twelve), (4, workloads.cfg4_three_gauss_u16(4096, 4096))):
        src = torch.from_numpy(px).cuda()
        out = torch.empty_like(src)
        for r in (4, 7, 15, 23, 31, 47, 63):
            row = []
            for label, env in (("old", {"MTB_U16_LIST": "0"}), ("ph4", {"MTB_LS_PH": "4"}), ("ph8", {"MTB_LS_PH": "8"}),
                               ("ph16", {"MTB_LS_PH": "16"}), ("ph24", {"MTB_LS_PH": "24"}), ("ph32", {"MTB_LS_PH": "32"}), ("pair", {"MTB_LS_HI": "pair"}), ("mma", {"MTB_LS_HI": "mma"})):
                if cfg in (4, 12) and label not in ("old", "ph8"):
                    continue
                for k in ("MTB_U16_LIST", "MTB_LS_PH", "MTB_LS_SEG", "MTB_LS_HI"):
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
