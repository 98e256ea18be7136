"""Small run exercising every kernel family AND the host pipelines (for
compute-sanitizer memcheck / racecheck; one tool per gpurun call):

    compute-sanitizer --tool memcheck  python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py

Device-resident calls cover each kernel family at tile-edge widths; the
host entries (filter_image -> mtb_filter_host_rows in bands or one
streaming launch, filter_host_frames -> mtb_filter_host_frames with the
streamed first frame, filter_images, multi-device slabs) run at r = 7, 15
and 63, 8- and 16-bit, pinned and pageable.  Every result is checked
against the oracle; exit 1 on any mismatch.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1105_3829_b200 as mtb  # noqa: E402
import workloads  # noqa: E402
from oracle import oracle as O  # noqa: E402

torch.cuda.set_device(0)
rng = np.random.default_rng(3)
px8 = rng.integers(0, 256, (90, 300), dtype=np.uint8)
px16 = rng.integers(0, 65536, (70, 90)).astype(np.uint16)
bad = []


def check(tag, got, ref):
    if not np.array_equal(got, ref):
        bad.append(tag)


# 3x3 kernels (TMA-staged for W % 16 == 0) and the merge networks at tile-edge widths
for W in (16, 1040, 1043):
    for bits, dt in ((8, np.uint8), (16, np.uint16)):
        im = rng.integers(0, 1 << bits, (37, W)).astype(dt)
        for r in (1, 2, 3):
            check(("net", W, bits, r), mtb.rank_filter(torch.from_numpy(im).cuda(), r).cpu().numpy(),
                  O.iot_filter(im, 2 * r + 1))
# CTMF with up-front snapshots in both register budgets
for ctb in ("1", "1000"):
    os.environ["MTB_CT_CTB4_R"] = ctb
    os.environ["MTB_KERNEL"] = "ctmf"
    check(("ctmf", ctb), mtb.rank_filter(torch.from_numpy(px8).cuda(), 40).cpu().numpy(), O.iot_filter(px8, 81))
os.environ.pop("MTB_CT_CTB4_R", None)
for fam in ("sortnet", "vert", "ctmf", "colhist16s", ""):
    os.environ["MTB_KERNEL"] = fam
    for r in (1, 2, 3, 5, 20, 40):
        check((fam, 8, r), mtb.rank_filter(torch.from_numpy(px8).cuda(), r).cpu().numpy(),
              O.iot_filter(px8, 2 * r + 1))
        r16 = min(r, 34)
        check((fam, 16, r16), mtb.rank_filter(torch.from_numpy(px16).cuda(), r16).cpu().numpy(),
              O.iot_filter(px16, 2 * r16 + 1))
    b = torch.from_numpy(np.stack([px8[:60, :80]] * 3)).cuda()
    out = mtb.rank_filter(b, 4).cpu().numpy()
    check((fam, "batch"), out[1], O.iot_filter(px8[:60, :80], 9))
os.environ.pop("MTB_KERNEL", None)

# host pipelines: bands (pageable), streaming launch (pinned, r >= 12), frames, batches, slabs
f8 = workloads.cfg2_blur_sp_u8(300, 280, seed=5)
f16 = workloads.cfg4_three_gauss_u16(280, 300, seed=6)
u16 = rng.integers(0, 65536, (260, 200)).astype(np.uint16)
for img in (f8, f16, u16):
    pin = torch.from_numpy(img).pin_memory().numpy()
    for r in (7, 15, 63):
        if 2 * r + 1 > 2 * min(img.shape) + 1:
            continue
        ref = O.iot_filter(img, 2 * r + 1)
        out, _ = mtb.filter_image(img, 2 * r + 1)
        check(("filter_image", img.dtype.name, r), out.pixels, ref)
        check(("host_pinned", img.dtype.name, r), mtb.filter_host_buffer(pin, r), ref)
        out, _ = mtb.filter_image(img, 2 * r + 1, devices=[0, 0])
        check(("slabs", img.dtype.name, r), out.pixels, ref)
    outs = mtb.filter_host_frames([pin, img, pin, img], [7, 15, 63, 3])
    for o, r in zip(outs, [7, 15, 63, 3]):
        check(("frames", img.dtype.name, r), o, O.iot_filter(img, 2 * r + 1))
b5 = workloads.cfg5_batch_u8(4, 128, 120)
outs = mtb.filter_images(b5, 15, devices=[0, 0])
for i in range(4):
    check(("images", i), outs[i], O.iot_filter(b5[i], 15))
torch.cuda.synchronize()
print("mismatches:", len(bad), bad[:10])
sys.exit(1 if bad else 0)
