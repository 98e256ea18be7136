"""Copy / filter timeline model of the frame-sequence host path
(mtb_filter_host_frames): three serial resources
(host->device copies, kernels, device->host copies), a ring of NB buffer
pairs, the first frame optionally streamed (its kernel starts after the first
quarter of its rows and cannot finish before the last; its results leave
in four chunks as its rows complete).  Prints the
best orders of the config-2 sweep and the time of the heavy/light default.

    python tools/frames_model.py [--copy-ms 0.31] [--nb 3]
"""

import argparse
import itertools

# config-2 kernel times per radius (ms, bench.py per-radius events)
KERNEL_MS = {1: 0.023, 3: 0.170, 7: 0.226, 15: 0.323, 31: 0.499, 63: 0.534}


def simulate(order, nb, copy_ms, stream_first=True):
    h_end = k_end = d_end = 0.0
    k_done, d_done = {}, {}
    for q, r in enumerate(order):
        hs = max(h_end, k_done[q - nb]) if q >= nb else h_end
        he = h_end = hs + copy_ms
        first = stream_first and q == 0
        ks = max(k_end, hs + copy_ms / 4 if first else he)
        if q >= nb:
            ks = max(ks, d_done[q - nb])
        ke = max(ks + KERNEL_MS[r], he if first else 0.0)
        k_end = k_done[q] = ke
        if first:  # results leave in 4 chunks as the kernel's rows complete
            for i in range(4):
                d_end = max(d_end, ks + KERNEL_MS[r] * (i + 1) / 4) + copy_ms / 4
            d_done[q] = d_end
        else:
            d_end = d_done[q] = max(d_end, ke) + copy_ms
    return d_end


def heavy_light(radii):
    byr = sorted(radii, reverse=True)
    lo, hi, out = 0, len(byr) - 1, []
    for q in range(len(byr)):
        if q & 1:
            out.append(byr[hi])
            hi -= 1
        else:
            out.append(byr[lo])
            lo += 1
    return tuple(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--copy-ms", type=float, default=0.31)
    ap.add_argument("--nb", type=int, default=3)
    a = ap.parse_args()
    res = sorted((simulate(o, a.nb, a.copy_ms), o) for o in itertools.permutations(KERNEL_MS))
    for t, o in res[:5]:
        print(f"{t:.3f} ms  {o}")
    hl = heavy_light(list(KERNEL_MS))
    print(f"heavy/light {hl}: {simulate(hl, a.nb, a.copy_ms):.3f} ms; input order: "
          f"{simulate(tuple(KERNEL_MS), a.nb, a.copy_ms):.3f} ms")


if __name__ == "__main__":
    main()
