"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) as markdown shares."""
import csv
import sys
from collections import defaultdict

src, dst = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(src)) if len(r) > 5]
hdr, data = rows[0], rows[1:]
ki, vi, gi, bi = (hdr.index(k) for k in ('Kernel Name', 'Metric Value', 'Grid Size', 'Block Size'))
agg, grid = defaultdict(list), {}
for r in data:
    agg[r[ki]].append(float(r[vi].replace(',', '')))
    grid[r[ki]] = (r[gi], r[bi])
tot = sum(sum(v) for k, v in agg.items() if 'mtb::' in k)
out = ["# ncu launch list -- `bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extra` (config-2 sweep)", "",
       "`ncu --metrics gpu__time_duration.sum --clock-control none --csv` on 1x B200.  Per-launch times are",
       "cold-cache and serialised: compare SHARES.  Raw csv beside this file.", "",
       "| kernel | launches | mean us | share of our kernel time | grid | block |", "|---|---|---|---|---|---|"]
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    share = f"{100 * sum(v) / tot:.1f}%" if 'mtb::' in k else "(L2 flush, not ours)"
    out.append(f"| `{k[:80]}` | {len(v)} | {sum(v) / len(v) / 1000:.1f} | {share} | {grid[k][0]} | {grid[k][1]} |")
open(dst, 'w').write("\n".join(out) + "\n")
print("\n".join(out))
