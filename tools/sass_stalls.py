"""Per-SASS-instruction executed counts and stall samples of an ncu report.
usage: python tools/sass_stalls.py REPORT.ncu-rep > listing.txt"""
import csv
import subprocess
import sys

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr = None
out = []
for r in rows:
    if "Instructions Executed" in r and "Source" in r:
        hdr = r
        ci, cs, csrc = r.index("Instructions Executed"), r.index("Warp Stall Sampling (All Samples)"), r.index("Source")
        cadr = r.index("Address") if "Address" in r else 0
        continue
    if hdr is None or len(r) <= max(ci, cs, csrc):
        continue
    try:
        out.append((r[cadr], int(r[ci]), int(r[cs]), r[csrc]))
    except ValueError:
        pass
tot = sum(x[2] for x in out) or 1
ti = sum(x[1] for x in out) or 1
print(f"# total warp-instructions {ti}, stall samples {tot}")
for a, i, s, src in out:
    print(f"{a[-5:]} {i:>10} {100.0 * i / ti:5.2f}% {100.0 * s / tot:5.2f}%  {src[:100]}")
