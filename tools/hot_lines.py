"""Top source lines of an ncu report by instructions executed / stall samples.
usage: python tools/hot_lines.py REPORT.ncu-rep [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
cur = None
ie = smp = None
res = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if "Instructions Executed" in r:
        ie = r.index("Instructions Executed")
        smp = r.index("Warp Stall Sampling (All Samples)")
        continue
    if ie is None:
        continue
    if len(r) > ie and r[0] not in ("", "Function Name") and len(r) > 2 and r[2] == "-":
        try:
            res.append((int(r[ie]), int(r[smp]), cur, int(r[0]), r[1][:90]))
        except ValueError:
            pass
tot = sum(x[0] for x in res) or 1
ts = sum(x[1] for x in res) or 1
print(f"total instructions {tot}")
for v, s_, f, ln, src in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{100 * v / tot:5.1f}% {100 * s_ / ts:5.1f}%  {f}:{ln}  {src}")
