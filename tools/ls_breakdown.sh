#!/bin/bash
# per-kernel times (ncu, cold) of one config-3 launch per radius: tools/ls_breakdown.sh "7 15 31"
mkdir -p gpurun_out/s5
for r in $1; do
  python tools/one_launch.py ${CFG:-3} $r > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum --clock-control none -k regex:k_ -s 5 --csv --log-file gpurun_out/s5/ls_launch_$r.csv python tools/one_launch.py ${CFG:-3} $r > /dev/null 2>&1
  python - <<P
import csv
rows=list(csv.reader(open("gpurun_out/s5/ls_launch_$r.csv")))
hdr=[i for i,x in enumerate(rows) if x and x[0]=="ID"][0]
d={}
for x in rows[hdr+1:]:
    d.setdefault((x[0],x[4][:48]),{})[x[-3]]=x[-1]
for (i,k),v in d.items():
    print($r, i, k, "us", float(v["gpu__time_duration.sum"].replace(",",""))/1e3, "Minst", float(v["sm__inst_executed.sum"].replace(",",""))/1e6)
P
done
