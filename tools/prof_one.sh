#!/bin/bash
# usage: tools/prof_one.sh NAME CFG R KERNEL [ENV=V ...]  -> gpurun_out/prof_NAME.ncu-rep
# (captures the 2nd launch matching KREGEX, default k_: the first call warms up;
# config 2 r = 63 launches the snapshot pre-pass and the tile kernel per call)
name=$1; cfg=$2; r=$3; kern=$4; shift 4
for kv in "$@"; do export "$kv"; done
python tools/one_launch.py $cfg $r $kern > /dev/null 2>&1 || { echo "run failed"; exit 1; }
ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-k_} -s ${KSKIP:-1} -c 1 -o gpurun_out/prof_$name python tools/one_launch.py $cfg $r $kern > gpurun_out/prof_$name.log 2>&1
tail -1 gpurun_out/prof_$name.log
