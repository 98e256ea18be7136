#!/bin/bash
# Round-end measurement bundle (run under gpurun): bench line, ncu launch list,
# --set full captures summarised ON THE BOX (the .ncu-rep files stay there,
# except the dominant kernel's), so gpurun_out/ stays small.
set -u
out=gpurun_out
python bench.py > $out/bench_full.json 2> $out/bench_full.err || exit 1
python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extra > /dev/null 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extra > $out/ncu_l.log 2>&1
for spec in "r1 2 1" "r3 2 3" "r7 2 7" "r15 2 15" "r31 2 31" "r63 2 63" "r63pre 2 63" "cfg4_r15 4 15" "cfg3_r15 3 15" "cfg3_r31 3 31"; do
  set -- $spec
  if [ "$1" = "r63pre" ]; then KREGEX=k_ctmf_pre KSKIP=1 tools/prof_one.sh f_$1 $2 $3 "" > /dev/null
  elif [ "$1" = "r63" ]; then KREGEX=k_ctmf_u8 KSKIP=1 tools/prof_one.sh f_$1 $2 $3 "" > /dev/null
  else tools/prof_one.sh f_$1 $2 $3 "" > /dev/null; fi
  python tools/ncu_summary.py $out/prof_f_$1.ncu-rep > $out/sum_f_$1.txt 2>&1
  python tools/hot_lines.py $out/prof_f_$1.ncu-rep 25 > $out/hot_f_$1.txt 2>&1
  ncu -i $out/prof_f_$1.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; un=rows[1]; v=rows[2]
scale={'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}
g=lambda k: float(v[h.index(k)].replace(',',''))*scale[un[h.index(k)]]
print(int(g('dram__bytes_read.sum')+g('dram__bytes_write.sum')))
" > $out/traffic_f_$1.txt
  [ "$1" = "${KEEP_REP:-r63}" ] || rm -f $out/prof_f_$1.ncu-rep
done
ls -la $out
