#!/bin/bash
# Round-end evidence bundle (one gpurun call, one GPU): GPU tests + smoke,
# bench line, reference arm, the issue-ceiling ncu pass (profiles/ncu_issue.json),
# the ncu launch list of the bench, and --set full captures of the changed
# kernels summarised on the box.  Every ncu command runs only after the same
# command exited 0 without ncu.
set -u
out=gpurun_out/ev
mkdir -p $out
timeout 1500 python -m pytest tests -q -m gpu > $out/gpu_tests.log 2>&1; echo "tests rc=$?" >> $out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
python bench.py > $out/bench.json 2> $out/bench.err
python bench.py --impl reference > $out/bench_ref.json 2> $out/bench_ref.err
python tools/ncu_issue.py run > $out/issue_plain.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum,sm__cycles_elapsed.avg,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:k_ --csv --log-file $out/issue.csv python tools/ncu_issue.py run > $out/issue_ncu.log 2>&1
cp gpurun_out/ncu_issue_manifest.json $out/ 2>/dev/null
python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extra > $out/launch_plain.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-extra > $out/launch_ncu.log 2>&1
for spec in "cfg2_r63 2 63 k_bandmma" "cfg2_r100 2 100 k_bandtc" "cfg3_r31 3 31 k_lowsel" "cfg3_r15 3 15 k_lowsel" "cfg3_r31hi 3 31 k_colhist4p"; do
  set -- $spec
  python tools/one_launch.py $2 $3 > /dev/null 2>&1 &&
    ncu --set full --import-source on --clock-control none -k regex:$4 -s 1 -c 1 -o $out/prof_$1 \
      python tools/one_launch.py $2 $3 > $out/prof_$1.log 2>&1
  python tools/ncu_summary.py $out/prof_$1.ncu-rep > $out/sum_$1.txt 2>&1
  python tools/hot_lines.py $out/prof_$1.ncu-rep 25 > $out/hot_$1.txt 2>&1
  rm -f $out/prof_$1.ncu-rep
done
ls -la $out
