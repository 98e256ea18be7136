#!/bin/bash
# Copies the bundle tools/round_evidence.sh left in gpurun_out/ev into profiles/ (run here, after gpurun).
set -e
ev=gpurun_out/ev
(cat $ev/gpu_tests.log; cat $ev/smoke.log) > profiles/r2_gpu_tests.log
cp $ev/bench.json profiles/r2_bench_final.json
cp $ev/bench_ref.json profiles/r2_bench_reference_arm.json
cp $ev/issue.csv profiles/r2_ncu_issue_launches.csv
cp $ev/ncu_issue_manifest.json profiles/r2_ncu_issue_manifest.json
cp $ev/launches.csv profiles/r2_ncu_launches.csv
[ -f $ev/stress_u16.txt ] && cp $ev/stress_u16.txt profiles/r2_stress_u16.txt
python tools/ncu_issue.py parse $ev/issue.csv $ev/ncu_issue_manifest.json > profiles/ncu_issue.json
for spec in "cfg2_r63 k_bandmma_u8 r2_ncu_bandmma_cfg2_r63" "cfg2_r100 k_bandtc_u8 r2_ncu_bandtc_cfg2_r100" \
            "cfg3_r31 k_lowsel_u16 r2_ncu_lowsel_cfg3_r31" "cfg3_r15 k_lowsel_u16 r2_ncu_lowsel_cfg3_r15" \
            "cfg3_r31hi k_colhist4p_u8<u16_coarse_key> r2_ncu_hi16_cfg3_r31"; do
  set -- $spec
  (echo "# ncu --set full, $2, ${1} (tools/round_evidence.sh); summary then hot source lines"; cat $ev/sum_$1.txt; echo; cat $ev/hot_$1.txt) > profiles/$3.txt
done
