for cfg in "8 24" "8 48" "8 96" "16 48" "16 96"; do set -- $cfg; python tools/probe.py --cfg 2 --radii 31,63 --kernels ctmf --reps 3 --env "MTB_CT_S=$1;MTB_CT_MIN_TH=$2;MTB_CT_TH=$2" 2>&1 | grep -v "^{" | sed "s/^/S=$1 TH=$2 /" ; done > gpurun_out/sweep2.log
python tools/probe.py --cfg 5 --radii 7,25 --kernels "" --reps 3 2>&1 | grep -v "^{" > gpurun_out/probe_cfg5.log || true
