#!/bin/bash
for dbg in ${DBGS:-0 2 4 6 8 16 24 26}; do
  echo "== DBG=$dbg (2: no row update, 4: no outputs, 8: no descent, 16: first k-tile only)"
  MTB_BM_DBG=$dbg MTB_BM_TW=${TW:-512} MTB_BM_WAVES=${WV:-1} timeout 300 python tools/probe.py --cfg 2 --radii ${RADII:-31,63} --kernels bandmma --reps 5 2>&1 | grep "^bandmma" | cut -c1-60
done
