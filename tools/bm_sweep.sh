#!/bin/bash
# timing sweep of the band-MMA kernel over stripe widths / waves (config 2)
for tw in ${TWS:-256 512}; do for wv in ${WVS:-1}; do
  echo "== TW=$tw WAVES=$wv"
  MTB_BM_TW=$tw MTB_BM_WAVES=$wv timeout 300 python tools/probe.py --cfg 2 --radii ${RADII:-15,31,63} --kernels bandmma --reps 5 2>&1 | grep "^bandmma" | cut -c1-75
done; done
