for ic in 2 4 8 16; do for oc in 2 4 8 16; do echo "in=$ic out=$oc"; MTB_HOST_IN_CHUNKS=$ic MTB_HOST_OUT_CHUNKS=$oc timeout 60 python tools/e2e_probe.py 2>&1 | grep "bands None"; done; done
