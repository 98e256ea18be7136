#!/bin/bash
# e2e (frame sequence) of the config-2 sweep under each streaming mode / a few orders
for s in 4 0 1 2 3; do
  echo -n "MTB_FRAMES_STREAM=$s: "
  MTB_FRAMES_STREAM=$s python bench.py --no-cpu --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e']['value'], d['value'])"
done
for perm in "0,5,1,4,2,3" "0,5,4,3,2,1" "1,5,0,4,2,3" "0,4,1,5,2,3" "5,0,4,1,3,2"; do
  echo -n "MTB_FRAMES_PERM=$perm: "
  MTB_FRAMES_PERM=$perm python bench.py --no-cpu --no-extra 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e']['value'])"
done
