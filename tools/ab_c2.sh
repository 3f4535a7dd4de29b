#!/bin/bash
# A/B of an env knob on the C2 bench, alternating on the same box.
# usage: KNOB=EF_BVH_SPLITS A=0 B=0.5 bash tools/ab_c2.sh
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in "$A" "$B"; do
    env $KNOB=$v timeout 600 python bench.py --config ${CFG:-c2} --steps ${STEPS:-200} --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$KNOB=$v', round(d['value']/1e9,4), 'step', round(d['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms_per_launch'],4), 'e2e', round(d['e2e']['value']/1e9,4))"
  done
done > gpurun_out/ab.txt 2>&1
cat gpurun_out/ab.txt
