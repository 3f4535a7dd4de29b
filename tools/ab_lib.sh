#!/bin/bash
# A/B two library builds on one box: OLD=path/to/old.so, config CFG (default c4)
for i in 1 2; do
  for lib in "$OLD" paper_1803_00430_b200/libechoforge_b200.so; do
    EF_LIB_PATH=$lib timeout 1500 python bench.py --config ${CFG:-c4} --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$lib'.split('/')[-1], d['value'], round(d['ms_per_step'],3), round(d['roofline']['frac'],3))"
  done
done
