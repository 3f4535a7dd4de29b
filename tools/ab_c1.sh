#!/bin/bash
for lib in "$OLD" paper_1803_00430_b200/libechoforge_b200.so "$OLD" paper_1803_00430_b200/libechoforge_b200.so; do
  EF_LIB_PATH=$lib timeout 900 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('c1', '$lib'.split('/')[-1], round(d['value']/1e9,4), round(d['ms_per_step'],4), round(d['roofline']['kernel_ms_per_launch'],4))"
done
