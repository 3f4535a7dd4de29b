#!/bin/bash
# A/B two library builds on one box over C2/C3/C5 (OLD=path/to/old.so)
for c in c2 c3 c5; do
  st=200; [ $c = c3 ] && st=10; [ $c = c5 ] && st=3
  for lib in "$OLD" paper_1803_00430_b200/libechoforge_b200.so "$OLD" paper_1803_00430_b200/libechoforge_b200.so; do
    EF_LIB_PATH=$lib timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$c', '$lib'.split('/')[-1], round(d['value']/1e9,4), round(d['ms_per_step'],3))"
  done
done
