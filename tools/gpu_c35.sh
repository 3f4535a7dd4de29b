#!/bin/bash
for c in c3 c5 c3 c5; do
  st=10; [ $c = c5 ] && st=3
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$c', round(d['value']/1e9,4), 'step', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3))"
done
