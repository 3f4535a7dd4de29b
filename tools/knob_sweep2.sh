#!/bin/bash
# BVH build knobs (SAH triangle cost, max leaf size) on the C2 bench line
for ci in 1 1.5 2 3; do for leaf in 2 4; do
  EF_BVH_CI=$ci EF_BVH_MAXLEAF=$leaf timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ci $ci leaf $leaf', round(d['value']/1e9,4), round(d['step_ms_quantiles']['p50'],4))"
done; done
