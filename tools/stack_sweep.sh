#!/bin/bash
# EF_SMEM_STACK sweep (shared traversal-stack entries per thread) for C3/C5 (768-thread kernels) and C2
for d in 12 8 4 16; do
  for c in c3 c5; do
    st=10; [ $c = c5 ] && st=3
    EF_SMEM_STACK=$d timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('stack $d $c', round(d['value']/1e9,4), round(d['ms_per_step'],3))"
  done
done
for d in 16 12 8; do
  EF_SMEM_STACK=$d timeout 900 python bench.py --config c2 --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('stack $d c2', round(d['value']/1e9,4), round(d['ms_per_step'],3))"
done
