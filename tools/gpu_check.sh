#!/bin/bash
# GPU tests, then C2 x3 / C3 / C5 bench lines and the single long C2 path.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 2 gpurun_out/pytest_gpu.log
for c in c2 c2 c2 c3 c5; do
  st=200; [ $c = c3 ] && st=10; [ $c = c5 ] && st=3
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$c', round(d['value']/1e9,4), 'step', round(d['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms_per_launch'],4), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']/1e9,4))"
done
python tools/probe_trace.py c2 single 2>&1 | tail -1
