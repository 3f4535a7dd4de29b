#!/bin/bash
# Round evidence: smoke, GPU tests, the default bench line (C2 + CPU
# baseline), the reference arm, and every config's bench line.
TAG=${TAG:-r01d}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c2.jsonl 2> gpurun_out/${TAG}_bench_c2.err
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_reference_c2.jsonl 2> gpurun_out/${TAG}_reference_c2.err
for c in c1 c3 c5; do
  st=200; [ $c = c3 ] && st=20; [ $c = c5 ] && st=5
  timeout 1500 python bench.py --config $c --steps $st --warmup 3 > gpurun_out/${TAG}_bench_$c.jsonl 2> gpurun_out/${TAG}_bench_$c.err
done
timeout 1500 python bench.py --config c4 --steps 20 --warmup 3 > gpurun_out/${TAG}_bench_c4.jsonl 2> gpurun_out/${TAG}_bench_c4.err
tail -n 2 gpurun_out/smoke.log gpurun_out/pytest_gpu.log
for f in gpurun_out/${TAG}_*.jsonl; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads([l for l in open(f) if l.startswith('{')][-1])
    r = d.get('roofline', {})
    print(f.split('/')[-1], d.get('value'), d.get('unit'), 'frac', r.get('frac'), 'e2e', (d.get('e2e') or {}).get('value'),
          'cpu', (d.get('cpu_baseline') or {}).get('value'))
except Exception as e:
    print(f, 'failed', e)
PY
done
