#!/bin/bash
# Quick A/B call: GPU tests (optional) + bench lines of the given configs.
#   TESTS=1 CONFIGS="c5 c3 c2" TAG=x bash tools/gpu_quick.sh
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-quick}
mkdir -p $O
if [ "${TESTS:-0}" = 1 ]; then
  timeout 900 python -m pytest tests -m gpu -q -x ${TESTARGS:-} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
  tail -15 $O/pytest_gpu.log
fi
for c in ${CONFIGS:-c5}; do
  st=20; [ $c = c5 ] && st=5; [ $c = c2 ] && st=100; [ $c = c1 ] && st=100
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > $O/bench_$c.jsonl 2> $O/bench_$c.err
  python - $O/bench_$c.jsonl <<'PY'
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1])
    r = d.get('roofline_device') or {}
    print(sys.argv[1].split('/')[-1], round(d['value'] / 1e9, 4), 'G/s', round(d['ms_per_step'], 3), 'ms',
          'nodes/seg', round(r.get('nodes_per_segment') or 0, 2), 'tris/seg', round(r.get('triangles_per_segment') or 0, 2),
          'dev frac', r.get('frac'), 'clk', d.get('clocks', {}).get('sm_mhz'))
except Exception as e:
    print(sys.argv[1], 'failed', e, open(sys.argv[1].replace('.jsonl', '.err')).read()[-800:])
PY
done
