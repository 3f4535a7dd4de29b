#!/bin/bash
# A/B of library builds on one box, alternating: LIBS="x.so y.so" CONFIGS="c5 c3"
# REPS=2 TESTS=1 (pytest -m gpu first) TAG=name
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-ab}
mkdir -p $O
if [ "${TESTS:-0}" = 1 ]; then
  timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q -x ${TESTARGS:-} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
  tail -15 $O/pytest_gpu.log
fi
for rep in $(seq 1 ${REPS:-2}); do
for c in ${CONFIGS:-c5}; do
  for lib in ${LIBS}; do
    st=20; [ $c = c5 ] && st=5; [ $c = c2 ] && st=100; [ $c = c1 ] && st=100
    EF_LIB_PATH=paper_1803_00430_b200/$lib timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > $O/b.jsonl 2> $O/b.err
    python - "$lib" "$c" $O/b.jsonl <<'PY'
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[3]) if l.startswith('{')][-1])
    r = d.get('roofline_device') or {}
    print(f"{sys.argv[1]:40s} {sys.argv[2]} {d['value']/1e9:.4f} G/s {d['ms_per_step']:.3f} ms nodes/seg {r.get('nodes_per_segment', 0):.2f} tris/seg {r.get('triangles_per_segment', 0):.2f} segs {d.get('segments_per_step')} clk {d.get('clocks', {}).get('sm_mhz')}", flush=True)
except Exception as e:
    print(sys.argv[1], sys.argv[2], 'failed', e, open(sys.argv[3].replace('.jsonl', '.err')).read()[-600:])
PY
  done
done
done
