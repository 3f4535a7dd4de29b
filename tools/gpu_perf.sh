# quick perf check of the trace configs (no CPU baseline), plus GPU tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ "${TESTS:-1}" = "1" ]; then
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
for c in ${CONFIGS:-c2 c3 c5}; do
  st=50; [ $c = c3 ] && st=5; [ $c = c5 ] && st=2
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/perf_$c.log 2>&1
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads([l for l in open(f"gpurun_out/perf_{c}.log") if l.startswith("{")][-1])
    r = d["roofline"]
    print(f"{c}: {d['value']/1e9:.3f} Gseg/s  step {d['ms_per_step']:.3f} ms  kernel {r['kernel_ms_per_launch']:.3f} ms  frac {r['frac']:.3f}  e2e {d['e2e']['value']/1e9:.3f}")
except Exception as e:
    print(c, "failed", e, open(f"gpurun_out/perf_{c}.log").read()[-500:])
PY
done > gpurun_out/perf_summary.txt 2>&1
cat gpurun_out/perf_summary.txt
