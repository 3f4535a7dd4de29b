#!/bin/bash
# Round-2 evidence in one gpurun call, everything under gpurun_out/ev2/ (the
# ncu reports are summarised on the box and deleted: gpurun copies back at
# most 64 MiB).  TAG names the files (default r02).
cd "$GRAFT_REPO_ROOT"
TAG=${TAG:-r02}
O=gpurun_out/ev2
mkdir -p $O
export EF_TRAFFIC_DIR=$O
./tools/micro/cache_bw > $O/${TAG}_micro_peaks.json 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
# the default line (C5) and the reference arm, as the driver runs them
timeout 900 python bench.py --steps 20 --warmup 5 > $O/${TAG}_bench_c5.jsonl 2> $O/${TAG}_bench_c5.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/${TAG}_reference_c5.jsonl 2> $O/${TAG}_reference_c5.err
for c in c1 c2 c3; do
  st=200; [ $c = c3 ] && st=20
  timeout 1500 python bench.py --config $c --steps $st --warmup 5 > $O/${TAG}_bench_$c.jsonl 2> $O/${TAG}_bench_$c.err
done
timeout 900 python bench.py --config c2 --steps 200 --warmup 5 --inflight 2 --no-cpu-baseline > $O/${TAG}_bench_c2_inflight2.jsonl 2> $O/${TAG}_bench_c2_inflight2.err
timeout 900 python bench.py --config c1 --steps 200 --warmup 5 --inflight 2 --no-cpu-baseline > $O/${TAG}_bench_c1_inflight2.jsonl 2> $O/${TAG}_bench_c1_inflight2.err
timeout 1500 python bench.py --config c4 --steps 20 --warmup 3 > $O/${TAG}_bench_c4.jsonl 2> $O/${TAG}_bench_c4.err
python tools/probe_simt.py c5 65536 > $O/${TAG}_simt.txt 2>&1
python tools/probe_simt.py c3 >> $O/${TAG}_simt.txt 2>&1
for c in c1 c2; do python tools/probe_step.py $c >> $O/${TAG}_step_anatomy.txt 2>&1; done
# launch lists + one full capture per hot kernel, summarised here
for c in c5 c2; do
  B="python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv $B > /dev/null 2>&1
done
cap() {  # config kernel-regex command...
  c=$1; k=$2; shift 2
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $O/prof_$c "$@" > /dev/null 2>&1
  L=""; [ -f $O/launches_$c.csv ] && L=$O/launches_$c.csv
  python tools/summarize_ncu.py "$L" $O/prof_$c.ncu-rep $O/${TAG}_$c $c > /dev/null 2>&1
  ncu -i $O/prof_$c.ncu-rep --page source --csv --print-source cuda,sass > $O/src_$c.csv 2>/dev/null
  python tools/ncu_lines.py $O/src_$c.csv 30 > $O/${TAG}_${c}_lines.txt 2>&1
  rm -f $O/prof_$c.ncu-rep $O/src_$c.csv
}
cap c5 trace_kernel python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline
cap c3 trace_kernel python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline
cap c2 trace_kernel python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline
cap c2tail tail_kernel python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline
cap c4 render_kernel python tools/c4_once.py 65536
tail -n 2 $O/smoke.log $O/pytest_gpu.log
for f in $O/${TAG}_*.jsonl; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads([l for l in open(f) if l.startswith('{')][-1])
    r = d.get('roofline', {})
    rd = d.get('roofline_device') or {}
    print(f.split('/')[-1], d.get('value'), d.get('unit'), 'frac', r.get('frac'), 'dev frac', rd.get('frac'),
          'e2e', (d.get('e2e') or {}).get('value'), 'cpu', (d.get('cpu_baseline') or {}).get('value'))
except Exception as e:
    print(f, 'failed', e)
PY
done
du -sh gpurun_out
