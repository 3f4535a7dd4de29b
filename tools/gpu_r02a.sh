#!/bin/bash
# Round-2 first evidence call: cache peaks, GPU tests, default (C5) bench, C5 launch list + full capture.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02a
mkdir -p $O
./tools/micro/cache_bw > $O/micro.json 2>&1
timeout 600 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_c5.jsonl 2> $O/bench_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 3 -c 1 \
  -o $O/prof_c5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c5.log 2>&1
ls -la $O
tail -3 $O/pytest_gpu.log
cat $O/micro.json
head -c 1500 $O/bench_c5.jsonl
