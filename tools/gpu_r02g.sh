#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r02g}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_c5.jsonl 2> $O/bench_c5.err
head -c 600 $O/bench_c5.jsonl; echo
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 3 -c 1 \
  -o $O/prof_c5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c5.log 2>&1
ls -la $O
