cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in c1 c2 c3 c5; do
  st=20; [ $c = c3 ] && st=10; [ $c = c5 ] && st=3
  timeout 900 python bench.py --config $c --steps $st --warmup 3 > gpurun_out/bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$c.log
done
