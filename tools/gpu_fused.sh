#!/bin/bash
# Fused trace + reduce-scatter: GPU tests, a 2-rank plumbing run of bench.py
# on one GPU (gloo; numbers meaningless), and a quick N=1 bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py -x -q > gpurun_out/fused_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/fused_tests.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29555 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo \
  > gpurun_out/bench_n2_gloo.log 2>&1
echo "n2 rc=$?" >> gpurun_out/bench_n2_gloo.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2_quick.log 2>&1
echo "c2 rc=$?" >> gpurun_out/bench_c2_quick.log
tail -n 3 gpurun_out/fused_tests.log gpurun_out/bench_n2_gloo.log gpurun_out/bench_c2_quick.log
