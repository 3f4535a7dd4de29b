#!/bin/bash
# Device BVH builder: GPU tests, then build/trace timings.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/bvh_smi.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_device_bvh.py -x -q > gpurun_out/bvh_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/bvh_tests.log
timeout 900 python tools/bvh_device_bench.py c2 c3 c5 > gpurun_out/bvh_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bvh_bench.log
tail -n 3 gpurun_out/bvh_tests.log gpurun_out/bvh_bench.log
