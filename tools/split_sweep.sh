#!/bin/bash
# Spatial-split sweep (EF_BVH_SPLITS budget, EF_BVH_SPLIT_ALPHA threshold):
# frame time, work per segment and the single long path, per config.
mkdir -p gpurun_out
for c in ${CONFIGS:-c2 c3 c5}; do
  for a in ${ALPHAS:-1e-5 1e-3 1e-2 1e-1}; do
    EF_BVH_SPLITS=${SPLITS:-0.5} EF_BVH_SPLIT_ALPHA=$a timeout 600 python tools/probe_trace.py $c knobs 2>&1 | sed "s/^/[alpha $a] /"
  done
done > gpurun_out/split_sweep.txt 2>&1
cat gpurun_out/split_sweep.txt
