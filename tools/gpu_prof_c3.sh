cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/c3_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 3 -c 1 -o gpurun_out/prof_c3 $B > gpurun_out/ncu_c3.log 2>&1
