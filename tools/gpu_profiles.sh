# round evidence: launch list (C2 bench) + one full capture per hot kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B1="python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline"
B2="python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline"
B3="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline"
B5="python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline"
B4="python tools/c4_once.py 65536"
$B2 > gpurun_out/p_c2.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $B2 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 3 -c 1 -o gpurun_out/prof_c2 $B2 > /dev/null 2>&1
$B1 > gpurun_out/p_c1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $B1 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 3 -c 1 -o gpurun_out/prof_c1 $B1 > /dev/null 2>&1
$B3 > gpurun_out/p_c3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 3 -c 1 -o gpurun_out/prof_c3 $B3 > /dev/null 2>&1
$B5 > gpurun_out/p_c5.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:trace_kernel -s 3 -c 1 -o gpurun_out/prof_c5 $B5 > /dev/null 2>&1
$B4 > gpurun_out/p_c4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 3 -c 1 -o gpurun_out/prof_c4 $B4 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
