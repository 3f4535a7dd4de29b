cd $GRAFT_REPO_ROOT
for big in 0 1; do
  for c in c2 c3 c5; do
    st=30; [ $c = c3 ] && st=4; [ $c = c5 ] && st=1
    EF_TRACE_BIG=$big python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/cs.log 2>&1
    python -c "
import json; d=json.loads([l for l in open('gpurun_out/cs.log') if l.startswith('{')][-1])
print('big=$big $c', round(d['value']/1e9,3), 'Gseg/s kernel', round(d['roofline']['kernel_ms_per_launch'],3), 'ms')"
  done
done > gpurun_out/shape_sweep.txt 2>&1
