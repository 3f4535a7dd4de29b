cd $GRAFT_REPO_ROOT
for rep in 1 2; do for big in 0 1; do
    EF_TRACE_BIG=$big python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cs.log 2>&1
    python -c "
import json; d=json.loads([l for l in open('gpurun_out/cs.log') if l.startswith('{')][-1])
print('big=$big c5', round(d['value']/1e9,3), 'Gseg/s kernel', round(d['roofline']['kernel_ms_per_launch'],3), 'ms', d['clocks'])"
done; done > gpurun_out/shape_sweep2.txt 2>&1
