cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/r02n
for f in 1 2 3 4; do for c in c2 c1; do
python bench.py --config $c --steps 100 --warmup 5 --inflight $f --no-cpu-baseline 2>gpurun_out/r02n/err_$c$f | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c','inflight',$f, round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],4), 'ms/frame', 'e2e', round(d['e2e']['value']/1e9,3), 'lat', d.get('frame_latency_ms',{}).get('p50'), d.get('step_ms_quantiles',{}).get('p50'))" || tail -3 gpurun_out/r02n/err_$c$f
done; done
