cd $GRAFT_REPO_ROOT
line() { python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('$1', round(d['value']/1e9,4), 'step ms', round(d['ms_per_step'],4))"; }
for ci in 1 1.5 2 3; do for lf in 2 3 4 6; do EF_BVH_CI=$ci EF_BVH_MAXLEAF=$lf timeout 300 python bench.py --config c2 --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | line "ci=$ci leaf=$lf c2"; done; done
for sp in 0 0.25 1.0; do EF_BVH_SPLITS=$sp timeout 300 python bench.py --config c2 --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | line "splits=$sp c2"; done
