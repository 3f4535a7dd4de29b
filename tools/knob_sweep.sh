cd $GRAFT_REPO_ROOT
for ci in 0.5 1 2 4; do for leaf in 1 2 4 8; do
EF_BVH_CI=$ci EF_BVH_MAXLEAF=$leaf python tools/probe_trace.py c2 knobs
done; done > gpurun_out/knobs.log 2>&1
