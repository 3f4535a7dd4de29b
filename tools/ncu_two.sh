#!/bin/bash
# Two full captures summarised on the box (raw + source CSV), reports deleted.
#   A="ENV=..." B="ENV=..." CFG=c3 TAG=x bash tools/ncu_two.sh
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-ncu2}
mkdir -p $O
for v in A B; do
  envs=${!v}
  [ -z "$envs" ] && continue
  env $envs timeout 900 ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-trace_kernel} -s ${SKIP:-2} -c 1 \
     -o $O/$v python bench.py --config ${CFG:-c3} --steps 1 --warmup 3 --no-cpu-baseline > $O/$v.log 2>&1
  ncu -i $O/$v.ncu-rep --page raw --csv > $O/${v}_raw.csv 2>/dev/null
  ncu -i $O/$v.ncu-rep --page source --csv --print-source cuda,sass > $O/${v}_src.csv 2>/dev/null
  gzip -f $O/${v}_src.csv
  rm -f $O/$v.ncu-rep
done
ls -la $O
