#!/bin/bash
# A/B of (library, environment) pairs: scripts/ab_env.sh TAG "lib|ENV=1" ...
TAG=$1; shift
mkdir -p gpurun_out
for rep in 1 2; do
for spec in "$@"; do
  L=${spec%%|*}; E=${spec#*|}; [ "$E" == "$spec" ] && E=""
  env $E B3D_LIB=$L timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-extra > gpurun_out/abe_${TAG}.log 2>&1
  echo "$spec rep$rep $(python -c "import json; d=json.loads(open('gpurun_out/abe_${TAG}.log').read().strip().splitlines()[-1]); print(round(d['value']/1e6,3),'Mhyp/s')")"
done; done
