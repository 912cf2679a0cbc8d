#!/bin/bash
# Same-box A/B of shared libraries: scripts/gpu_ablib.sh TAG lib1 lib2 ...
TAG=$1; shift
mkdir -p gpurun_out
for rep in 1 2; do
for L in "$@"; do
  B3D_LIB=$L timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${TAG}.log 2>&1
  echo "$L rep$rep $(python -c "import json; d=json.loads(open('gpurun_out/ab_${TAG}.log').read().strip().splitlines()[-1]); print(round(d['value']/1e6,3),'Mhyp/s')")"
done; done
