#!/bin/bash
# Same-box A/B with kernel-only time and the hypothesis-count sweep per library.
TAG=$1; shift
mkdir -p gpurun_out
for L in "$@"; do
  B3D_LIB=$L timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-extra > gpurun_out/abd_${TAG}.log 2>&1
  echo "$L $(python -c "import json; d=json.loads(open('gpurun_out/abd_${TAG}.log').read().strip().splitlines()[-1]); print(round(d['value']/1e6,3),'Mhyp/s kernel_ms',round(d['kernel_ms'],4),'step_ms',round(d['ms_per_step'],4))")"
  B3D_LIB=$L timeout 300 python scripts/hyp_scaling.py 888 1024 2048
done
