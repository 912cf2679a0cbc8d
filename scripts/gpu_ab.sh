#!/bin/bash
# A/B quick bench: scripts/gpu_ab.sh TAG  -> tests + bench with cull off/on
TAG=${1:-ab}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_${TAG}.log
B3D_OCCLUSION_CULL=1 timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_${TAG}_cull.log 2>&1; echo "pytest(cull) rc=$?"; tail -2 gpurun_out/pytest_${TAG}_cull.log
for c in 0 1; do
  B3D_OCCLUSION_CULL=$c timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_c$c.log 2>&1
  echo "cull=$c $(python -c "import json,sys; d=json.loads(open('gpurun_out/bench_${TAG}_c$c.log').read().strip().splitlines()[-1]); print(round(d['value']/1e6,3),'Mhyp/s kernel_ms', d['roofline'] and d['roofline']['kernel_ms'], 'e2e', round(d['e2e']['value']/1e6,3))")"
done
