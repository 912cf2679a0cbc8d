#!/bin/bash
# Full bench line (all legs) per library: scripts/ab_full.sh TAG lib1 lib2 ...
TAG=$1; shift
mkdir -p gpurun_out
for L in "$@"; do
  B3D_LIB=$L timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --tracking-frames 40 > gpurun_out/abf_${TAG}.log 2>&1
  echo "$L $(python -c "
import json; d=json.loads(open('gpurun_out/abf_${TAG}.log').read().strip().splitlines()[-1])
print('cfg1', round(d['value']/1e6,3), 'c2f', round(d['coarse_to_fine']['value']/1e6,3), 'track_fps', round(d['tracking']['fps'],1), 'scene', round(d['scene_graph']['value']/1e6,3), 'cfg5', round(d['sharded_enumeration']['value']/1e6,3))")"
done
