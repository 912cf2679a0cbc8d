#!/bin/bash
# Same-box A/B of one env switch: scripts/ab_quick.sh VAR "v0 v1 ..." [legs]
VAR=$1; VALS=$2; LEGS=$3
for v in $VALS $VALS; do
  env $VAR=$v timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-extra 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$VAR=$v cfg1 value', round(d['value']), 'kernel_us', round(1e3*d['kernel_ms'],1), 'e2e', round(d['e2e']['value']))"
  for leg in $LEGS; do
    env $VAR=$v timeout 300 python scripts/leg.py $leg 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('   $leg', {k: d.get(k) for k in ('value','fps','s','ms_per_schedule')})"
  done
done
