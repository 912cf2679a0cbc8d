#!/bin/bash
# Same-box A/B of library builds over the cfg1 bench and the legs:
#   scripts/ab_libs.sh "lib1 lib2" "legs..."   ("" = the in-tree build)
LIBS=$1; LEGS=$2
for rep in 1 2; do
for L in $LIBS; do
  [ "$L" == "cur" ] && unset B3D_LIB || export B3D_LIB=$L
  timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-extra 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L cfg1 value', round(d['value']), 'kernel_us', round(1e3*d['kernel_ms'],1))"
  for leg in $LEGS; do
    timeout 300 python scripts/leg.py $leg 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('   $leg', {k: d.get(k) for k in ('value','fps','s')})"
  done
done; done
