# SMC leg timing, in-tree library vs another build (B3D_LIB), with the phase profile
#   scripts/smc_ab.sh LIB
for L in cur $1; do
  [ "$L" == "cur" ] && unset B3D_LIB || export B3D_LIB=$L
  for i in 1 2; do
    B3D_SMC_PROFILE=1 timeout 300 python scripts/leg.py smc > /tmp/smc_$i.log 2>&1
    echo "$L run $i: $(tail -1 /tmp/smc_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['seconds'], d['renders_device'])")"
    grep -v "^{" /tmp/smc_$i.log | tail -12
  done
done
