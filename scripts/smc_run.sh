# SMC leg: GPU parity tests of run_smc / b3d_infer, then the leg twice
timeout 600 python -m pytest tests -q -m gpu -k "smc or infer or capi" 2>&1 | tail -3
for i in 1 2; do timeout 300 python scripts/leg.py smc 2>&1 | tail -1 | python -c "
import json, sys; d = json.loads(sys.stdin.read())
print({k: d[k] for k in ('seconds', 'renders', 'renders_device', 'log_evidence', 'map_child')})"; done
