import json, sys
sys.path.insert(0, ".")
import bench
from paper_2312_08715_b200 import b3d, configs
bench.LEG_CPU["enabled"] = True
ctx = b3d.GpuContext(0)
out = bench.run_smc_leg(ctx, b3d, configs)
print(json.dumps({k: out[k] for k in ("seconds", "renders_device", "cpu_baseline")}))
