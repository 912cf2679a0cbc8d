#!/bin/bash
# Device time of the SMC leg's kernels vs its wall time (is run_smc kernel-bound?)
timeout 300 python scripts/leg.py smc > gpurun_out/smc_leg.log 2>&1; tail -1 gpurun_out/smc_leg.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smc_launches.csv python scripts/leg.py smc > /dev/null 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/smc_launches.csv")))
hdr = None; tot = {}; n = {}
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"].split("(")[0][:50]
            v = float(d["Metric Value"].replace(",", "")) * (1e-3 if d["Metric Unit"] == "nsecond" else 1)
            tot[k] = tot.get(k, 0) + v; n[k] = n.get(k, 0) + 1
for k in sorted(tot, key=lambda k: -tot[k]): print(f"{tot[k]/1e3:9.2f} ms  {n[k]:6d}  {k}")
PY
