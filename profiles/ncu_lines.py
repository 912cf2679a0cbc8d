"""Summarise an ncu source page (--print-source cuda,sass --csv) per CUDA
source line: instructions executed, stall samples, average active threads.
Usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > m.csv
       python profiles/ncu_lines.py m.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = "?"
agg = {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 10 or r[2] != "-":
        continue
    try:
        ie = float(r[hdr.index("Instructions Executed")])
        st = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
        th = float(r[hdr.index("Thread Instructions Executed")])
    except (ValueError, IndexError):
        continue
    key = (fname, int(r[0]))
    a = agg.setdefault(key, [0.0, 0.0, 0.0, r[1][:80]])
    a[0] += ie
    a[1] += st
    a[2] += th
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instructions {ti:.3e}  stall samples {ts:.0f}")
for (f, ln), v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    act = v[2] / v[0] if v[0] else 0
    print(f"{v[0]/ti*100:5.1f}% inst {v[1]/ts*100:5.1f}% stall thr{act:5.1f} {f}:{ln:<4d} {v[3]}")
