"""Group an ncu source page (--print-source cuda,sass --csv) by kernel phase
(line ranges of render_score.cu given as name:lo-hi) and print warp-
instructions and stall samples per phase.
Usage: python profiles/ncu_phases.py m.csv name:lo-hi ..."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
ranges = []
for a in sys.argv[2:]:
    n, r = a.split(":")
    lo, hi = r.split("-")
    ranges.append((n, int(lo), int(hi)))
fname, hdr = "?", None
agg = {}
tot_i = tot_s = 0.0
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
    except (ValueError, IndexError):
        continue
    tot_i += ie
    tot_s += st
    ln = int(r[0])
    name = "other:" + fname
    if fname.startswith("render_score.cu"):
        for n, lo, hi in ranges:
            if lo <= ln <= hi:
                name = n
                break
    a = agg.setdefault(name, [0.0, 0.0])
    a[0] += ie
    a[1] += st
print(f"total warp-instructions {tot_i:.3e} stall samples {tot_s:.0f}")
for n, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{n:28s} inst {v[0]/tot_i*100:5.1f}%  stall {v[1]/tot_s*100:5.1f}%")
