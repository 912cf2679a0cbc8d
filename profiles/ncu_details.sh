#!/bin/bash
# Committed summary of an ncu --set full capture:
#   profiles/ncu_details.sh X.ncu-rep > profiles/rNN_render_score_details.txt
# (section summary, the raw counters bench.py's roofline reads, stall reasons per issue)
R=$1
bash "$(dirname "$0")/ncu_summary.sh" "$R"
ncu -i "$R" --page raw --csv 2>/dev/null | python3 -c "
import csv, sys
r = list(csv.reader(sys.stdin))
h, u, v = r[0], r[1], r[2]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'smsp__inst_executed.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'launch__registers_per_thread',
        'launch__grid_size']
for w in want:
    if w in h:
        i = h.index(w)
        print(f'{w:75s} {v[i]} {u[i]}')
st = {n.split('stalled_')[1].split('_per_issue')[0]: float(v[i]) for i, n in enumerate(h)
      if n.startswith('smsp__average_warps_issue_stalled_') and n.endswith('_per_issue_active.ratio')}
print('stalls/issue: ' + ' '.join(f'{k}={x:.2f}' for k, x in sorted(st.items(), key=lambda kv: -kv[1]) if x >= 0.05))
"
