#!/bin/bash
# Key counters of an ncu --set full report: profiles/ncu_summary.sh X.ncu-rep
ncu -i "$1" --page details --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin))
keep=('Duration','Executed Ipc Active','Issue Slots Busy','Achieved Active Warps Per SM','Eligible Warps Per Scheduler','Avg. Active Threads Per Warp','Executed Instructions','Theoretical Occupancy','Registers Per Thread','Dynamic Shared Memory Per Block','Warp Cycles Per Issued Instruction','Compute (SM) Throughput','DRAM Throughput','L1/TEX Hit Rate','L2 Hit Rate','Grid Size','Block Size')
seen=set()
for row in r[1:]:
    if row[-4] in keep and row[-4] not in seen: seen.add(row[-4]); print(f'{row[-4]:45s} {row[-2]:>14s} {row[-3]}')
"
