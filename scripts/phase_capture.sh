#!/bin/bash
# ncu --set full capture of one score launch of a bench leg, exported as the
# per-line source page and grouped into kernel phases (render_score.cuh lines).
#   scripts/phase_capture.sh TAG LEG SKIP     e.g. r2s sharded 1
TAG=$1; LEG=$2; SKIP=${3:-1}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:render_score_kernel<\\(bool\\)0, \\(bool\\)1" -s "$SKIP" -c 1 \
    -o gpurun_out/ph_${TAG}_${LEG} python scripts/leg.py $LEG > gpurun_out/ph_${TAG}_${LEG}.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/ph_${TAG}_${LEG}.ncu-rep --page source --csv --print-source cuda,sass \
    > gpurun_out/ph_${TAG}_${LEG}_src.csv 2>/dev/null
bash profiles/ncu_details.sh gpurun_out/ph_${TAG}_${LEG}.ncu-rep > gpurun_out/ph_${TAG}_${LEG}_details.txt
python profiles/ncu_phases.py gpurun_out/ph_${TAG}_${LEG}_src.csv \
    rasterbox:106-150 clipped:151-327 windows:340-411 tilemask:240-290 sweep:447-627 \
    drain_small:629-696 drain_queue:698-787 zinit:848-867 seg:868-885 phase1:886-1007 \
    huge:1008-1017 staging:1018-1039 out:1040-1062 D1:1064-1090 coef:1091-1107 \
    D2:1108-1161 D3:1162-1208 kernelA:1296-1337 vertexB:1338-1396 region:1397-1465 \
    > gpurun_out/ph_${TAG}_${LEG}_phases.txt
python profiles/ncu_lines.py gpurun_out/ph_${TAG}_${LEG}_src.csv 40 > gpurun_out/ph_${TAG}_${LEG}_lines.txt
rm -f gpurun_out/ph_${TAG}_${LEG}_src.csv
