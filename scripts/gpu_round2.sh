#!/bin/bash
# One GPU-box pass (round 2): parity tests, smoke, bench, e2e breakdown, and
# with `ncu` the launch list + `--set full` captures of the score kernel of
# every leg (cfg1 bench, cfg2 coarse-to-fine, cfg3 scene graph, cfg4
# tracking, cfg5 sharded).
#   scripts/gpu_round2.sh TAG [ncu] [notest]
TAG=${1:-run}
mkdir -p gpurun_out
if [ "$3" != "notest" ]; then
  timeout 1500 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/pytest_${TAG}.log 2>&1
  echo "pytest rc=$?"; tail -3 gpurun_out/pytest_${TAG}.log
  timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
  tail -1 gpurun_out/smoke_${TAG}.log
fi
timeout 900 python bench.py --steps 30 --warmup 5 --cpu-seconds 8 > gpurun_out/bench_${TAG}.log 2>&1
echo "bench rc=$?"; tail -1 gpurun_out/bench_${TAG}.log | cut -c1-600
timeout 300 python scripts/e2e_breakdown.py > gpurun_out/e2e_${TAG}.log 2>&1; echo "e2e rc=$?"
cat gpurun_out/e2e_${TAG}.log
if [ "$2" == "ncu" ]; then
  B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra"
  timeout 300 $B > gpurun_out/plain_${TAG}.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_${TAG}.csv $B > /dev/null 2>&1
  echo "launch list rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_score \
      -s 2 -c 1 -o gpurun_out/prof_${TAG}_cfg1 $B > gpurun_out/ncu_${TAG}_cfg1.log 2>&1
  echo "ncu cfg1 rc=$?"
  # leg captures: skip the observation renders / warm-up launches
  # (score-mode launches only: demangled names "render_score_kernel<false, true, ...")
  for spec in "coarse_to_fine 5" "scene_graph 1" "tracking 10" "sharded 1"; do
    set -- $spec
    timeout 600 python scripts/leg.py $1 > gpurun_out/leg_${TAG}_$1.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
        -k "regex:render_score_kernel<\\(bool\\)0, \\(bool\\)1" \
        -s $2 -c 1 -o gpurun_out/prof_${TAG}_$1 python scripts/leg.py $1 \
        > gpurun_out/ncu_${TAG}_$1.log 2>&1
    echo "ncu $1 rc=$?"
  done
fi
