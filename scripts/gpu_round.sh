#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench, optional ncu captures.
#   scripts/gpu_round.sh TAG [ncu]
TAG=${1:-run}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?" ; tail -3 gpurun_out/pytest_${TAG}.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_${TAG}.log
timeout 600 python bench.py --steps 30 --warmup 5 --cpu-seconds 8 > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_${TAG}.log
if [ "$2" == "ncu" ]; then
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/plain_${TAG}.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_score -s 2 -c 1 -o gpurun_out/prof_${TAG} python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/ncu_${TAG}.log 2>&1
  echo "ncu rc=$?"; tail -2 gpurun_out/ncu_${TAG}.log
fi
