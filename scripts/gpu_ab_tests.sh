#!/bin/bash
# GPU parity tests, then a same-box A/B of library builds: scripts/gpu_ab_tests.sh TAG lib1 lib2 ...
TAG=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_${TAG}.log
bash scripts/gpu_ablib.sh $TAG "$@"
