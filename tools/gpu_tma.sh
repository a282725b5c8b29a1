#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for rep in 1 2; do
for v in 0 4; do
  RAVNEST_B200_TMA_VARIANT=$v timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/tmav_$v.log 2>&1
  echo "N1 tma variant=$v rc=$? $(grep -o '"avg_kernel_ms": [0-9.]*' gpurun_out/tmav_$v.log) $(grep -o '"frac": [0-9.]*' gpurun_out/tmav_$v.log)"
done
done
