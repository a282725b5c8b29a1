#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
for v in 0 1 2 3; do
  for rep in 1 2; do
  RAVNEST_B200_TMA_VARIANT=$v timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/tmav_$v.log 2>&1
  echo "N1 tma variant=$v rc=$? $(grep -o '"avg_kernel_ms": [0-9.]*' gpurun_out/tmav_$v.log) $(grep -o '"frac": [0-9.]*' gpurun_out/tmav_$v.log)"
  done
done
RAVNEST_B200_TMA=0 timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/tma_0.log 2>&1
echo "N1 no-tma rc=$? $(grep -o '"avg_kernel_ms": [0-9.]*' gpurun_out/tma_0.log) $(grep -o '"frac": [0-9.]*' gpurun_out/tma_0.log)"
