#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for tma in 1 0; do
  RAVNEST_B200_TMA=$tma timeout 300 python bench.py --steps 40 --warmup 5 > gpurun_out/tma_$tma.log 2>&1
  echo "N1 tma=$tma rc=$? $(grep -o '"avg_kernel_ms": [0-9.]*' gpurun_out/tma_$tma.log) $(grep -o '"frac": [0-9.]*' gpurun_out/tma_$tma.log)"
  RAVNEST_B200_TMA=$tma timeout 300 python bench.py --steps 20 --warmup 5 --workload resnet50 > gpurun_out/tma_r_$tma.log 2>&1
  echo "N1 resnet tma=$tma rc=$? $(grep -o '"avg_kernel_ms": [0-9.]*' gpurun_out/tma_r_$tma.log) $(grep -o '"frac": [0-9.]*' gpurun_out/tma_r_$tma.log)"
done
