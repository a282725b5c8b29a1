#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29523"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for algo in default Ring; do
  for wl in bert gpt2; do
    if [ $algo = default ]; then unset NCCL_ALGO; else export NCCL_ALGO=$algo; fi
    timeout 300 $TR bench.py --gpus $NG --workload $wl > gpurun_out/algo_${algo}_$wl.log 2>&1
    echo "NCCL_ALGO=$algo $wl rc=$? ours $(grep -o '"bus_gbps_per_gpu": [0-9.]*, "higher' gpurun_out/algo_${algo}_$wl.log) nccl $(grep -o '"nccl_compare": {.*"best": "[a-z]*"}' gpurun_out/algo_${algo}_$wl.log | grep -o '"bus_gbps_per_gpu": [0-9.]*, "best": "[a-z]*"')"
  done
done
