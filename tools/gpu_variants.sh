#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for v in 0 1 2 3; do
  RAVNEST_B200_VARIANT=$v timeout 300 python bench.py --steps 30 --warmup 5 > gpurun_out/var_$v.log 2>&1
  echo "N1 variant $v rc=$? $(grep -o '"avg_kernel_ms": [0-9.]*' gpurun_out/var_$v.log) $(grep -o '"frac": [0-9.]*' gpurun_out/var_$v.log)"
done
for v in 0 1 3; do
  RAVNEST_B200_VARIANT=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus $NG --steps 30 --warmup 5 --protocol pull --nccl 0 > gpurun_out/varN_$v.log 2>&1
  echo "N$NG pull variant $v rc=$? $(grep -o '"bus_gbps_per_gpu": [0-9.]*' gpurun_out/varN_$v.log)"
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus $NG --steps 30 --warmup 5 > gpurun_out/bench_auto.log 2>&1
echo "N$NG auto rc=$? $(grep -o '"bus_gbps_per_gpu": [0-9.]*' gpurun_out/bench_auto.log) $(grep -o '"protocol": "[a-z]*"' gpurun_out/bench_auto.log)"
