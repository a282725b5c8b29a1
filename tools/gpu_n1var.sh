#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
for v in 0 3 1; do
  RAVNEST_B200_VARIANT=$v timeout 300 python bench.py --steps 40 --warmup 5 --nccl 0 > gpurun_out/var_$v.log 2>&1
  echo "N1 variant $v rc=$? $(grep -o '"avg_kernel_ms": [0-9.]*' gpurun_out/var_$v.log) $(grep -o '"frac": [0-9.]*' gpurun_out/var_$v.log)"
done
for v in 0 3; do
  RAVNEST_B200_VARIANT=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus 2 --steps 30 --warmup 5 --protocol pull --nccl 0 > gpurun_out/varN_$v.log 2>&1
  echo "N2 pull variant $v rc=$? $(grep -o '"bus_gbps_per_gpu": [0-9.]*' gpurun_out/varN_$v.log)"
done
