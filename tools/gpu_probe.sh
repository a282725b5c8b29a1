#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
timeout 300 ./tools/nvlink_probe > gpurun_out/probe.log 2>&1; echo "probe rc=$?"; cat gpurun_out/probe.log
timeout 600 python -m pytest tests/test_dist_gpu.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo "dist rc=$?"; tail -3 gpurun_out/pytest_dist.log
NG=$(nvidia-smi -L | wc -l)
for proto in pull push; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29512 \
     bench.py --gpus $NG --steps 30 --warmup 5 --protocol $proto --workload resnet50 --nccl 0 > gpurun_out/b_${proto}_resnet50.log 2>&1
  echo "$proto resnet50 rc=$? $(grep -o '"bus_gbps_per_gpu": [0-9.]*' gpurun_out/b_${proto}_resnet50.log)"
done
