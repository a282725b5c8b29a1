#!/bin/bash
# protocol / lane comparison at the box's GPU count, plus the dist parity test
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_dist_gpu.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo "dist rc=$?"; tail -3 gpurun_out/pytest_dist.log
for proto in pull push; do
 for lanes in 1 4; do
  for wl in bert resnet50; do
   timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29512 \
     bench.py --gpus $NG --steps 30 --warmup 5 --protocol $proto --lanes $lanes --workload $wl --nccl 0 > gpurun_out/b_${proto}_${lanes}_${wl}.log 2>&1
   echo "$proto lanes=$lanes $wl rc=$? $(grep -o '"bus_gbps_per_gpu": [0-9.]*' gpurun_out/b_${proto}_${lanes}_${wl}.log) $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/b_${proto}_${lanes}_${wl}.log | head -1)"
  done
 done
done
