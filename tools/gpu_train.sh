#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29517"
timeout 900 python -m pytest tests/test_dist_gpu.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo "dist rc=$?"; tail -2 gpurun_out/pytest_dist.log
for mb in 32 64 128 0; do
  timeout 300 $TR bench.py --gpus $NG --nccl 0 --max-blocks $mb > gpurun_out/bench_mb$mb.log 2>&1; echo "N$NG max_blocks=$mb rc=$? $(grep -o '"bus_gbps_per_gpu": [0-9.]*' gpurun_out/bench_mb$mb.log)"
done
timeout 900 $TR examples/train_async.py > gpurun_out/train_async.log 2>&1; echo "train rc=$?"; grep '^{' gpurun_out/train_async.log
