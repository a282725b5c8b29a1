#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29521"
for it in 2 4 8 16 32; do
  for wl in bert gpt2 resnet50; do
    RAVNEST_B200_PUSH_ITEMS=$it timeout 300 $TR bench.py --gpus $NG --nccl 0 --trace 1 --workload $wl --protocol push > gpurun_out/items_${it}_$wl.log 2>&1
    echo "items=$it $wl rc=$? $(grep -o '"bus_gbps_per_gpu": [0-9.]*' gpurun_out/items_${it}_$wl.log) $(grep -o '"phases_us": {[^}]*}' gpurun_out/items_${it}_$wl.log)"
  done
done
