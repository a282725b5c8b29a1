#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29520"
timeout 300 $TR bench.py --gpus $NG > gpurun_out/bench_n$NG.log 2>&1; echo "bench rc=$?"; grep -o '"bus_gbps_per_gpu": [0-9.]*, "higher\|"nccl_compare": {.*}}' gpurun_out/bench_n$NG.log | head -3
timeout 900 $TR tools/sweep.py --out gpurun_out/sweep_r01d_n$NG.jsonl > gpurun_out/sweep.log 2>&1; echo "sweep rc=$? $(wc -l < gpurun_out/sweep_r01d_n$NG.jsonl)"
