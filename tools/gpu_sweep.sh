#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
export CUDA_DEVICE_MAX_CONNECTIONS=32
NG=$(nvidia-smi -L | wc -l)
for n in $NG 2; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n tools/sweep.py --out gpurun_out/sweep_r02_n$n.jsonl > gpurun_out/sweep_n$n.log 2>&1; echo "sweep n=$n rc=$? $(wc -l < gpurun_out/sweep_r02_n$n.jsonl)"
done
