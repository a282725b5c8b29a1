#!/bin/bash
# BASELINE configs 4 (GPT-2 + tau=4 blend) and 5 (sweep) at the box's GPU count
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29513"
timeout 300 python bench.py --workload gpt2 --blend 1 --steps 10 --warmup 3 > gpurun_out/cfg4_n1.log 2>&1; echo "cfg4 n1 rc=$?"; grep '^{' gpurun_out/cfg4_n1.log | cut -c1-400
for proto in pull push; do
timeout 300 $TR bench.py --gpus $NG --workload gpt2 --blend 1 --steps 20 --warmup 3 --protocol $proto --nccl 1 > gpurun_out/cfg4_n${NG}_$proto.log 2>&1; echo "cfg4 n$NG $proto rc=$?"; grep '^{' gpurun_out/cfg4_n${NG}_$proto.log | cut -c1-600
done
timeout 900 $TR tools/sweep.py --out gpurun_out/sweep_n$NG.jsonl > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/sweep_n$NG.jsonl
