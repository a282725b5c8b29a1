#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29514"
timeout 600 python -m pytest tests/test_dist_gpu.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo "dist rc=$?"; tail -2 gpurun_out/pytest_dist.log
timeout 600 $TR tools/sweep.py --shards 1,4,16,128 --rings 1,4 --out gpurun_out/sweep_small_n$NG.jsonl > gpurun_out/sweep_small.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/sweep_small_n$NG.jsonl
for proto in pull push; do
timeout 300 $TR bench.py --gpus $NG --steps 30 --warmup 5 --protocol $proto --nccl 0 > gpurun_out/bert_n${NG}_$proto.log 2>&1; echo "bert $proto rc=$? $(grep -o '"bus_gbps_per_gpu": [0-9.]*' gpurun_out/bert_n${NG}_$proto.log)"
done
