#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29527"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 $TR tools/latency.py 2>&1 | grep "^{"
timeout 900 $TR tools/sweep.py --shards 1,4,16 --rings 1,2,4 --out gpurun_out/sweep_ll_n$NG.jsonl > gpurun_out/sweep_ll.log 2>&1; echo "sweep rc=$?"
