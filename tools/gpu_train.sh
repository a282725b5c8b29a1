#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench_n1.log 2>&1; echo "N1 rc=$? $(grep -o '"frac": [0-9.]*' gpurun_out/bench_n1.log) $(grep -o '"e2e": {[^}]*}' gpurun_out/bench_n1.log)"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $NG > gpurun_out/bench_n$NG.log 2>&1; echo "N$NG rc=$? $(grep -o '"bus_gbps_per_gpu": [0-9.]*' gpurun_out/bench_n$NG.log) $(grep -o '"e2e": {[^}]*}' gpurun_out/bench_n$NG.log)"
for g in 0 1; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29518 examples/train_async.py --graph $g > gpurun_out/train_async_g$g.log 2>&1; echo "train graph=$g rc=$?"; grep '^{' gpurun_out/train_async_g$g.log
done
