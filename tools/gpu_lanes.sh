#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29522"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for el in 4 16 32; do
  timeout 300 python bench.py --steps 20 --e2e-lanes $el > gpurun_out/e2e1_$el.log 2>&1; echo "N1 e2e lanes=$el rc=$? $(grep -o '"e2e": {[^}]*}' gpurun_out/e2e1_$el.log | cut -c1-80)"
  timeout 300 $TR bench.py --gpus $NG --steps 20 --nccl 0 --e2e-lanes $el > gpurun_out/e2eN_$el.log 2>&1; echo "N$NG e2e lanes=$el rc=$? $(grep -o '"e2e": {[^}]*}' gpurun_out/e2eN_$el.log | cut -c1-80)"
done
