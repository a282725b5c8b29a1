#!/bin/bash
# 8 ranks over the box's GPUs in one process (the CB = 8 kernels at C = 8 over
# real NVLink), against 1 rank per GPU; plus the spread-rank parity tests.
set -u
OUT=gpurun_out/emulate
mkdir -p $OUT
export RAVNEST_B200_TIMEOUT_S=20
export CUDA_DEVICE_MAX_CONNECTIONS=32
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_loopback_gpu.py -m gpu -q -k "spread" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
for r in $NG 8 16; do for proto in push pull; do
  timeout 600 python tools/emulate_ranks.py --ranks $r --proto $proto 2>>$OUT/err.log | tee -a $OUT/emulate.jsonl
done; done
