#!/bin/bash
# 8 ranks over the box's GPUs: GPT-2 medium plain and config 4 (fused blend).
set -u
OUT=gpurun_out/emulate2
mkdir -p $OUT
export RAVNEST_B200_TIMEOUT_S=20
export CUDA_DEVICE_MAX_CONNECTIONS=32
NG=$(nvidia-smi -L | wc -l)
for r in $NG 8; do for b in 0 1; do
  timeout 900 python tools/emulate_ranks.py --ranks $r --workload gpt2 --blend $b --check $((1 - b)) --steps 20 2>>$OUT/err.log | tee -a $OUT/emulate_gpt2.jsonl
done; done
