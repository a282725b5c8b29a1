#!/bin/bash
# After the cp.async blend passes: config 4 (GPT-2, tau=4) at the box's GPU
# count -- fused vs cycle alone vs separate blend -- and the 8-rank emulation.
set -u
OUT=gpurun_out/n4blend
mkdir -p $OUT
export RAVNEST_B200_TIMEOUT_S=20
export CUDA_DEVICE_MAX_CONNECTIONS=32
NG=$(nvidia-smi -L | wc -l)
for rep in 1 2; do for cfg in "1 1" "0 1" "1 0"; do
  set -- $cfg
  timeout 600 python bench.py --gpus $NG --workload gpt2 --blend $1 --fused-blend $2 --steps 30 --nccl 0 --e2e-lanes 8 2>>$OUT/err.log | grep '^{' >> $OUT/gpt2_n${NG}.jsonl
  tail -1 $OUT/gpt2_n${NG}.jsonl | python -c "import json,sys; d=json.load(sys.stdin); print('gpt2 n=$NG blend=$1 fused=$2', d['ms_per_step'], d['ms_per_step_median'], d.get('phases_us'))"
done; done
timeout 900 python tools/emulate_ranks.py --ranks 8 --workload gpt2 --blend 1 --check 0 --steps 20 2>>$OUT/err.log | tee -a $OUT/emulate_gpt2_blend.jsonl
