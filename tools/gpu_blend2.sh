#!/bin/bash
# Fused push blend (split into delta + add halves): parity first, then config 4
# (GPT-2, tau=4) at the box's GPU count: cycle alone, fused, separate blend.
set -u
OUT=gpurun_out/blend2
mkdir -p $OUT
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
timeout 1200 python -m pytest tests/test_loopback_gpu.py tests/test_fullsize_gpu.py tests/test_dist_gpu.py -m gpu -q \
  -k "blend or config4 or dist or averager" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
for rep in 1 2; do
for cfg in "0 1" "1 1" "1 0"; do
  set -- $cfg
  timeout 600 python bench.py --gpus $NG --workload gpt2 --blend $1 --fused-blend $2 --steps 30 --nccl 0 --e2e-lanes 8 2>>$OUT/err.log | grep '^{' >> $OUT/gpt2_n${NG}.jsonl
  tail -1 $OUT/gpt2_n${NG}.jsonl | python -c "import json,sys; d=json.load(sys.stdin); print('gpt2 n=$NG blend=$1 fused=$2', d['ms_per_step'], d['ms_per_step_median'], d['avg_kernel_ms'], d.get('phases_us'))"
done; done
