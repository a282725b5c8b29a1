#!/bin/bash
# Fused push blend variants (tools/_ab/*.so): parity of NEW, then config 4
# (GPT-2, tau=4) at the box's GPU count, alternating VARIANTS.
# Round 2: split (first half in the scatter item) vs onepass; then cpasync
# (operands streamed through shared memory with cp.async) vs split vs onepass.
set -u
OUT=gpurun_out/blend3
mkdir -p $OUT
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
LIB=paper_2401_01728_b200/libravnest_b200.so
cp tools/_ab/${NEW:-split}.so $LIB
timeout 1500 python -m pytest tests/test_loopback_gpu.py tests/test_fullsize_gpu.py tests/test_dist_gpu.py tests/test_averager_gpu.py -m gpu -q \
  -k "blend or config4 or dist or averager" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
for rep in 1 2 3; do for v in ${VARIANTS:-split onepass}; do
  cp tools/_ab/$v.so $LIB
  timeout 600 python bench.py --gpus $NG --workload gpt2 --blend 1 --steps 30 --nccl 0 --e2e-lanes 8 2>>$OUT/err.log | grep '^{' > $OUT/cur.json
  python -c "import json; d=json.load(open('$OUT/cur.json')); print('$v n=$NG', d['ms_per_step'], d['ms_per_step_median'], d.get('phases_us'))" | tee -a $OUT/ab.txt
done; done
cp tools/_ab/${NEW:-split}.so $LIB
