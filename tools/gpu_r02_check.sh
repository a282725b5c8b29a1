#!/bin/bash
# Regression + evidence session: the full GPU suite, lanes > rings at N GPUs
# after the lane-grid fix, and one ncu --set full of the N=1 kernel.
set -u
OUT=gpurun_out/r02check
mkdir -p $OUT
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests -m gpu -q -rs > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
for wl in resnet50 bert; do for l in 1 4 8; do
  timeout 600 python bench.py --gpus $NG --workload $wl --lanes $l --steps 30 --nccl 0 2>>$OUT/err.log | grep '^{' >> $OUT/lanes_n${NG}.jsonl
  tail -1 $OUT/lanes_n${NG}.jsonl | python -c "import json,sys; d=json.load(sys.stdin); print('$wl lanes=$l', d['bus_gbps_per_gpu'], d['bus_gbps_per_gpu_median'], d.get('phases_us'))"
done; done
python tools/profile_n1.py bert 8 f64 > $OUT/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ring_ -s 2 -c 1 \
    -o $OUT/prof_r02_n1_bert_c8 -f python tools/profile_n1.py bert 8 f64 > $OUT/prof_ncu.log 2>&1
echo "ncu full rc=$?"
