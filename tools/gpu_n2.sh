#!/bin/bash
# 2-GPU session: the driver's plain `bench.py --gpus 2` (self-spawned ranks) and
# its reference arm; config 4 (GPT-2, tau=4 blend) fused / lag sweep / separate /
# cycle alone with device phase traces; ResNet-50 lanes; the numpy drop-in probe.
set -u
OUT=gpurun_out/n2
mkdir -p $OUT
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
timeout 900 python bench.py --impl reference --gpus $NG --steps 20 --warmup 5 > $OUT/ref.out 2> $OUT/ref.err; echo "ref rc=$?"; tail -1 $OUT/ref.out | cut -c1-400
timeout 900 python bench.py --gpus $NG --steps 20 --warmup 5 > $OUT/ours.out 2> $OUT/ours.err; echo "ours rc=$?"; tail -1 $OUT/ours.out
for cfg in "0 1 -1" "1 1 -1" "1 1 0" "1 1 148" "1 1 592" "1 0 -1"; do
  set -- $cfg
  timeout 600 python bench.py --gpus $NG --workload gpt2 --blend $1 --fused-blend $2 --blend-lag $3 --steps 30 --nccl 0 --e2e-lanes 8 2>>$OUT/err.log | grep '^{' > $OUT/gpt2_b$1_f$2_l$3.jsonl
  python -c "import json; d=json.load(open('$OUT/gpt2_b$1_f$2_l$3.jsonl')); print('gpt2 blend=$1 fused=$2 lag=$3', d['ms_per_step'], d['ms_per_step_median'], d['avg_kernel_ms'], d.get('phases_us'))"
done
for l in 1 8; do
  timeout 600 python bench.py --gpus $NG --workload resnet50 --lanes $l --steps 50 --nccl 0 2>>$OUT/err.log | grep '^{' > $OUT/resnet_l$l.jsonl
  python -c "import json; d=json.load(open('$OUT/resnet_l$l.jsonl')); print('resnet lanes=$l', d['bus_gbps_per_gpu'], d['ms_per_step_median'], d.get('phases_us'))"
done
timeout 600 python tools/e2e_seam_probe.py > $OUT/e2e_seam_probe.txt 2>&1; cat $OUT/e2e_seam_probe.txt
