#!/bin/bash
# 8-GPU readiness at 4 GPUs: the CB = 8 push kernel (what an 8-rank job
# selects) against the CB = 4 default at equal bytes -- bench lines
# (alternating), then one ncu --set full of each on the last device of a
# single process driving the 4 GPUs (never a multi-rank command under ncu).
# Also ResNet-50 lanes 1/2/4/8 (mid-size headroom).
set -u
OUT=gpurun_out/cb8
mkdir -p $OUT
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
for rep in 1 2; do for cb in 0 8; do
  timeout 600 python bench.py --gpus $NG --steps 30 --warmup 5 --nccl 0 --min-cb $cb 2>$OUT/bench_err.log | grep '^{' >> $OUT/bench_bert_cb.jsonl
done; done
for rep in 1 2; do for l in 1 2 4 8; do
  timeout 600 python bench.py --gpus $NG --workload resnet50 --steps 50 --warmup 5 --nccl 0 --lanes $l 2>>$OUT/bench_err.log | grep '^{' >> $OUT/bench_resnet_lanes.jsonl
done; done
python - <<'PY'
import json
for f in ("bench_bert_cb", "bench_resnet_lanes"):
    for ln in open(f"gpurun_out/cb8/{f}.jsonl"):
        d = json.loads(ln)
        print(f, d["n_gpus"], d["config"].get("plan_options"), d["config"]["lanes"], d["bus_gbps_per_gpu"],
              d.get("bus_gbps_per_gpu_median"), d["avg_kernel_ms"], d["roofline"]["frac"], d.get("phases_us"))
PY
for cb in 8 0; do
  timeout 300 python tools/profile_p2p.py bert push --gpus $NG --min-cb $cb > $OUT/p2p_cb$cb.log 2>&1; tail -1 $OUT/p2p_cb$cb.log
done
L=$((NG - 1))
for cb in 8 0; do
  timeout 1200 ncu --devices $L --replay-mode application --set full --clock-control none --import-source on \
    -k regex:ring_push -s 3 -c 1 -o $OUT/prof_push_n${NG}_cb$cb -f \
    python tools/profile_p2p.py bert push --gpus $NG --min-cb $cb > $OUT/ncu_cb$cb.log 2>&1
  echo "ncu cb=$cb rc=$?"
done
