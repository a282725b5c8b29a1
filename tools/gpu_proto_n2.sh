#!/bin/bash
# Transport crossover at 2 GPUs: the round-2 sweep shows pull ahead of push up
# to ~128 MiB per cluster at C = 2 (32 MiB at C = 4); check on the named
# workloads, alternating.
set -u
OUT=gpurun_out/proto_n2
mkdir -p $OUT
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
for rep in 1 2; do for wl in resnet50 bert; do for pr in pull push; do
  timeout 600 python bench.py --gpus $NG --workload $wl --protocol $pr --steps 50 --nccl 0 --trace 0 2>>$OUT/err.log | grep '^{' > $OUT/cur.json
  python -c "import json; d=json.load(open('$OUT/cur.json')); print('$wl', '$pr', d['bus_gbps_per_gpu'], d['bus_gbps_per_gpu_median'], d['ms_per_step_median'])" | tee -a $OUT/proto.txt
done; done; done
