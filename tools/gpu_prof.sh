#!/bin/bash
# ncu evidence for the N=1 kernel (single process; never a multi-rank command),
# one ncu per call:  tools/gpu_prof.sh <tag> full|launches
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
TAG=${1:-r01}
MODE=${2:-full}
if [ "$MODE" = full ]; then
  python tools/profile_n1.py bert 8 f64 > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ring_ -s 2 -c 1 \
      -o gpurun_out/prof_${TAG}_n1_bert_c8 -f python tools/profile_n1.py bert 8 f64 > gpurun_out/prof_ncu.log 2>&1
  echo "ncu full rc=$?"
else
  python bench.py --steps 3 --warmup 3 --nccl 0 > gpurun_out/launch_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_n1.csv \
      python bench.py --steps 3 --warmup 3 --nccl 0 > gpurun_out/launch_ncu.log 2>&1
  echo "ncu launches rc=$?"
fi
