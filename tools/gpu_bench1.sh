#!/bin/bash
# The driver's N=1 pair: the reference arm, then ours (default flags), then the
# same command under ncu (launch list, gpu__time_duration per launch).
set -u
OUT=gpurun_out/bench1
mkdir -p $OUT
export RAVNEST_B200_TIMEOUT_S=10
T0=$(date +%s); timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/ref.out 2> $OUT/ref.err; echo "ref rc=$?"
echo "ref wall $(( $(date +%s) - T0 )) s"; tail -1 $OUT/ref.out | cut -c1-900; tail -3 $OUT/ref.err
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/ours.out 2> $OUT/ours.err; echo "ours rc=$?"
tail -1 $OUT/ours.out; tail -3 $OUT/ours.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --e2e-seam 0 --cpu-sample-params 100000 --cpu-port-params 100000 > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
