#!/bin/bash
# Fused-blend TMA kernel consumer count: 256 (library) vs 192 / 320.
set -u
OUT=gpurun_out/ab_bl_consumers
mkdir -p $OUT
LIB=paper_2401_01728_b200/libravnest_b200.so
for v in bl192 bl320; do
  cp tools/_ab/$v.so $LIB
  timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "blend_in_cycle" > $OUT/pytest_$v.log 2>&1
  echo "$v pytest rc=$? $(tail -1 $OUT/pytest_$v.log)"
done
B="--steps 20 --warmup 5 --e2e-seam 0 --cpu-port-params 100000 --cpu-sample-params 100000"
for rep in 1 2 3; do for v in bl256 bl192 bl320; do
  cp tools/_ab/$v.so $LIB
  for wl in gpt2 bert; do
    timeout 300 python bench.py --workload $wl --blend 1 $B 2>>$OUT/err.log | grep '^{' > $OUT/cur.json
    python -c "import json; d=json.load(open('$OUT/cur.json')); print('$v', '$wl', d['avg_kernel_ms'], d['roofline']['frac'])" | tee -a $OUT/ab.txt
  done
done; done
cp tools/_ab/bl256.so $LIB
