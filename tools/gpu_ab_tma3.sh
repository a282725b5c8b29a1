#!/bin/bash
# Round 2, third TMA layout A/B for the plain co-resident kernel: small
# tiles in 3-4 stages (the layout that won for the fused-blend kernel) vs
# the 2 x 64 KB default; parity first, then alternating timings.
set -u
OUT=gpurun_out/ab_tma3
mkdir -p $OUT
LIB=paper_2401_01728_b200/libravnest_b200.so
for v in p3x24 p4x24 p3x32; do
  cp tools/_ab/$v.so $LIB
  timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "bitwise or misaligned or wider or lanes" > $OUT/pytest_$v.log 2>&1
  echo "$v pytest rc=$? $(tail -1 $OUT/pytest_$v.log)"
done
B="--steps 30 --warmup 5 --e2e-seam 0 --cpu-port-params 100000 --cpu-sample-params 100000"
for rep in 1 2 3; do for v in p2x64 p3x24 p4x24 p3x32; do
  cp tools/_ab/$v.so $LIB
  for wl in bert resnet50; do
    timeout 300 python bench.py --workload $wl $B 2>>$OUT/err.log | grep '^{' > $OUT/cur.json
    python -c "import json; d=json.load(open('$OUT/cur.json')); print('$v', '$wl', d['avg_kernel_ms'], d['roofline']['frac'])" | tee -a $OUT/ab.txt
  done
done; done
cp tools/_ab/p2x64.so $LIB
