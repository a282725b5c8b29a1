#!/bin/bash
# TMA kernels: consumer warps per CTA (RV_TMA_CONSUMERS builds) -- 256 (the
# library) vs 128 / 384 / 512; parity first, then alternating timings.
set -u
OUT=gpurun_out/ab_consumers
mkdir -p $OUT
LIB=paper_2401_01728_b200/libravnest_b200.so
for v in c128 c384 c512; do
  cp tools/_ab/$v.so $LIB
  timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "bitwise or misaligned or wider or lanes or blend_in_cycle" > $OUT/pytest_$v.log 2>&1
  echo "$v pytest rc=$? $(tail -1 $OUT/pytest_$v.log)"
done
B="--steps 30 --warmup 5 --e2e-seam 0 --cpu-port-params 100000 --cpu-sample-params 100000"
for rep in 1 2 3; do for v in c256 c128 c384 c512; do
  cp tools/_ab/$v.so $LIB
  for wl in bert resnet50; do
    timeout 300 python bench.py --workload $wl $B 2>>$OUT/err.log | grep '^{' > $OUT/cur.json
    python -c "import json; d=json.load(open('$OUT/cur.json')); print('$v', '$wl', d['avg_kernel_ms'], d['roofline']['frac'])" | tee -a $OUT/ab.txt
  done
  timeout 300 python bench.py --workload gpt2 --blend 1 $B 2>>$OUT/err.log | grep '^{' > $OUT/cur.json
  python -c "import json; d=json.load(open('$OUT/cur.json')); print('$v', 'gpt2-blend', d['avg_kernel_ms'], d['roofline']['frac'])" | tee -a $OUT/ab.txt
done; done
cp tools/_ab/c256.so $LIB
