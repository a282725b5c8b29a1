#!/bin/bash
# Round 2, second TMA layout A/B: plain kernel 2x64 (in bl3x48.so, the library)
# vs 3x48 / 3x40; fused-blend kernel 3x48 vs 4x40 / 4x32.  Parity of every
# candidate first (co-resident tests), then alternating timings.
set -u
OUT=gpurun_out/ab_tma2
mkdir -p $OUT
LIB=paper_2401_01728_b200/libravnest_b200.so
for v in p3x48 p3x40 bl4x40 bl4x32; do
  cp tools/_ab/$v.so $LIB
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_gpu.py -m gpu -q \
    -k "bitwise or misaligned or wider or lanes or blend_in_cycle_co_resident or co_resident" > $OUT/pytest_$v.log 2>&1
  echo "$v pytest rc=$? $(tail -1 $OUT/pytest_$v.log)"
done
B="--steps 30 --warmup 5 --e2e-seam 0 --cpu-port-params 100000 --cpu-sample-params 100000"
for rep in 1 2 3; do
  for v in bl3x48 p3x48 p3x40; do
    cp tools/_ab/$v.so $LIB
    for wl in bert resnet50; do
      timeout 300 python bench.py --workload $wl $B 2>>$OUT/err.log | grep '^{' > $OUT/cur.json
      python -c "import json; d=json.load(open('$OUT/cur.json')); print('plain', '$v', '$wl', d['avg_kernel_ms'], d['roofline']['frac'])" | tee -a $OUT/ab.txt
    done
  done
  for v in bl3x48 bl4x40 bl4x32; do
    cp tools/_ab/$v.so $LIB
    timeout 300 python bench.py --workload gpt2 --blend 1 $B 2>>$OUT/err.log | grep '^{' > $OUT/cur.json
    python -c "import json; d=json.load(open('$OUT/cur.json')); print('blend', '$v', 'gpt2', d['avg_kernel_ms'], d['roofline']['frac'])" | tee -a $OUT/ab.txt
  done
done
cp tools/_ab/bl3x48.so $LIB
