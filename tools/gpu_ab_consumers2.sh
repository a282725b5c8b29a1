#!/bin/bash
# Plain TMA kernel consumer count, second A/B: 128 (the library now) vs 64 /
# 96 / 192; the library's parity suite first (all co-resident / TMA tests).
set -u
OUT=gpurun_out/ab_consumers2
mkdir -p $OUT
LIB=paper_2401_01728_b200/libravnest_b200.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_gpu.py tests/test_averager_gpu.py -m gpu -q > $OUT/pytest_lib.log 2>&1
echo "library pytest rc=$? $(tail -1 $OUT/pytest_lib.log)"
for v in c64 c96 c192; do
  cp tools/_ab/$v.so $LIB
  timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "bitwise or misaligned or wider or lanes" > $OUT/pytest_$v.log 2>&1
  echo "$v pytest rc=$? $(tail -1 $OUT/pytest_$v.log)"
done
B="--steps 30 --warmup 5 --e2e-seam 0 --cpu-port-params 100000 --cpu-sample-params 100000"
for rep in 1 2 3; do for v in c128 c64 c96 c192; do
  cp tools/_ab/$v.so $LIB
  for wl in bert resnet50 gpt2; do
    timeout 300 python bench.py --workload $wl $B 2>>$OUT/err.log | grep '^{' > $OUT/cur.json
    python -c "import json; d=json.load(open('$OUT/cur.json')); print('$v', '$wl', d['avg_kernel_ms'], d['roofline']['frac'])" | tee -a $OUT/ab.txt
  done
done; done
cp tools/_ab/c128.so $LIB
