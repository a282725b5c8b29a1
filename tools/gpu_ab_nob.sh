#!/bin/bash
# Fused-blend TMA kernel: 2 (library) vs 3 output buffers at CB >= 8
# (RV_TMA_BL_NOB3 build), config 4 at N=1, alternating; parity first.
set -u
OUT=gpurun_out/ab_nob
mkdir -p $OUT
LIB=paper_2401_01728_b200/libravnest_b200.so
cp tools/_ab/nob3.so $LIB
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_gpu.py -m gpu -q -k "blend or co_resident or wider" > $OUT/pytest_nob3.log 2>&1
echo "nob3 pytest rc=$? $(tail -1 $OUT/pytest_nob3.log)"
B="--steps 30 --warmup 5 --e2e-seam 0 --cpu-port-params 100000 --cpu-sample-params 100000"
for rep in 1 2 3; do for v in nob2 nob3; do
  cp tools/_ab/$v.so $LIB
  for wl in gpt2 bert; do
    timeout 300 python bench.py --workload $wl --blend 1 $B 2>>$OUT/err.log | grep '^{' > $OUT/cur.json
    python -c "import json; d=json.load(open('$OUT/cur.json')); print('$v', '$wl', d['avg_kernel_ms'], d['roofline']['frac'])" | tee -a $OUT/ab.txt
  done
done; done
cp tools/_ab/nob2.so $LIB
