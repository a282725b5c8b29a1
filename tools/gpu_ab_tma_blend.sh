#!/bin/bash
# A/B of the co-resident fused-blend TMA kernel's stage layout (config 4 at
# N=1), alternating, 3 repetitions: blend parity first on the candidate builds.
set -u
OUT=gpurun_out/ab_tma_blend
mkdir -p $OUT
LIB=paper_2401_01728_b200/libravnest_b200.so
for v in bl2x72 bl3x48 bl3x40; do
  cp tools/_ab/$v.so $LIB
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_gpu.py -m gpu -q -k "blend_in_cycle_co_resident or co_resident" > $OUT/pytest_$v.log 2>&1
  echo "$v pytest rc=$? $(tail -1 $OUT/pytest_$v.log)"
done
for rep in 1 2 3; do for v in bl2x64 bl2x72 bl3x48 bl3x40; do
  cp tools/_ab/$v.so $LIB
  timeout 300 python bench.py --workload gpt2 --blend 1 --steps 20 --warmup 5 --e2e-seam 0 --cpu-port-params 100000 \
    --cpu-sample-params 100000 2>>$OUT/err.log | grep '^{' > $OUT/cur.json
  python -c "import json; d=json.load(open('$OUT/cur.json')); print('$v', d['avg_kernel_ms'], d['ms_per_step_median'], d['roofline']['frac'])" | tee -a $OUT/ab.txt
done; done
cp tools/_ab/bl2x64.so $LIB
