#!/bin/bash
# A/B of TMA co-resident kernel layouts (tools/build_ab.sh variants), N=1 BERT
# C=8, alternating, 3 repetitions; plus the fp32 fold on the default layout.
set -u
OUT=gpurun_out/ab_tma
mkdir -p $OUT
LIB=paper_2401_01728_b200/libravnest_b200.so
cp $LIB tools/_ab/product.so
for rep in 1 2 3; do
  for v in s2x64 s3x64 s4x48 contig; do  # contig: a since-removed RV_TMA_CONTIG build (one contiguous tile run per block)
    cp tools/_ab/$v.so $LIB
    for wl in bert resnet50; do
      timeout 300 python bench.py --workload $wl --steps 40 --warmup 5 --e2e-seam 0 --cpu-port-params 100000 \
        --cpu-sample-params 100000 2>>$OUT/err.log | grep '^{' > $OUT/cur.json
      python -c "import json; d=json.load(open('$OUT/cur.json')); print('$v', '$wl', d['avg_kernel_ms'], d['ms_per_step_median'], d['roofline']['frac'])" | tee -a $OUT/ab.txt
    done
  done
  cp tools/_ab/s2x64.so $LIB
  timeout 300 python bench.py --acc native --steps 40 --warmup 5 --e2e-seam 0 --cpu-port-params 100000 \
    --cpu-sample-params 100000 2>>$OUT/err.log | grep '^{' > $OUT/cur.json
  python -c "import json; d=json.load(open('$OUT/cur.json')); print('s2x64-native', 'bert', d['avg_kernel_ms'], d['ms_per_step_median'], d['roofline']['frac'])" | tee -a $OUT/ab.txt
done
cp tools/_ab/product.so $LIB
