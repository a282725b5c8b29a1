#!/bin/bash
# e2e (host fp32 buffers through rv_allreduce_mean_host) at N=1 vs pipeline
# lanes, after co-resident lanes got the whole grid; alternating, 2 reps.
set -u
OUT=gpurun_out/e2e_lanes
mkdir -p $OUT
for rep in 1 2; do for l in 8 16 32 64; do
  timeout 300 python bench.py --steps 10 --e2e-lanes $l --e2e-seam 0 --cpu-port-params 100000 --cpu-sample-params 100000 \
    2>>$OUT/err.log | grep '^{' > $OUT/cur.json
  python -c "import json; d=json.load(open('$OUT/cur.json')); print('lanes', $l, d['e2e']['ms_per_step'], d['e2e']['value'])" | tee -a $OUT/e2e_lanes.txt
done; done
