#!/bin/bash
# Last one-GPU session: the N=1 bench pair as the driver runs it, the launch
# list of the same command, and ncu --set full of the co-resident kernel.
set -u
OUT=gpurun_out/final_n1
mkdir -p $OUT
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/ref_n1.log 2>&1; echo "ref rc=$?"
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/n1_bert.log 2>&1; echo "ours rc=$?"; tail -1 $OUT/n1_bert.log | cut -c1-400
timeout 600 python bench.py --workload gpt2 --e2e-seam 0 > $OUT/n1_gpt2.log 2>&1; echo "gpt2 rc=$?"
timeout 600 python bench.py --workload resnet50 --e2e-seam 0 > $OUT/n1_resnet50.log 2>&1; echo "resnet rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --e2e-seam 0 --cpu-sample-params 100000 --cpu-port-params 100000 > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/profile_n1.py bert 8 f64 > $OUT/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ring_ -s 2 -c 1 \
    -o $OUT/prof_r02_n1_bert_c8_c128 -f python tools/profile_n1.py bert 8 f64 > $OUT/prof_ncu.log 2>&1; echo "ncu full rc=$?"
for f in $OUT/*.log; do grep -h '^{' $f > ${f%.log}.jsonl 2>/dev/null || rm -f ${f%.log}.jsonl; done
exit 0
