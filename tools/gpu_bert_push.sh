#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29519"
for rep in 1 2; do
timeout 300 $TR bench.py --gpus $NG --nccl 0 > gpurun_out/bert_push_$rep.log 2>&1; echo "bert rc=$? $(grep -o '"bus_gbps_per_gpu": [0-9.]*' gpurun_out/bert_push_$rep.log) $(grep -o '"phases_us": {[^}]*}' gpurun_out/bert_push_$rep.log) $(grep -o '"avg_kernel_ms": [0-9.]*' gpurun_out/bert_push_$rep.log) $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bert_push_$rep.log| head -1)"
done
timeout 600 $TR tools/sweep.py --shards 104,105,128 --rings 4 > gpurun_out/sweep_bertlike.log 2>&1; echo "sweep rc=$?"; grep '^{' gpurun_out/sweep_bertlike.log | python3 -c "
import sys,json
for l in sys.stdin:
  r=json.loads(l); print(r['shard_mib'], r['rings'], 'push', r['push']['bus_gbps'], r['push']['phases_us'], 'pull', r['pull']['bus_gbps'])"
