#!/bin/bash
# (Round 2, not kept: no change.) LL fold: peek at every member's word pair at once (llpeek) vs one polled
# load per member in turn (llseq): LL parity tests, then the small-shard
# sweep points at the box's GPU count, alternating.
set -u
OUT=gpurun_out/ll_ab
mkdir -p $OUT
export RAVNEST_B200_TIMEOUT_S=10
export CUDA_DEVICE_MAX_CONNECTIONS=32
NG=$(nvidia-smi -L | wc -l)
LIB=paper_2401_01728_b200/libravnest_b200.so
cp tools/_ab/llpeek.so $LIB
timeout 900 python -m pytest tests/test_loopback_gpu.py -m gpu -q -k "ll" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
for rep in 1 2; do for v in llpeek llseq; do
  cp tools/_ab/$v.so $LIB
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2961$rep \
    tools/sweep.py --shards 1,4 --rings 1,2,4 --out $OUT/sweep_${v}_$rep.jsonl > $OUT/sweep_${v}_$rep.log 2>&1
  python - <<PY
import json
for ln in open("$OUT/sweep_${v}_$rep.jsonl"):
    d = json.loads(ln)
    ll = d.get("ll")
    if ll: print("$v", d["shard_mib"], d["rings"], "ll ms", ll["ms"], "graph ms", ll["graph_ms"], "nccl ms", d["nccl"]["ms"])
PY
done; done
cp tools/_ab/llpeek.so $LIB
