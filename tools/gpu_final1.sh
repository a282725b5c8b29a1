#!/bin/bash
# One-GPU end-of-round check, as the driver runs it: the GPU suite, smoke(),
# the N=1 bench pair, and the config-4 line (N=1).
set -u
OUT=gpurun_out/final1
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -rs > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/ref_n1.log 2>&1; echo "ref rc=$?"
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/n1_bert.log 2>&1; echo "ours rc=$?"; tail -1 $OUT/n1_bert.log | cut -c1-300
timeout 600 python bench.py --workload gpt2 --blend 1 --e2e-seam 0 > $OUT/n1_gpt2_blend.log 2>&1; echo "blend rc=$?"
for f in $OUT/*.log; do grep -h '^{' $f > ${f%.log}.jsonl 2>/dev/null || rm -f ${f%.log}.jsonl; done
exit 0
