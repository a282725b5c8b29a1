#!/bin/bash
# consolidated end-of-round measurements (profiles/<round>/final/*.jsonl;
# tools/summarize_final.py builds SUMMARY.md).  N > 1 lines use bench.py's own
# rank spawning (the driver's plain command); the reference arm runs the
# unmodified ravnest.multiring.apply_ring_mean on the full workload.
set -u
OUT=gpurun_out/final
mkdir -p $OUT
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests -m gpu -q -rs > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $OUT/n1_bert.log 2>&1; echo "n1 bert rc=$?"
timeout 600 python bench.py --workload resnet50 > $OUT/n1_resnet50.log 2>&1; echo "n1 resnet rc=$?"
timeout 600 python bench.py --workload gpt2 --e2e-seam 0 > $OUT/n1_gpt2.log 2>&1; echo "n1 gpt2 rc=$?"
timeout 600 python bench.py --workload gpt2 --blend 1 --e2e-seam 0 > $OUT/n1_gpt2_blend.log 2>&1; echo "n1 gpt2 blend rc=$?"
timeout 900 python bench.py --impl reference > $OUT/ref_n1.log 2>&1; echo "ref n1 rc=$?"
for n in 2 $NG; do
  [ $n -gt $NG ] && continue
  timeout 600 python bench.py --gpus $n > $OUT/n${n}_bert.log 2>&1; echo "n$n bert rc=$?"
  timeout 600 python bench.py --gpus $n --lanes 4 > $OUT/n${n}_bert_lanes4.log 2>&1; echo "n$n bert lanes4 rc=$?"
  timeout 600 python bench.py --gpus $n --min-cb 8 --nccl 0 > $OUT/n${n}_bert_cb8.log 2>&1; echo "n$n bert cb8 rc=$?"
  timeout 600 python bench.py --gpus $n --workload resnet50 > $OUT/n${n}_resnet50.log 2>&1; echo "n$n resnet rc=$?"
  timeout 600 python bench.py --gpus $n --workload gpt2 > $OUT/n${n}_gpt2.log 2>&1; echo "n$n gpt2 rc=$?"
  timeout 600 python bench.py --gpus $n --workload gpt2 --blend 1 --nccl 0 > $OUT/n${n}_gpt2_blend.log 2>&1; echo "n$n gpt2 blend rc=$?"
  timeout 900 python bench.py --impl reference --gpus $n > $OUT/ref_n$n.log 2>&1; echo "ref n$n rc=$?"
  [ $n -eq $NG ] && break
done
for f in $OUT/*.log; do grep -h '^{' $f > ${f%.log}.jsonl 2>/dev/null; done
