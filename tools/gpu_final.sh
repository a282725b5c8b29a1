#!/bin/bash
# consolidated end-of-round measurements (profiles/r01/final/*.jsonl; tools/summarize_final.py builds SUMMARY.md)
set -u
mkdir -p gpurun_out/final
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python bench.py > gpurun_out/final/n1_bert.log 2>&1; echo "n1 bert rc=$?"
timeout 300 python bench.py --workload resnet50 > gpurun_out/final/n1_resnet50.log 2>&1; echo "n1 resnet rc=$?"
timeout 300 python bench.py --workload gpt2 > gpurun_out/final/n1_gpt2.log 2>&1; echo "n1 gpt2 rc=$?"
timeout 300 python bench.py --workload gpt2 --blend 1 > gpurun_out/final/n1_gpt2_blend.log 2>&1; echo "n1 gpt2 blend rc=$?"
timeout 300 python bench.py --impl reference > gpurun_out/final/ref_n1.log 2>&1; echo "ref n1 rc=$?"
for n in 2 $NG; do
  timeout 300 $TR --nproc-per-node $n --master-port 2953$n bench.py --gpus $n > gpurun_out/final/n${n}_bert.log 2>&1; echo "n$n bert rc=$?"
  timeout 300 $TR --nproc-per-node $n --master-port 2953$n bench.py --gpus $n --lanes 4 > gpurun_out/final/n${n}_bert_lanes4.log 2>&1; echo "n$n bert lanes4 rc=$?"
  timeout 300 $TR --nproc-per-node $n --master-port 2953$n bench.py --gpus $n --workload resnet50 > gpurun_out/final/n${n}_resnet50.log 2>&1; echo "n$n resnet rc=$?"
  timeout 300 $TR --nproc-per-node $n --master-port 2953$n bench.py --gpus $n --workload gpt2 > gpurun_out/final/n${n}_gpt2.log 2>&1; echo "n$n gpt2 rc=$?"
  timeout 300 $TR --nproc-per-node $n --master-port 2953$n bench.py --gpus $n --workload gpt2 --blend 1 --nccl 0 > gpurun_out/final/n${n}_gpt2_blend.log 2>&1; echo "n$n gpt2 blend rc=$?"
  timeout 300 $TR --nproc-per-node $n --master-port 2953$n bench.py --impl reference --gpus $n > gpurun_out/final/ref_n$n.log 2>&1; echo "ref n$n rc=$?"
done
for f in gpurun_out/final/*.log; do grep -h '^{' $f > ${f%.log}.jsonl 2>/dev/null; done
