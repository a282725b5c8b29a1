# verification after the last kernel edits: full GPU suite, smoke, and spot benches
export RAVNEST_B200_TIMEOUT_S=10
mkdir -p gpurun_out/verify
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/verify/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/verify/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
timeout 300 python bench.py > gpurun_out/verify/n1_bert.jsonl 2>/dev/null; echo "n1 rc=$?"
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 $TR --nproc-per-node 4 --master-port 29680 bench.py --gpus 4 > gpurun_out/verify/n4_bert.jsonl 2>/dev/null; echo "n4 bert rc=$?"
timeout 300 $TR --nproc-per-node 4 --master-port 29681 bench.py --gpus 4 --workload gpt2 --blend 1 --nccl 0 > gpurun_out/verify/n4_gpt2_blend.jsonl 2>/dev/null; echo "n4 blend rc=$?"
for f in gpurun_out/verify/*.jsonl; do python -c "
import json,sys
l=[x for x in open('$f') if x.startswith('{')][-1]; d=json.loads(l)
print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
