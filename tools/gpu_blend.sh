# fused delayed-update blend: parity, then config 4 (GPT-2, tau=4) fused vs separate launches
export RAVNEST_B200_TIMEOUT_S=10
timeout 900 python -m pytest tests/test_dist_gpu.py tests/test_gpu_parity.py -x -q -k "blend or dist" > gpurun_out/blend_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/blend_tests.log
for fb in 1 0; do
  timeout 300 python bench.py --workload gpt2 --blend 1 --fused-blend $fb --steps 20 --cpu-sample-params 200000 2>/dev/null | grep '^{' > gpurun_out/blend_n1_f$fb.jsonl
  python -c "import json; d=json.load(open('gpurun_out/blend_n1_f$fb.jsonl')); print('n=1 fused=$fb', d['value'], d['ms_per_step'], d['avg_kernel_ms'], d['roofline']['frac'], d['gpu_launches'])"
done
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
for cfg in "1 auto" "1 0" "1 64" "1 512" "0 auto"; do
  set -- $cfg
  if [ $2 = auto ]; then LAG=-1; else LAG=$2; fi
  timeout 300 $TR --nproc-per-node $n --master-port 2964$n bench.py --gpus $n --workload gpt2 --blend 1 --nccl 0 --fused-blend $1 --blend-lag $LAG 2>/dev/null | grep '^{' > gpurun_out/blend_n${n}_f$1_l$2.jsonl
  python -c "import json; d=json.load(open('gpurun_out/blend_n${n}_f$1_l$2.jsonl')); print('n=$n fused=$1 lag=$2', d['value'], d['ms_per_step'], d['avg_kernel_ms'], d['gpu_launches'], d.get('phases_us'))"
done; done
