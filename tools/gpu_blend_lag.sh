# fused blend: lag (in groups of C items) between a unit's fold and its blends
export RAVNEST_B200_TIMEOUT_S=10
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 4 2; do
for rounds in 2 4 8 16; do
  lag=$(( rounds * 296 / n ))
  RAVNEST_B200_BLEND_LAG=$lag timeout 300 $TR --nproc-per-node $n --master-port 2965$n bench.py --gpus $n --workload gpt2 --blend 1 --nccl 0 2>/dev/null | grep '^{' > gpurun_out/bl_n${n}_$lag.jsonl
  python -c "import json; d=json.load(open('gpurun_out/bl_n${n}_$lag.jsonl')); print('n=$n rounds=$rounds lag=$lag', d['value'], d['ms_per_step'], d.get('phases_us'))"
done; done
