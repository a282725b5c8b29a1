# fused blend: blend items interleaved (0) vs a dedicated set of blend-only blocks
# historical: the kernel variant this measured was removed afterwards (DESIGN.md tuning table); the knob is now ignored
export RAVNEST_B200_TIMEOUT_S=10
RAVNEST_B200_BLEND_BLOCKS=64 RAVNEST_DIST_QUICK=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29670 tests/dist_worker.py 2>&1 | grep "DIST"
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do
for bb in 0 48 96 148 0; do
  RAVNEST_B200_BLEND_BLOCKS=$bb timeout 300 $TR --nproc-per-node $n --master-port 2967$n bench.py --gpus $n --workload gpt2 --blend 1 --nccl 0 2>/dev/null | grep '^{' > gpurun_out/bs_n${n}_$bb.jsonl
  python -c "import json; d=json.load(open('gpurun_out/bs_n${n}_$bb.jsonl')); print('n=$n blend_blocks=$bb', d['value'], d['ms_per_step'], d.get('phases_us'))"
done; done
