for it in 1 2 3 4 6 8; do
  RAVNEST_B200_PUSH_ITEMS=$it python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 4 --steps 50 --warmup 5 --workload resnet50 --nccl 0 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('items $it', d['bus_gbps_per_gpu'], d['ms_per_step'], d.get('phases_us'))"
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --steps 50 --warmup 5 --workload resnet50 --nccl 0 --protocol pull 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pull', d['bus_gbps_per_gpu'], d['ms_per_step'], d.get('phases_us'))"
