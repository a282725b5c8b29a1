# push work order: fold items interleaved after a lag of N resident-grid rounds
# historical: the kernel variant this measured was removed afterwards (DESIGN.md tuning table); the knob is now ignored
RAVNEST_B200_PUSH_LAG=1 RAVNEST_DIST_QUICK=1 RAVNEST_B200_TIMEOUT_S=10 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29620 tests/dist_worker.py 2>&1 | grep "DIST" 
RAVNEST_B200_PUSH_LAG=0.3 RAVNEST_DIST_QUICK=1 RAVNEST_B200_TIMEOUT_S=10 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29621 tests/dist_worker.py 2>&1 | grep "DIST"
for wl in resnet50 bert; do
for lag in none 0.5 1 2; do
  if [ $lag = none ]; then unset RAVNEST_B200_PUSH_LAG; else export RAVNEST_B200_PUSH_LAG=$lag; fi
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29622 bench.py --gpus 4 --steps 50 --warmup 5 --workload $wl --nccl 0 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl lag $lag', d['bus_gbps_per_gpu'], d['ms_per_step'], d.get('phases_us'))"
done; done
