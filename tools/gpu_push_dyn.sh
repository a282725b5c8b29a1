# push work distribution: static stride vs a work counter, with and without interleaved folds
# historical: RAVNEST_B200_PUSH_LAG (fold interleaving) was removed afterwards; only the PUSH_DYN legs still apply
export RAVNEST_B200_TIMEOUT_S=10
for d in 1; do
RAVNEST_B200_PUSH_DYN=$d RAVNEST_DIST_QUICK=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29630 tests/dist_worker.py 2>&1 | grep "DIST"
RAVNEST_B200_PUSH_DYN=$d RAVNEST_B200_PUSH_LAG=0.5 RAVNEST_DIST_QUICK=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29631 tests/dist_worker.py 2>&1 | grep "DIST"
done
for wl in resnet50 bert gpt2; do
for cfg in "0 none" "1 none" "1 1" "1 2" "0 1"; do
  set -- $cfg
  export RAVNEST_B200_PUSH_DYN=$1
  if [ $2 = none ]; then unset RAVNEST_B200_PUSH_LAG; else export RAVNEST_B200_PUSH_LAG=$2; fi
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 4 --steps 50 --warmup 5 --workload $wl --nccl 0 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl dyn $1 lag $2', d['bus_gbps_per_gpu'], d['ms_per_step'], d.get('phases_us'))"
done; done
