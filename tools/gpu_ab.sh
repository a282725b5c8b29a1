# A/B of two builds of the library on one box (tools/_ab/{old,new}.so), N=4 BERT
export RAVNEST_B200_TIMEOUT_S=10
LIB=paper_2401_01728_b200/libravnest_b200.so
cp $LIB tools/_ab/keep.so
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for rep in 1 2 3; do for v in new old; do
  cp tools/_ab/$v.so $LIB
  timeout 300 $TR --nproc-per-node 4 --master-port 29700 bench.py --gpus 4 --nccl 0 --trace 0 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'])"
done; done
cp tools/_ab/keep.so $LIB
