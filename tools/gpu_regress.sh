#!/bin/bash
# regression + headline numbers at the box's GPU count
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29516"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python bench.py > gpurun_out/bench_n1.log 2>&1; echo "N1 rc=$? $(grep -o '"avg_kernel_ms": [0-9.]*' gpurun_out/bench_n1.log) $(grep -o '"frac": [0-9.]*' gpurun_out/bench_n1.log)"
for proto in pull push auto; do
  timeout 300 $TR bench.py --gpus $NG --protocol $proto --nccl 0 > gpurun_out/bench_n${NG}_$proto.log 2>&1
  echo "N$NG $proto rc=$? $(grep -o '"bus_gbps_per_gpu": [0-9.]*' gpurun_out/bench_n${NG}_$proto.log)"
done
for wl in resnet50 gpt2; do
  timeout 300 $TR bench.py --gpus $NG --workload $wl --nccl 1 > gpurun_out/bench_n${NG}_$wl.log 2>&1
  echo "N$NG $wl rc=$? $(grep -o '"bus_gbps_per_gpu": [0-9.]*' gpurun_out/bench_n${NG}_$wl.log) $(grep -o '"nccl_compare": {[^}]*}' gpurun_out/bench_n${NG}_$wl.log)"
done
