#!/bin/bash
# One GPU session: tests, smoke, short benches.  Logs land in gpurun_out/.
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=${RAVNEST_B200_TIMEOUT_S:-10}
NG=$(nvidia-smi -L | wc -l)
{ nvidia-smi; nvidia-smi topo -m; } > gpurun_out/nvsmi.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.log 2>&1; echo "bench1 rc=$?"; tail -2 gpurun_out/bench1.log
if [ "$NG" -ge 2 ]; then
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $NG --steps 10 --warmup 3 > gpurun_out/bench$NG.log 2>&1; echo "bench$NG rc=$?"; tail -3 gpurun_out/bench$NG.log
fi
