#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=10
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29524"
nvidia-smi topo -m > gpurun_out/topo.log 2>&1; head -8 gpurun_out/topo.log
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p.pci_domain_id, p.pci_bus_id, p.pci_device_id)"
for nb in 0 1; do
  timeout 300 $TR bench.py --gpus $NG --steps 20 --nccl 0 --numa-bind $nb > gpurun_out/numa_$nb.log 2>&1; echo "numa_bind=$nb rc=$? $(grep -o '"e2e": {[^}]*}' gpurun_out/numa_$nb.log)"
done
