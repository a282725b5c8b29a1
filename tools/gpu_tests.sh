#!/bin/bash
# One GPU session: the GPU test suite and smoke().  Logs land in gpurun_out/.
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=${RAVNEST_B200_TIMEOUT_S:-10}
{ nvidia-smi; free -g; nproc; } > gpurun_out/nvsmi.log 2>&1
timeout ${PYTEST_TIMEOUT:-1200} python -m pytest ${TESTS:-tests} -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
