#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=3
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "local_group" > gpurun_out/pytest_local.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_local.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_protocol.sum,nvltx__bytes_data_protocol.sum
python tools/profile_p2p.py bert push > gpurun_out/p2p_push_plain.log 2>&1 && \
ncu --devices 1 --replay-mode application --clock-control none --metrics $M -k regex:ring_ -s 3 -c 1 --csv --log-file gpurun_out/p2p_push_ncu.csv python tools/profile_p2p.py bert push > gpurun_out/p2p_push_ncu.log 2>&1
echo "ncu rc=$?"; cat gpurun_out/p2p_push_plain.log
