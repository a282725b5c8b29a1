#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=3
python tools/profile_p2p.py > gpurun_out/p2p_plain.log 2>&1 && \
ncu --devices 1 --replay-mode application --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_protocol.sum,nvltx__bytes_data_protocol.sum \
    -k regex:ring_ -s 3 -c 1 --csv --log-file gpurun_out/p2p_ncu.csv python tools/profile_p2p.py > gpurun_out/p2p_ncu.log 2>&1
echo "rc=$?"
cat gpurun_out/p2p_plain.log; tail -5 gpurun_out/p2p_ncu.log; cat gpurun_out/p2p_ncu.csv | tail -12
