#!/bin/bash
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=5
python tools/profile_p2p.py bert push > gpurun_out/p2p_push_plain.log 2>&1 && \
timeout 1500 ncu --devices 1 --replay-mode application --set full --clock-control none --import-source on \
    -k regex:ring_push -s 3 -c 1 -o gpurun_out/prof_r01_push_c2 -f python tools/profile_p2p.py bert push > gpurun_out/p2p_push_full.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/p2p_push_full.log; cat gpurun_out/p2p_push_plain.log | tail -1
