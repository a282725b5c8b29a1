#!/bin/bash
set -u
mkdir -p gpurun_out
M=gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_protocol.sum,nvltx__bytes_data_protocol.sum
for mode in write read mixed bulkstore bulkload; do
  ./tools/nvlink_probe 437928960 $mode > gpurun_out/probe_$mode.log 2>&1 || echo "plain $mode failed"
done
for mode in write read mixed bulkstore bulkload; do
  ncu --devices 1 --clock-control none --metrics $M -k regex:probe -s 2 -c 1 --csv --log-file gpurun_out/probe_ncu_$mode.csv ./tools/nvlink_probe 437928960 $mode > /dev/null 2>&1
  echo "$mode: $(cat gpurun_out/probe_$mode.log | tail -1)"
  grep -E "nvl|duration" gpurun_out/probe_ncu_$mode.csv | awk -F'","' '{print "   ", $(NF-2), $NF}'
done
