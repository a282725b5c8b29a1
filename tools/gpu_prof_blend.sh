#!/bin/bash
# ncu --set full of a fused-blend kernel (one ncu per call):
#   tools/gpu_prof_blend.sh n1    co-resident TMA, BERT C=8 (1 GPU)
#   tools/gpu_prof_blend.sh push  push, 2 GPUs in one process, device 1 profiled
set -u
mkdir -p gpurun_out
export RAVNEST_B200_TIMEOUT_S=5
if [ "${1:-n1}" = n1 ]; then
  python tools/profile_n1.py bert 8 f64 blend > gpurun_out/prof_blend_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:ring_ -s 2 -c 1 \
      -o gpurun_out/prof_${TAG:-r02}_n1_bert_c8_blend -f python tools/profile_n1.py bert 8 f64 blend > gpurun_out/prof_blend_ncu.log 2>&1
  echo "ncu n1 blend rc=$?"
else
  python tools/profile_p2p.py bert push blend > gpurun_out/p2p_blend_plain.log 2>&1 && \
  timeout 1500 ncu --devices 1 --replay-mode application --set full --clock-control none --import-source on \
      -k regex:ring_push -s 3 -c 1 -o gpurun_out/prof_${TAG:-r02}_push_c2_blend -f python tools/profile_p2p.py bert push blend \
      > gpurun_out/p2p_blend_full.log 2>&1
  echo "ncu push blend rc=$?"; tail -1 gpurun_out/p2p_blend_plain.log
fi
