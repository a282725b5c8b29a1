# fp64 push path after the vectors-per-pass change + PCIe ceilings for the e2e leg
export RAVNEST_B200_TIMEOUT_S=10
timeout 900 python -m pytest tests/test_dist_gpu.py -x -q > gpurun_out/dist_f64.log 2>&1; echo "dist tests rc=$?"; tail -1 gpurun_out/dist_f64.log
timeout 300 python tools/pcie_probe.py > gpurun_out/pcie_probe.json 2>&1; cat gpurun_out/pcie_probe.json
