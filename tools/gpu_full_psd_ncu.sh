#!/bin/bash
# full validation + bench lines, then one ncu capture of k_psd_grid (side 1000)
bash tools/gpu_full.sh
grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -1
SCS_PSD_GRID=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_psd_grid -c 1 \
  -o gpurun_out/psd_grid_1000 python tools/psd_bench.py 1000 > gpurun_out/ncu_psd.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/ncu_psd.log
