#!/bin/bash
# full ncu capture of k_psd_small on config 4 (11,111 PSD blocks of side 3-8)
export SCS_LOOP_GRAPH=0
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_psd_small -c 1 -o gpurun_out/r02_psd_small_kc python tools/ncu_c4.py > gpurun_out/r02_psd_small.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/r02_psd_small.log
