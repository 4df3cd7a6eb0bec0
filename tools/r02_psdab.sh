#!/bin/bash
# A/B of k_psd_small builds on config 4 (us/iteration, device-timed) and the kernel's own time
cp paper_1312_3039_b200/libscs_b200.so /tmp/lib_keep.so
for v in orig kc lb4 lb6 orig lb4; do
  cp tools/_ab/lib_$v.so paper_1312_3039_b200/libscs_b200.so
  SCS_LOOP_GRAPH=0 timeout 300 python tools/ncu_c4.py > gpurun_out/ab_$v.log 2>&1
  SCS_LOOP_GRAPH=0 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:k_psd_small --csv --log-file gpurun_out/ab_$v.csv python tools/ncu_c4.py > /dev/null 2>&1
  echo "$v $(tail -1 gpurun_out/ab_$v.log | grep -o '[0-9.]* us/iteration') psd_small $(grep gpu__time_duration gpurun_out/ab_$v.csv | tail -1 | awk -F'\",\"' '{print $NF}')"
done
cp /tmp/lib_keep.so paper_1312_3039_b200/libscs_b200.so
