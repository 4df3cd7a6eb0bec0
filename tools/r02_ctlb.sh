#!/bin/bash
# k_cone_tail register caps: none (76 regs), 64, 40 -- kernel time at configs 5 and 4
export SCS_LOOP_GRAPH=0
cp paper_1312_3039_b200/libscs_b200.so /tmp/lib_keep.so
for v in ct0 ct4 ct6 ct0 ct4; do
  cp tools/_ab/lib_$v.so paper_1312_3039_b200/libscs_b200.so
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:k_cone --csv --log-file gpurun_out/ct_${v}_c5.csv python tools/ncu_iteration.py c5 --kernels > /dev/null 2>&1
  timeout 300 python tools/ncu_c4.py > gpurun_out/ct_${v}_c4.log 2>&1
  echo "$v c5: $(grep gpu__time_duration gpurun_out/ct_${v}_c5.csv | awk -F'","' '{print $5":"$NF}' | tr -d '"' | tr '\n' ' ')  c4: $(tail -1 gpurun_out/ct_${v}_c4.log | grep -o '[0-9.]* us/iteration')"
done
cp /tmp/lib_keep.so paper_1312_3039_b200/libscs_b200.so
