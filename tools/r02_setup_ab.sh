#!/bin/bash
# setup-time A/B on one box: staged H2D and slab-width prediction on/off
for v in "1 1" "0 1" "1 0" "0 0" "1 1"; do
  set -- $v
  SCS_H2D_STAGED=$1 SCS_STREAM_PREDICT=$2 timeout 600 python tools/r02_setup_probe.py c5 > gpurun_out/ab_$1_$2.log 2>&1
  echo "staged=$1 predict=$2: $(grep '^setup' gpurun_out/ab_$1_$2.log | tr '\n' ' ')"
done
nproc; free -g | head -2
