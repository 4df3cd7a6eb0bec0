#!/bin/bash
timeout 600 python tools/r02_setup_probe.py c5 > gpurun_out/r10_setup.log 2>&1; echo rc=$?
grep -v "stream pin\|stream layout\|stream sched\|piece cap" gpurun_out/r10_setup.log | tail -25
SCS_LOOP_GRAPH=0 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r10_c1_launches.csv python tools/ncu_c1.py > gpurun_out/r10_c1.log 2>&1; echo c1_rc=$?; tail -1 gpurun_out/r10_c1.log
timeout 300 python tools/ncu_c1.py > gpurun_out/r10_c1_plain.log 2>&1; tail -1 gpurun_out/r10_c1_plain.log
