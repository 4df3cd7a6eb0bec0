#!/bin/bash
# where config-5 setup time goes (SCS_DEBUG timestamps), twice in one process
SCS_DEBUG=1 timeout 900 python tools/r02_setup_probe.py > gpurun_out/sh.log 2> gpurun_out/sh.err; echo rc=$?
grep -E "create enter|validated|L2 pers|create m=|values copied|row indices|matrices built|equilibrated|streamed format built|graph built|setup " gpurun_out/sh.err gpurun_out/sh.log | head -40
