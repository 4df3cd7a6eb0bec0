#!/bin/bash
timeout 600 python tools/r02_h2d_probe.py > gpurun_out/h2d.log 2>&1; echo rc=$?; cat gpurun_out/h2d.log; nproc; free -g | head -2
