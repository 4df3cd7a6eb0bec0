#!/bin/bash
timeout 1200 python tools/r02_stream_vs_csr.py --crossover > gpurun_out/co.log 2>&1; echo rc=$?; cat gpurun_out/co.log
