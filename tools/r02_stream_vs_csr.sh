#!/bin/bash
SCS_DEBUG=1 timeout 1200 python tools/r02_stream_vs_csr.py > gpurun_out/svc.log 2> gpurun_out/svc.err; echo rc=$?
cat gpurun_out/svc.log; grep -E "stream layout" gpurun_out/svc.err | head -20
