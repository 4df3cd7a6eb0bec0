#!/bin/bash
SCS_DEBUG=1 timeout 900 python tools/r02_stream_edge.py > gpurun_out/se.log 2> gpurun_out/se.err; echo rc=$?
cat gpurun_out/se.log; grep -E "stream layout|stream pin|narrow|flag|csr_sb" gpurun_out/se.err | head -20
