#!/bin/bash
timeout 1200 python tools/r02_stream_vs_csr.py --small > gpurun_out/sg.log 2>&1; echo rc=$?; cat gpurun_out/sg.log
