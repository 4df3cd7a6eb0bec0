#!/bin/bash
# sharded format agreement (every rank streams a matrix or none)
timeout 1500 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_multiproc.py tests/test_gpu_stream.py -q -x --timeout 1400 > gpurun_out/ag_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/ag_tests.log
