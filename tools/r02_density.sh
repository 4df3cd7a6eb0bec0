#!/bin/bash
# format choice by tile density: the new production-heuristic tests, the sparse-shape timings, C3/C5 unchanged
timeout 1200 python -m pytest tests/test_gpu_stream.py -q -x -k "density" --timeout 1100 > gpurun_out/de_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/de_tests.log
SCS_DEBUG=1 timeout 1200 python tools/r02_stream_vs_csr.py > gpurun_out/de_svc.log 2> gpurun_out/de_svc.err; echo rc=$?; cat gpurun_out/de_svc.log
timeout 1200 python -m pytest tests/test_gpu_production.py -q -x --timeout 1100 > gpurun_out/de_prod.log 2>&1; echo prod_rc=$?; tail -2 gpurun_out/de_prod.log
