#!/bin/bash
timeout 1200 python -m pytest tests/test_gpu_production.py -q -x -k mid_size --timeout 1100 > gpurun_out/ms_tests.log 2>&1; echo tests_rc=$?; tail -15 gpurun_out/ms_tests.log
