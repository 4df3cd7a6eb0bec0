#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_optin.py tests/test_gpu_bands.py tests/test_gpu_parity.py -q -x --timeout 300 -o timeout_method=thread > gpurun_out/pytest_optin.log 2>&1; echo rc=$?; tail -5 gpurun_out/pytest_optin.log
grep -E "^(FAILED|ERROR)|Error|assert" gpurun_out/pytest_optin.log | head -20
