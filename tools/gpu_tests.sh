#!/bin/bash
# GPU tests only (optionally a subset: TESTS="tests/test_x.py ...")
timeout 1200 python -m pytest ${TESTS:-tests} -m gpu -q -x --timeout 300 -o timeout_method=thread > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log; grep -E "^(FAILED|ERROR)|Error|assert " gpurun_out/pytest_gpu.log | head -30
