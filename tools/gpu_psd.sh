#!/bin/bash
# large-PSD cooperative-grid Jacobi: parity tests + timing
timeout 900 python -m pytest tests/test_gpu_psd_large.py tests/test_gpu_parity.py -k "psd or PSD" -m gpu -q -x --durations=8 --timeout 600 -o timeout_method=thread > gpurun_out/pytest_psd.log 2>&1; echo pytest_rc=$?
tail -14 gpurun_out/pytest_psd.log; grep -E "^(FAILED|ERROR)|Error|assert " gpurun_out/pytest_psd.log | head -20
PSD_BENCH_OLD_MAX=256 timeout 600 python tools/psd_bench.py 256 500 1000 2000 > gpurun_out/psd_bench.log 2>&1; echo bench_rc=$?
cat gpurun_out/psd_bench.log | tail -8
