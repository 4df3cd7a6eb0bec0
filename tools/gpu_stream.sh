#!/bin/bash
# streamed-tile kernel: GPU tests, then C3 / C5 bench lines
timeout 900 python -m pytest tests/test_gpu_stream.py -m gpu -q -x --timeout 300 -o timeout_method=thread > gpurun_out/pytest_stream.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_stream.log; grep -E "^(FAILED|ERROR)|Error|assert " gpurun_out/pytest_stream.log | head -20
if [ "${BENCH:-1}" = "1" ]; then
SCS_DEBUG=1 timeout 600 python bench.py --config c3 --steps 50 --no-cpu --no-tte --no-optin > gpurun_out/bench_c3_stm.log 2> gpurun_out/bench_c3_stm.err; echo c3_rc=$?
grep -E "stream" gpurun_out/bench_c3_stm.err | head; tail -c 600 gpurun_out/bench_c3_stm.log
SCS_DEBUG=1 timeout 900 python bench.py --steps 20 --no-cpu --no-tte --no-optin > gpurun_out/bench_c5_stm.log 2> gpurun_out/bench_c5_stm.err; echo c5_rc=$?
grep -E "stream|create|built|graph" gpurun_out/bench_c5_stm.err | head -20; tail -c 900 gpurun_out/bench_c5_stm.log
fi
