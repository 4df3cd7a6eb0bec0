#!/bin/bash
# full validation: every GPU test, smoke, default bench (N=1), config-3 bench, reference arm
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 2300 > gpurun_out/va_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/va_tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/va_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/va_smoke.log
timeout 1200 python bench.py > gpurun_out/va_bench.log 2> gpurun_out/va_bench.err; echo bench_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/va_bench.log').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], 'clk', d['clocks'])
print('tte', d.get('time_to_eps',{}).get('time_to_eps_s'), d.get('time_to_eps',{}).get('check',{}).get('ok'))"
SCS_BENCH_CONFIG=c3 timeout 900 python bench.py --steps 20 --warmup 5 --no-configs > gpurun_out/va_bench_c3.log 2> gpurun_out/va_bench_c3.err; echo c3_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/va_bench_c3.log').read().strip().splitlines()[-1])
print('c3 value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'])"
