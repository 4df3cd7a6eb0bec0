#!/bin/bash
# final bench lines: the driver's default invocation (N=1) and config 3
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fz_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/fz_smoke.log
timeout 1200 python bench.py > gpurun_out/fz_bench.log 2> gpurun_out/fz_bench.err; echo bench_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/fz_bench.log').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], d['roofline']['kernel'], 'clk', d['clocks']['sm_mhz'], 'tte', d['time_to_eps']['time_to_eps_s'], d['time_to_eps']['check']['ok'])"
SCS_BENCH_CONFIG=c3 timeout 900 python bench.py --steps 20 --warmup 5 --no-configs > gpurun_out/fz_bench_c3.log 2> gpurun_out/fz_bench_c3.err; echo c3_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/fz_bench_c3.log').read().strip().splitlines()[-1])
print('c3 value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'])"
