#!/bin/bash
# per-device dynamic shared-memory ceilings (smem_optin) + the kernels that use them
timeout 1500 python -m pytest tests/test_gpu_psd_large.py tests/test_gpu_stream.py tests/test_gpu_c4.py tests/test_gpu_parity.py -q -x --timeout 1400 > gpurun_out/sa_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/sa_tests.log
SCS_BENCH_CONFIG=c5 timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/sa_c5.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/sa_c5.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('c5 value %.2f e2e %.2f A %.3f At %.3f frac %.3f sm %s' % (d['value'], d['e2e']['value'], k['spmv_A(q=A p)']['ms'], k['spmv_At_cg(Gp=p+A^T q; p\'Gp)']['ms'], d['roofline']['frac'], d['clocks']['sm_mhz']))"
