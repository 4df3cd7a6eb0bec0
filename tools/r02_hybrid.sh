#!/bin/bash
# (historical: measured and reverted; the variant and its knob are no longer in the tree -- DESIGN §5.1)
# hybrid split schedules (whole units beside split ones) vs uniform splits
timeout 1200 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -x --timeout 1100 > gpurun_out/hy_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/hy_tests.log
for hy in 1 0 1; do
for c in c3; do
  SCS_DEBUG=1 SCS_STREAM_HYBRID=$hy SCS_BENCH_CONFIG=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/hy${hy}_$c.log 2> gpurun_out/hy${hy}_$c.err
  grep "stream sched" gpurun_out/hy${hy}_$c.err | head -4
  python -c "
import json;d=json.loads(open('gpurun_out/hy${hy}_$c.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('hy=$hy $c value %.2f e2e %.2f A %.3f At %.3f sm %s' % (d['value'], d['e2e']['value'], k['spmv_A(q=A p)']['ms'], k['spmv_At_cg(Gp=p+A^T q; p\'Gp)']['ms'], d['clocks']['sm_mhz']))"
done
done
SCS_BENCH_CONFIG=c5 timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/hy_c5.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/hy_c5.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('c5 value %.2f e2e %.2f A %.3f At %.3f sm %s' % (d['value'], d['e2e']['value'], k['spmv_A(q=A p)']['ms'], k['spmv_At_cg(Gp=p+A^T q; p\'Gp)']['ms'], d['clocks']['sm_mhz']))"
export SCS_LOOP_GRAPH=0
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/hy_c3.csv python tools/ncu_iteration.py c3 --kernels > gpurun_out/hy_c3l.log 2>&1; echo list_rc=$?
