#!/bin/bash
# (historical: measured and reverted; the variant and its knob are no longer in the tree -- DESIGN §5.1)
# in-kernel combine of split partials (StmOut mode 2) vs the combine kernel
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py -q -x --timeout 800 > gpurun_out/ic_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/ic_tests.log
for ic in 1 0; do
for c in c3 c5; do
  SCS_STREAM_INCOMBINE=$ic SCS_BENCH_CONFIG=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/ic${ic}_$c.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/ic${ic}_$c.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('ic=$ic $c value %.2f e2e %.2f A %.3f At %.3f sm %s' % (d['value'], d['e2e']['value'], k['spmv_A(q=A p)']['ms'], k['spmv_At_cg(Gp=p+A^T q; p\'Gp)']['ms'], d['clocks']['sm_mhz']))"
done
done
export SCS_LOOP_GRAPH=0
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ic_c3.csv python tools/ncu_iteration.py c3 --kernels > gpurun_out/ic_c3.log 2>&1; echo list_rc=$?
