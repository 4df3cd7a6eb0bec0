#!/bin/bash
# (historical: measured and reverted; the variant and its knob are no longer in the tree -- DESIGN §5.1)
# k_split_combine4 (four threads per row) vs the one-thread-per-row combine
timeout 900 python -m pytest tests/test_gpu_stream.py -q -x --timeout 800 > gpurun_out/c4_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/c4_tests.log
for m in 8 1000; do
for c in c3; do
  SCS_DEBUG=1 SCS_COMBINE4_MIN=$m SCS_BENCH_CONFIG=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/cm${m}_$c.log 2> gpurun_out/cm${m}_$c.err
  grep "stream sched" gpurun_out/cm${m}_$c.err | head -4
  python -c "
import json;d=json.loads(open('gpurun_out/cm${m}_$c.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('m=$m $c value %.2f e2e %.2f A %.3f At %.3f sm %s' % (d['value'], d['e2e']['value'], k['spmv_A(q=A p)']['ms'], k['spmv_At_cg(Gp=p+A^T q; p\'Gp)']['ms'], d['clocks']['sm_mhz']))"
done
done
export SCS_LOOP_GRAPH=0
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/cm_c3.csv python tools/ncu_iteration.py c3 --kernels > gpurun_out/cm_c3.log 2>&1; echo list_rc=$?
