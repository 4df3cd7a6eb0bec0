#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 1200 > gpurun_out/r02_gpu8_tests.log 2>&1; echo tests_rc=$?
tail -6 gpurun_out/r02_gpu8_tests.log
for c in c5 c3; do
  SCS_BENCH_CONFIG=$c timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-tte --no-optin --no-cpu > gpurun_out/q8_$c.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/q8_$c.log').read().strip().splitlines()[-1])
k=d['roofline']['kernels']; print('$c value %.2f e2e %.2f A %.3f At %.3f' % (d['value'], d['e2e']['value'], k['spmv_A(q=A p)']['ms'], k['spmv_At_cg(Gp=p+A^T q; p\'Gp)']['ms']))"
done
SCS_BENCH_FORCE_SHARDED=1 SCS_BENCH_CONFIG=c3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --steps 10 --warmup 3 > gpurun_out/q8_nccl1.log 2>&1; echo nccl1_rc=$?; tail -c 300 gpurun_out/q8_nccl1.log
