#!/bin/bash
# config-4 cone kernel timings, the bench's sharded path as 2 processes on one GPU (host group), the CPU reference arm
SCS_LOOP_GRAPH=0 timeout 300 python tools/ncu_c4.py > gpurun_out/r02_c4_plain.log 2>&1; echo c4_rc=$?; tail -1 gpurun_out/r02_c4_plain.log
SCS_LOOP_GRAPH=0 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_c4_launches.csv python tools/ncu_c4.py > gpurun_out/r02_c4_ncu.log 2>&1; echo c4ncu_rc=$?
SCS_BENCH_HOSTCOMM=1 SCS_BENCH_CONFIG=c3 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r02_bench_2proc_c3.log 2> gpurun_out/r02_bench_2proc_c3.err; echo twoproc_rc=$?
tail -c 600 gpurun_out/r02_bench_2proc_c3.log
( time timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/r02_bench_ref.log 2> gpurun_out/r02_bench_ref.err; echo ref_rc=$?
tail -c 800 gpurun_out/r02_bench_ref.log; tail -4 gpurun_out/r02_bench_ref.err
