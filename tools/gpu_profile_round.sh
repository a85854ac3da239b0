#!/bin/bash
# round profile: default bench (plain) -> its ncu launch list -> one --set full capture of the query kernel
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv python bench.py > gpurun_out/ncu_launches.log 2>&1
echo launches_rc=$? >> gpurun_out/ncu_launches.log
CMD="python bench.py --queries 100000000 --bin on --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:query_kernel -c 1 -o gpurun_out/prof_query $CMD > gpurun_out/ncu_full.log 2>&1
echo full_rc=$? >> gpurun_out/ncu_full.log
timeout 900 ncu --set full --clock-control none -k regex:rs_scatter -c 1 -o gpurun_out/prof_scatter $CMD > gpurun_out/ncu_scatter.log 2>&1
echo scatter_rc=$? >> gpurun_out/ncu_scatter.log
