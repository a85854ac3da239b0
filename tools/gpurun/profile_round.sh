#!/bin/bash
# round profile: default bench (plain) -> ncu launch list of the same command -> --set full captures
# of the query kernel (full size, first launch), the radix scatter, and the sampling kernel
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv python bench.py > gpurun_out/ncu_launches.log 2>&1
echo launches_rc=$? >> gpurun_out/ncu_launches.log
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-parity"
timeout 600 $CMD > gpurun_out/plain_full.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:query_kernel -c 1 -o gpurun_out/prof_query_full $CMD > gpurun_out/ncu_full.log 2>&1
echo full_rc=$? >> gpurun_out/ncu_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rs_scatter -c 1 -o gpurun_out/prof_scatter_full $CMD > gpurun_out/ncu_scatter.log 2>&1
echo scatter_rc=$? >> gpurun_out/ncu_scatter.log
SCMD="python bench.py --op sample --steps 1 --warmup 1"
timeout 600 $SCMD > gpurun_out/plain_sample.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sample_kernel -c 1 -o gpurun_out/prof_sample $SCMD > gpurun_out/ncu_sample.log 2>&1
echo sample_rc=$? >> gpurun_out/ncu_sample.log
