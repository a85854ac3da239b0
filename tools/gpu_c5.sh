#!/bin/bash
# config-5 GPU session: full-size parity test, full bench, ncu launch list + one full capture of the query kernel
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,pci.bus_id,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k config5 > gpurun_out/pytest_c5.log 2>&1; echo rc=$? >> gpurun_out/pytest_c5.log
timeout 900 python bench.py > gpurun_out/bench_c5.log 2>&1; echo rc=$? >> gpurun_out/bench_c5.log
timeout 600 python bench.py --bin off --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5_binoff.log 2>&1; echo rc=$? >> gpurun_out/bench_c5_binoff.log
SMALL="python bench.py --queries 20000000 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $SMALL > gpurun_out/plain_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv $SMALL > gpurun_out/ncu_launches.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:query_kernel -c 1 -o gpurun_out/prof_c5 $SMALL > gpurun_out/ncu_full.log 2>&1
echo ncu_rc=$? >> gpurun_out/ncu_full.log
