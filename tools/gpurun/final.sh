#!/bin/bash
# full GPU validation + round evidence: tests, smoke, benches of every op, ncu launch list + captures
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
for c in 1 2 3 4; do timeout 600 python bench.py --config $c > gpurun_out/bench_c$c.log 2>&1; done
for op in sample sg wang wang_sample; do timeout 600 python bench.py --op $op > gpurun_out/bench_$op.log 2>&1; done
timeout 600 python bench.py --op blocked --config 2 > gpurun_out/bench_blocked.log 2>&1
timeout 600 python bench.py --op blocked_sample --config 2 > gpurun_out/bench_blocked_sample.log 2>&1
timeout 600 python bench.py --op als --config 2 > gpurun_out/bench_als.log 2>&1
timeout 900 python bench.py --op als_map --config 3 --steps 10 > gpurun_out/bench_als_map.log 2>&1
timeout 900 python bench.py --op sweep > gpurun_out/bench_sweep.log 2>&1
timeout 600 python bench.py --config 3 --s0 4 > gpurun_out/bench_c3_s04.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv python bench.py > gpurun_out/ncu_launches.log 2>&1
echo launches_rc=$? >> gpurun_out/ncu_launches.log
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-parity"
timeout 600 $CMD > gpurun_out/plain_full.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:query_g5 -c 1 -o gpurun_out/prof_query_full -f $CMD > gpurun_out/ncu_full.log 2>&1
echo full_rc=$? >> gpurun_out/ncu_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rs_scatter -c 1 -o gpurun_out/prof_scatter_full -f $CMD > gpurun_out/ncu_scatter.log 2>&1
echo scatter_rc=$? >> gpurun_out/ncu_scatter.log
SCMD="python bench.py --op sample --steps 1 --warmup 1"
timeout 600 $SCMD > gpurun_out/plain_sample.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sample_kernel -c 1 -o gpurun_out/prof_sample -f $SCMD > gpurun_out/ncu_sample.log 2>&1
echo sample_rc=$? >> gpurun_out/ncu_sample.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_als_map.csv python bench.py --op als_map --config 3 --steps 2 --warmup 3 --no-e2e > gpurun_out/ncu_als_map_l.log 2>&1
echo done >> gpurun_out/ncu_als_map_l.log
