#!/bin/bash
# A/B (ab_env.sh) then one ncu --set full capture of the default query kernel (KREGEX) on a 2e8-query config-5 batch
bash tools/gpurun/ab_env.sh
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-parity --queries ${PQ:-200000000}"
timeout 600 $CMD > gpurun_out/plain_prof.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-query_g5} -c 1 -o gpurun_out/prof_${PNAME:-g5} -f $CMD > gpurun_out/ncu_prof.log 2>&1
echo prof_rc=$? >> gpurun_out/ncu_prof.log; tail -1 gpurun_out/ncu_prof.log
