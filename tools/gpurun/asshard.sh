#!/bin/bash
# per-GPU cost of the 2/4/8-GPU config-5 jobs on one GPU (bench.py --as-shard 0/W), spatial and index sharding
mkdir -p gpurun_out
for W in 2 4 8; do
  for S in spatial index; do
    timeout 900 python bench.py --as-shard 0/$W --shard $S --no-cpu-baseline --no-e2e > gpurun_out/bench_asshard_${S}_$W.log 2>&1
    python - "$S" "$W" <<'PY'
import json,sys
S,W=sys.argv[1:3]
try:
    L=[l for l in open(f"gpurun_out/bench_asshard_{S}_{W}.log").read().splitlines() if l.startswith("{")]
    d=json.loads(L[-1]); print(S, W, "%.4g q/s"%d["value"], "ms/step %.2f"%d["ms_per_step"], d["config"].get("queries_per_rank"))
except Exception as e:
    print(S, W, "ERR", e)
PY
  done
done
