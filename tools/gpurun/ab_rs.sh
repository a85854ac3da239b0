#!/bin/bash
# radix tile-size A/B: "name:lib:env" triples
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
for spec in $SPECS; do
  name=${spec%%:*}; rest=${spec#*:}; lib=${rest%%:*}; vars=${rest#*:}
  e=""; [ "$lib" != "base" ] && e="PNDF_LIB=$PWD/paper_2109_14807_b200/libpndf_$lib.so"
  env $e ${vars//,/ } timeout 600 $B > gpurun_out/ab_$name.log 2>&1
  python - "$name" <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/ab_{f}.log").read().strip().splitlines()[-1])
    r=d["roofline"]; ps=d.get("parity_sample") or {}
    print(f"{f:12s} value {d['value']:.3e} kernel_ms {r['kernel_ms']:.2f} bin_ms {r['binning_ms']:.2f} parity {ps.get('pass')}")
except Exception as e:
    print(f, "ERR", e, open(f"gpurun_out/ab_{f}.log").read()[-800:])
PY
done
