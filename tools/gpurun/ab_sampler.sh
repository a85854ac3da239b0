mkdir -p gpurun_out
for v in base s1 old; do
  case $v in base) env="";; *) env="PNDF_LIB=$PWD/paper_2109_14807_b200/libpndf_$v.so";; esac
  for c in 5 2; do
    env $env timeout 600 python bench.py --op sample --config $c --steps 3 --warmup 3 > gpurun_out/abs_${v}_$c.log 2>&1
    tail -1 gpurun_out/abs_${v}_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $c, '%.3e'%d['value'], d['parity_sample'])"
  done
done
