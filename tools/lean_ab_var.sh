#!/bin/bash
# bench kernel line (config 3, 2^28) for library variants, alternating: tools/lean_ab_var.sh VARIANT...
for rep in 1 2; do
  for v in "$@"; do
    if [ $v = main ]; then unset KOG2_LIB; else export KOG2_LIB=$PWD/paper_2407_13116_b200/lib/libkog2_$v.so; fi
    timeout 200 python bench.py --no-e2e --no-study --no-cpu --no-configs --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3), round(d['value']/1e9,3))"
  done
done
