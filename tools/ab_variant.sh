#!/bin/bash
# A/B of the bench kernel line: alternate lib/libkog2.so ("main") and lib/libkog2_<variant>.so
# usage: tools/ab_variant.sh VARIANT [bench args...]
cd "$(dirname "$0")/.."
V=$1; shift
for v in main $V main $V main $V; do
  if [ $v = main ]; then unset KOG2_LIB; else export KOG2_LIB=$PWD/paper_2407_13116_b200/lib/libkog2_$v.so; fi
  python bench.py --no-e2e --no-study --no-cpu --no-configs --steps 10 --warmup 3 "$@" 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'], 3), round(d['value']/1e9, 3))"
done
