#!/bin/bash
# A/B of the study leg of bench.py (2^28 matrices, config-5 rule) across lib variants ("main" = lib/libkog2.so)
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = main ]; then unset KOG2_LIB; else export KOG2_LIB=$PWD/paper_2407_13116_b200/lib/libkog2_$v.so; fi
    python bench.py --no-e2e --no-cpu --no-configs --steps 3 --warmup 3 --study-count 268435456 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['study']['value']/1e6, 1), d['study']['csv'][-60:])"
  done
done
