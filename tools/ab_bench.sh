#!/bin/bash
# A/B: alternate bench.py (kernel only) between lib/libkog2_base.so and lib/libkog2.so
cd "$(dirname "$0")/.."
for v in base main base main; do
  if [ $v = base ]; then export KOG2_LIB=$PWD/paper_2407_13116_b200/lib/libkog2_base.so; else unset KOG2_LIB; fi
  python bench.py --no-e2e --no-study --no-cpu --no-configs --steps 10 --warmup 3 "$@" 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'], 3), round(d['value']/1e9, 3))"
done
