#!/bin/bash
# Time bench.py (kernel only) for each named lib variant in turn, twice:
#   tools/ab_multi.sh base main [variant ...] [-- extra bench.py args]   ("main" = lib/libkog2.so)
cd "$(dirname "$0")/.."
vars=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do vars+=("$1"); shift; done
[ "$1" = "--" ] && shift
for rep in 1 2; do
  for v in "${vars[@]}"; do
    if [ "$v" = main ]; then unset KOG2_LIB; else export KOG2_LIB=$PWD/paper_2407_13116_b200/lib/libkog2_$v.so; fi
    python bench.py --no-e2e --no-study --no-cpu --steps 10 --warmup 3 "$@" 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'], 3), round(d['value']/1e9, 3))"
  done
done
