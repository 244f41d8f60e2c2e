#!/bin/bash
# A/B kernel timings (bench.py, kernel only): each argument is "label:ENV=VAL,ENV2=VAL" (empty env
# = main library defaults; KOG2_LIB=... selects a built variant).  Runs the list twice, interleaved.
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for spec in "$@"; do
    label=${spec%%:*}; envs=${spec#*:}
    (
      IFS=',' ; for e in $envs; do [ -n "$e" ] && export "$e"; done; unset IFS
      python bench.py --no-e2e --no-study --no-cpu --steps 10 --warmup 3 ${BENCH_ARGS} 2>/dev/null |
        python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$label', round(d['ms_per_step'], 3), round(d['value']/1e9, 3))"
    )
  done
done
