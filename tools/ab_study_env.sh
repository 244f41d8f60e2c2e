#!/bin/bash
# A/B of the study leg of bench.py (2^28 matrices, config-5 rule) across environment settings:
# each argument is "label:ENV=VAL,ENV2=VAL" (empty env = defaults).  Runs the list twice, interleaved.
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for spec in "$@"; do
    label=${spec%%:*}; envs=${spec#*:}
    (
      IFS=',' ; for e in $envs; do [ -n "$e" ] && export "$e"; done; unset IFS
      python bench.py --no-e2e --no-cpu --no-configs --steps 3 --warmup 3 --study-count 268435456 2>/dev/null |
        python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$label', round(d['study']['value']/1e6, 1), d['study']['csv'][-40:])"
    )
  done
done
