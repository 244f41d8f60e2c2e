#!/bin/bash
# the two-speed kernel against k_svd2_fast alone over batch sizes (config 3): where kLeanMin belongs
for n in 4194304 8388608 16777216 33554432 67108864; do
  for v in lean nolean; do
    if [ $v = nolean ]; then export KOG2_SVD2_NO_LEAN=1; else unset KOG2_SVD2_NO_LEAN; fi
    timeout 200 python bench.py --no-e2e --no-study --no-cpu --no-configs --steps 20 --warmup 5 --count $n 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$n $v', round(d['ms_per_step'],4), round(d['value']/1e9,3))"
  done
done
