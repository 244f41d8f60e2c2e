#!/bin/bash
# the two-speed kernel against k_svd2_fast alone over batch sizes (config 3): where kLeanMin belongs
# (the library's threshold is lowered through KOG2_LEAN_MIN_LOG2, read by bench.py)
for n in 1048576 2097152 4194304 8388608 16777216 67108864; do
  for v in lean nolean; do
    if [ $v = nolean ]; then export KOG2_SVD2_NO_LEAN=1; else unset KOG2_SVD2_NO_LEAN; fi
    KOG2_LEAN_MIN_LOG2=16 timeout 200 python bench.py --no-e2e --no-study --no-cpu --no-configs --steps 20 --warmup 5 --count $n 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$n $v', round(d['ms_per_step'],4), round(d['value']/1e9,3))"
  done
done
