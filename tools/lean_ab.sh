#!/bin/bash
# bench kernel line with and without the lean kernel (no tests)
P=${1:-lean}
for v in lean nolean lean nolean; do
  if [ $v = nolean ]; then export KOG2_SVD2_NO_LEAN=1; else unset KOG2_SVD2_NO_LEAN; fi
  timeout 300 python bench.py --no-e2e --no-study --no-cpu --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', 'cfg3', round(d['ms_per_step'],3), round(d['value']/1e9,3), {k:(round(c['ms_per_step'],3), round(c['value']/1e9,2)) for k,c in d.get('configs',{}).items()} if isinstance(d.get('configs'),dict) else d.get('configs'))" >> gpurun_out/${P}_ab.txt 2>&1
done
cat gpurun_out/${P}_ab.txt
