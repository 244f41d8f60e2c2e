#!/bin/bash
# quick GPU check of a kernel change: svd2 parity subsets, then the bench kernel line with and without the lean kernel
P=${1:-leanq}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_parity.py tests/test_gpu_reentrancy.py -m gpu -x -q > gpurun_out/${P}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${P}_pytest.log
for v in lean nolean lean nolean; do
  if [ $v = nolean ]; then export KOG2_SVD2_NO_LEAN=1; else unset KOG2_SVD2_NO_LEAN; fi
  timeout 300 python bench.py --no-e2e --no-study --no-cpu --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', 'cfg3', round(d['ms_per_step'],3), round(d['value']/1e9,3), {k:(round(c['ms_per_step'],3), round(c['value']/1e9,2)) for k,c in d.get('configs',{}).items()} if isinstance(d.get('configs'),dict) else d.get('configs'))" >> gpurun_out/${P}_ab.txt 2>&1
done
cat gpurun_out/${P}_ab.txt
tail -3 gpurun_out/${P}_pytest.log
