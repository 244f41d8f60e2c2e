#!/bin/bash
# time k_svd2 for each built library variant and occupancy setting
for lib in paper_2407_13116_b200/lib/libkog2*.so; do
  for m in 2 3; do
    r=$(KOG2_LIB=$PWD/$lib KOG2_SVD2_MINB=$m python bench.py --steps 5 --warmup 3 --no-study --no-e2e --no-cpu --count 67108864 ${BENCH_ARGS} 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print(round(d['roofline']['kernel_ms'],3), '%.3e'%d['value'])")
    echo "$(basename $lib) minb=$m $r"
  done
done
