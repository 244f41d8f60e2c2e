#!/bin/bash
# DRAM traffic of one kog_svd2_batch call per config (full size) under ncu -> profiles/svd2_traffic.json
P=${1:-r2}
mkdir -p gpurun_out
specs=""
for c in 1 2 3 4; do
  case $c in 1) N=1048576;; 2) N=67108864;; *) N=268435456;; esac
  CMD="python tools/prof_svd2.py --config $c --count $N --iters 1"
  $CMD > gpurun_out/${P}_traffic_plain_$c.log 2>&1 &&
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:k_svd2 --csv --log-file gpurun_out/${P}_traffic_$c.csv $CMD > gpurun_out/${P}_traffic_ncu_$c.log 2>&1
  specs="$specs $c:$N:gpurun_out/${P}_traffic_$c.csv"
done
python tools/traffic_json.py gpurun_out/${P}_svd2_traffic.json $specs
