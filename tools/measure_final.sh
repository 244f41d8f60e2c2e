#!/bin/bash
# Round-end measurement call: tools/measure_all.sh (GPU tests, bench line, launch list, traffic, ncu of the
# f64 fast kernel) plus the bench lines of configs 1, 2, 4 and an ncu capture of the binary32 fast kernel.
P=${1:-r8}
bash tools/measure_all.sh $P
for c in 1 2 4; do
  python bench.py --config $c --no-study >> gpurun_out/${P}_configs.jsonl 2>> gpurun_out/${P}_configs.err
done
FCMD="python tools/prof_svd2.py --config 4 --count 16777216 --iters 1"
$FCMD > gpurun_out/${P}_plain_f32.log 2>&1 &&
ncu --set full --import-source on --clock-control none -k regex:k_svd2_fast -c 1 -f -o gpurun_out/${P}_fast_f32 $FCMD > gpurun_out/${P}_ncu_f32.log 2>&1
echo done
