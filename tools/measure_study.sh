#!/bin/bash
# One GPU call: the default bench line (study with its reference run_batch baseline), the bench
# lines of configs 1, 2, 4, and a full ncu capture of k_study over one 2^22 config-5 chunk.
# Outputs land in gpurun_out/ with the prefix given as $1.
P=${1:-r7b}
mkdir -p gpurun_out
python bench.py > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err; echo "bench rc=$?" >> gpurun_out/${P}_bench.err
for c in 1 2 4; do
  python bench.py --config $c --no-study >> gpurun_out/${P}_configs.jsonl 2>> gpurun_out/${P}_configs.err
done
SCMD="python tools/prof_svd2.py --study --count 4194304 --iters 1"
$SCMD > gpurun_out/${P}_plain_study.log 2>&1 &&
ncu --set full --import-source on --clock-control none -k regex:k_study -c 1 -f -o gpurun_out/${P}_study $SCMD > gpurun_out/${P}_ncu_study.log 2>&1
echo done
