#!/bin/bash
# full ncu capture of the binary64 decomposition kernel on 2^24 config-3 matrices (gpurun_out/$1_lean.ncu-rep)
P=${1:-lean}
FCMD="python tools/prof_svd2.py --config ${2:-3} --count 16777216 --iters 1"
$FCMD > gpurun_out/${P}_plain.log 2>&1 &&
ncu --set full --import-source on --clock-control none -k regex:k_svd2_ -c 2 -f -o gpurun_out/${P}_lean $FCMD > gpurun_out/${P}_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/${P}_lean.ncu-rep "$P" | tee gpurun_out/${P}_summary.txt
