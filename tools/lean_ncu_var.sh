#!/bin/bash
# ncu summary (+ DRAM bytes) of k_svd2_lean for library variants: tools/lean_ncu_var.sh PREFIX COUNT VARIANT...
P=$1; shift
N=$1; shift
for v in "$@"; do
  if [ $v = main ]; then unset KOG2_LIB; else export KOG2_LIB=$PWD/paper_2407_13116_b200/lib/libkog2_$v.so; fi
  FCMD="python tools/prof_svd2.py --config 3 --count $N --iters 1"
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_svd2_lean -c 1 -f -o gpurun_out/${P}_$v $FCMD > gpurun_out/${P}_${v}_ncu.log 2>&1
  python tools/ncu_summary.py gpurun_out/${P}_$v.ncu-rep "$P $v" | tee -a gpurun_out/${P}_summary.txt
done
