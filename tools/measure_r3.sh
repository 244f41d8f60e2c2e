#!/bin/bash
# Round-3-style measurement call (run under gpurun from the repo root): the full GPU test suite, the default
# bench line, the reference arm, and the ncu captures of the two-speed kernel (2^26 config-3 matrices).
P=${1:-r3}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${P}_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${P}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${P}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err; echo "bench rc=$?" >> gpurun_out/${P}_bench.err
LCMD="python bench.py --no-e2e --no-cpu --steps 2 --warmup 3 --study-count 33554432"
timeout 600 $LCMD > gpurun_out/${P}_plain_launch.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches.csv $LCMD > gpurun_out/${P}_ncu_launch.log 2>&1
TCMD="python tools/prof_svd2.py --config 3 --count 268435456 --iters 1"
timeout 300 $TCMD > gpurun_out/${P}_plain_traffic.log 2>&1 &&
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_svd2 --csv --log-file gpurun_out/${P}_traffic.csv $TCMD > gpurun_out/${P}_ncu_traffic.log 2>&1
FCMD="python tools/prof_svd2.py --config 3 --count 67108864 --iters 1"
timeout 300 $FCMD > gpurun_out/${P}_plain_full.log 2>&1 &&
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_svd2_lean -c 1 -f -o gpurun_out/${P}_lean $FCMD > gpurun_out/${P}_ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/${P}_lean.ncu-rep "$P k_svd2_lean 2^26 cfg3" > gpurun_out/${P}_lean_summary.txt 2>&1
tail -3 gpurun_out/${P}_pytest_gpu.log; tail -c 1500 gpurun_out/${P}_bench.json; cat gpurun_out/${P}_lean_summary.txt
echo done
