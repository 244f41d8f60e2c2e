#!/bin/bash
# One GPU call's worth of round measurements (run under gpurun from the repo root):
# full GPU test suite, the default bench line, the launch list of the bench command under ncu,
# the DRAM traffic of one 2^28 cfg3 svd2 call and a full ncu capture of k_svd2_fast at 2^24.
# Outputs land in gpurun_out/ with the prefix given as $1 (default r2).
P=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${P}_smi.txt
python -m pytest tests -m gpu -x -q > gpurun_out/${P}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${P}_pytest_gpu.log
python bench.py > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err; echo "bench rc=$?" >> gpurun_out/${P}_bench.err
LCMD="python bench.py --no-e2e --no-cpu --steps 2 --warmup 3 --study-count 33554432"
$LCMD > gpurun_out/${P}_plain_launch.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches.csv $LCMD > gpurun_out/${P}_ncu_launch.log 2>&1
TCMD="python tools/prof_svd2.py --config 3 --count 268435456 --iters 1"
$TCMD > gpurun_out/${P}_plain_traffic.log 2>&1 &&
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_svd2 --csv --log-file gpurun_out/${P}_traffic.csv $TCMD > gpurun_out/${P}_ncu_traffic.log 2>&1
FCMD="python tools/prof_svd2.py --config 3 --count 16777216 --iters 1"
$FCMD > gpurun_out/${P}_plain_full.log 2>&1 &&
ncu --set full --import-source on --clock-control none -k regex:k_svd2_fast -c 1 -f -o gpurun_out/${P}_fast $FCMD > gpurun_out/${P}_ncu_full.log 2>&1
echo done
