#!/bin/bash
# per-kernel launch list of the phased study (two chunks of 2^23 by default): time, executed instructions, issue rate, registers
# usage (on the GPU box): tools/study_launches.sh PREFIX   -> gpurun_out/PREFIX_study_launches.csv
P=${1:-r9}
SCMD="python tools/prof_svd2.py --study --count ${STUDY_COUNT:-16777216} --iters 1"
timeout 300 $SCMD > gpurun_out/${P}_plain.log 2>&1 &&
timeout 500 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none --csv --log-file gpurun_out/${P}_study_launches.csv $SCMD > gpurun_out/${P}_ncu.log 2>&1
echo done
