#!/bin/bash
# ncu source-line profile of the deferred tail kernel (lane-size launch)
set -u
T=${1:-pt}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_kernel -s 8 -c 1 -o /tmp/${T}_tail python scripts/chain_phases.py 4 > gpurun_out/${T}_tail.log 2>&1
ncu -i /tmp/${T}_tail.ncu-rep --page source --print-source cuda,sass --csv > /tmp/src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/src.csv 30 > gpurun_out/${T}_tail_lines.txt 2>&1
python scripts/ncu_summary.py /tmp/${T}_tail.ncu-rep > gpurun_out/${T}_tail_summary.txt 2>&1
cp /tmp/${T}_tail.ncu-rep gpurun_out/
