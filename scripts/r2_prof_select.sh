#!/bin/bash
# ncu source-line profile of the build's threshold and select kernels (b=1, C=2048, rho=1280)
set -u
T=${1:-ps}
mkdir -p gpurun_out
for k in select_kernel kth_value_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o /tmp/${T}_$k python scripts/build_sweep.py --batch 1 --C 2048 --rho 1280 --reps 1 > gpurun_out/${T}_$k.log 2>&1
  ncu -i /tmp/${T}_$k.ncu-rep --page source --print-source cuda,sass --csv > /tmp/src.csv 2>/dev/null
  python scripts/ncu_lines.py /tmp/src.csv 30 > gpurun_out/${T}_${k}_lines.txt 2>&1
  python scripts/ncu_summary.py /tmp/${T}_$k.ncu-rep > gpurun_out/${T}_${k}_summary.txt 2>&1
done
