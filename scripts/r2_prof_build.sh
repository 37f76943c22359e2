#!/bin/bash
# Full ncu capture of the build's filter-pass GEMM (b=1, C=2048, rho=1280)
# with source-line stall attribution.  Usage: bash scripts/r2_prof_build.sh TAG
set -u
T=${1:-pb}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scores_tc -s 1 -c 1 -o /tmp/${T}_btc python scripts/build_sweep.py --batch 1 --C 2048 --rho 1280 --reps 1 > gpurun_out/${T}_ncu.log 2>&1
ncu -i /tmp/${T}_btc.ncu-rep --page raw --csv > gpurun_out/${T}_raw.csv 2>/dev/null
ncu -i /tmp/${T}_btc.ncu-rep --page source --print-source cuda,sass --csv > /tmp/src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/src.csv 40 > gpurun_out/${T}_lines.txt 2>&1
ncu -i /tmp/${T}_btc.ncu-rep --page source --print-source sass --csv > /tmp/sass.csv 2>/dev/null
python scripts/ncu_sass_top.py /tmp/sass.csv 40 > gpurun_out/${T}_sass.txt 2>&1
gzip -f gpurun_out/${T}_raw.csv
