#!/bin/bash
# GPU: the gs=16 geometry fix + GPU suite, then the build's launch list and
# one full ncu capture of the filter-pass GEMM (tensor-pipe counters).
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_tests.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_build_launches.csv python scripts/build_sweep.py --batch 8 --C 2048 --rho 1280 --reps 1 > gpurun_out/r2_build_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scores_tc -s 1 -c 1 -o gpurun_out/r2_build_tc python scripts/build_sweep.py --batch 8 --C 2048 --rho 1280 --reps 1 > gpurun_out/r2_ncu_build.log 2>&1
ncu -i gpurun_out/r2_build_tc.ncu-rep --page raw --csv > gpurun_out/r2_build_tc_raw.csv 2>/dev/null
ncu -i gpurun_out/r2_build_tc.ncu-rep --page source --print-source cuda,sass --csv > /tmp/src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/src.csv 40 > gpurun_out/r2_build_tc_lines.txt 2>&1
