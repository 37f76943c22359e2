#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 300 python scripts/build_sweep.py --batch 1 --C 256,2048 --rho 1280 --check > gpurun_out/r2c_sweep_chk.txt 2>&1; echo "rc=$?" >> gpurun_out/r2c_sweep_chk.txt
timeout 600 python scripts/build_sweep.py --batch 8 --C 2048 --rho 1280 --check > gpurun_out/r2c_sweep_b8.txt 2>&1; echo "rc=$?" >> gpurun_out/r2c_sweep_b8.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2c_build_launches.csv python scripts/build_sweep.py --batch 8 --C 2048 --rho 1280 --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scores_tc -s 1 -c 1 -o gpurun_out/r2c_build_tc python scripts/build_sweep.py --batch 8 --C 2048 --rho 1280 --reps 1 > gpurun_out/r2c_ncu_build.log 2>&1
ncu -i gpurun_out/r2c_build_tc.ncu-rep --page raw --csv > gpurun_out/r2c_build_tc_raw.csv 2>/dev/null
ncu -i gpurun_out/r2c_build_tc.ncu-rep --page source --print-source cuda,sass --csv > /tmp/src.csv 2>/dev/null
python scripts/ncu_lines.py /tmp/src.csv 40 > gpurun_out/r2c_build_tc_lines.txt 2>&1
