#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 300 python scripts/build_sweep.py --batch 1 --C 256,2048 --rho 1280 --check > gpurun_out/r2b_sweep_chk.txt 2>&1; echo "rc=$?" >> gpurun_out/r2b_sweep_chk.txt
timeout 600 python scripts/build_sweep.py --batch 8 --C 2048 --rho 1280 --check > gpurun_out/r2b_sweep_b8.txt 2>&1; echo "rc=$?" >> gpurun_out/r2b_sweep_b8.txt
timeout 600 python -m pytest tests -m gpu -q -x -k "build or tc or fast or scale" > gpurun_out/r2b_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2b_tests.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2b_build_launches.csv python scripts/build_sweep.py --batch 8 --C 2048 --rho 1280 --reps 1 > /dev/null 2>&1
