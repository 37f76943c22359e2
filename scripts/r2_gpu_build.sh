#!/bin/bash
# GPU: test suite, cfg4 build sweep, ncu of the tcgen05 build.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -s > gpurun_out/r2_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_tests.txt
timeout 600 python scripts/build_sweep.py --batch 1 > gpurun_out/r2_sweep_b1.txt 2>&1
timeout 600 python scripts/build_sweep.py --batch 8 --C 2048 --rho 1280 --check > gpurun_out/r2_sweep_b8.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_build_launches.csv python scripts/build_sweep.py --batch 8 --C 2048 --rho 1280 --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scores_tc -s 1 -c 1 -o gpurun_out/r2_build_tc python scripts/build_sweep.py --batch 8 --C 2048 --rho 1280 --reps 1 > gpurun_out/r2_ncu_build.log 2>&1
