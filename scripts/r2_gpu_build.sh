#!/bin/bash
# GPU: build correctness + sweep (new tcgen05 epilogue), test suite, bench.
set -u
mkdir -p gpurun_out
timeout 300 python scripts/build_sweep.py --batch 1 --C 256,2048 --rho 1280 --check > gpurun_out/r2_sweep_chk.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_sweep_chk.txt
timeout 600 python scripts/build_sweep.py --batch 1 > gpurun_out/r2_sweep_b1.txt 2>&1
timeout 600 python scripts/build_sweep.py --batch 8 --C 2048 --rho 1280 --check > gpurun_out/r2_sweep_b8.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -s -x > gpurun_out/r2_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_tests.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_bench.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scores_tc|kth|select|gather_sample|fallback" --csv --log-file gpurun_out/r2_build_launches2.csv python scripts/build_sweep.py --batch 8 --C 2048 --rho 1280 --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scores_tc -s 1 -c 1 -o gpurun_out/r2_build_tc2 python scripts/build_sweep.py --batch 8 --C 2048 --rho 1280 --reps 1 > gpurun_out/r2_ncu_build2.log 2>&1
