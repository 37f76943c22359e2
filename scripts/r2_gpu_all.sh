#!/bin/bash
# GPU round trip: smoke, build check, GPU suite, bench, build launch list.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/r2_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_smoke.txt
timeout 300 python scripts/build_sweep.py --batch 1 --C 256,2048 --rho 1280 --check > gpurun_out/r2_sweep_chk.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_sweep_chk.txt
timeout 1500 python -m pytest tests -m gpu -q -s -x > gpurun_out/r2_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_tests.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_bench.txt
timeout 600 python scripts/build_sweep.py --batch 1 > gpurun_out/r2_sweep_b1.txt 2>&1
