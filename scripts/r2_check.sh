#!/bin/bash
# Change check: build correctness + cfg4 sweep point, GPU suite, bench line,
# steady-state timeline.  Usage: bash scripts/r2_check.sh TAG
set -u
T=${1:-chk}
mkdir -p gpurun_out
timeout 300 python scripts/build_sweep.py --batch 1 --C 256,2048 --rho 1280 --check > gpurun_out/${T}_sweep_chk.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_sweep_chk.txt
timeout 600 python scripts/build_sweep.py --batch 8 --C 2048 --rho 1280 > gpurun_out/${T}_sweep_b8.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_sweep_b8.txt
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${T}_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.txt
timeout 900 python bench.py > gpurun_out/${T}_bench.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench.txt
timeout 600 python scripts/kernel_timeline.py 8 4 > gpurun_out/${T}_tl.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tl.txt
