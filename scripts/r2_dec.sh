#!/bin/bash
# Decode change check: GPU suite (engine + scale parity first), bench line,
# steady-state timeline.  Usage: bash scripts/r2_dec.sh TAG
set -u
T=${1:-dec}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_scale_parity_gpu.py -q -x -p no:cacheprovider > gpurun_out/${T}_tests_eng.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests_eng.txt
timeout 900 python bench.py > gpurun_out/${T}_bench.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench.txt
timeout 600 python scripts/kernel_timeline.py 8 4 > gpurun_out/${T}_tl.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tl.txt
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${T}_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.txt
