#!/bin/bash
# Round-2 GPU round trip: scale parity, the GPU suite, one bench line.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_scale_parity_gpu.py -x -q -s > gpurun_out/r2_scale.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_scale.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_tests.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_bench.txt
