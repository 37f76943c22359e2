#!/bin/bash
# Round-2 GPU round trip: smoke, the GPU suite, one bench line.
set -u
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_smoke.txt
timeout 1200 python -m pytest tests -m gpu -q -s > gpurun_out/r2_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_tests.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_bench.txt
