#!/bin/bash
# GPU: decode change check -- GPU suite, bench line, steady-state timeline.
set -u
mkdir -p gpurun_out
T=${1:-dec}
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench.txt
timeout 600 python scripts/kernel_timeline.py 8 4 > gpurun_out/${T}_tl.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tl.txt
