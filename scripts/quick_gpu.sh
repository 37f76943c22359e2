#!/bin/bash
# One GPU round trip after a kernel change: parity tests, chain phases,
# steady-state timeline and a short bench (outputs under gpurun_out/).
set -u
T=${1:-full}
if [ "$T" = "full" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/q_tests.txt
fi
timeout 300 python scripts/chain_phases.py 8 > gpurun_out/q_cp8.txt 2>&1
timeout 300 python scripts/kernel_timeline.py 8 8 > gpurun_out/q_kt.txt 2>&1
timeout 600 python bench.py --parity-steps 0 --steps 20 --warmup 5 > gpurun_out/q_bench.txt 2>&1
