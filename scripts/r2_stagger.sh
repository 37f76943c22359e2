#!/bin/bash
# Lane staggering experiment: steady-state timelines and bench lines with the
# lanes' scans unranked (0) and ranked in lane order (1).
set -u
mkdir -p gpurun_out
T=${1:-stg}
for s in 0 1; do
  timeout 600 python scripts/kernel_timeline.py 8 4 $s > gpurun_out/${T}_tl$s.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tl$s.txt
done
for s in 0 1; do
  timeout 900 python bench.py --parity-steps 0 --stagger $s > gpurun_out/${T}_bench$s.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench$s.txt
done
timeout 900 python bench.py --parity-steps 0 --stagger 1 --lanes 8 > gpurun_out/${T}_bench1_l8.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench1_l8.txt
