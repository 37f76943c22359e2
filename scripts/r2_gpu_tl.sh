#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 600 python scripts/kernel_timeline.py 8 4 > gpurun_out/r2_tl.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_tl.txt
timeout 600 python scripts/scan2_timeline.py > gpurun_out/r2_s2tl.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_s2tl.txt
timeout 600 python scripts/chain_phases.py 4 > gpurun_out/r2_chain.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_chain.txt
