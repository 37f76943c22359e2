#!/bin/bash
# Decode re-measurement after a kernel change: smoke, GPU suite, default
# bench line, reference arm, the decode ncu set (scripts/profile_ncu.sh) and
# every BASELINE config (scripts/r2_configs.sh).  Usage: bash scripts/r2_final.sh TAG
set -u
T=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$T.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$T.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$T.log
timeout 900 python bench.py > gpurun_out/bench_$T.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$T.log
timeout 600 python bench.py --impl reference --steps 8 --warmup 2 > gpurun_out/bench_ref_$T.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref_$T.log
bash scripts/profile_ncu.sh $T > gpurun_out/profile_ncu_$T.log 2>&1
bash scripts/r2_configs.sh
