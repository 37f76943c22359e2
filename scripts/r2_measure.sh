#!/bin/bash
# Round-2 measurement set: smoke, GPU suite, default bench (with parity leg),
# reference arm, cfg4 build sweep, then the ncu set (scripts/profile_ncu.sh)
# and one full capture of the build GEMM for its tensor-pipe counters.
# Usage: bash scripts/r2_measure.sh TAG
set -u
T=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$T.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$T.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$T.log
timeout 900 python bench.py > gpurun_out/bench_$T.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$T.log
timeout 600 python bench.py --impl reference --steps 8 --warmup 2 > gpurun_out/bench_ref_$T.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref_$T.log
timeout 900 python scripts/build_sweep.py --batch 1 > gpurun_out/sweep_$T.txt 2>&1; echo "rc=$?" >> gpurun_out/sweep_$T.txt
bash scripts/profile_ncu.sh $T > gpurun_out/profile_ncu_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scores_tc -s 1 -c 1 -o /tmp/build_tc_$T python scripts/build_sweep.py --batch 8 --C 2048 --rho 1280 --reps 1 > gpurun_out/ncu_build_$T.log 2>&1
ncu -i /tmp/build_tc_$T.ncu-rep --page raw --csv > gpurun_out/ncu_build_raw_$T.csv 2>/dev/null
python scripts/ncu_summary.py /tmp/build_tc_$T.ncu-rep > gpurun_out/ncu_build_summary_$T.txt 2>&1
gzip -f gpurun_out/ncu_build_raw_$T.csv
