# Measurement set for profiles/ (run under gpurun): gpu tests, smoke, default
# bench, the ncu launch list, and full ncu captures of the decode kernels at
# lane size and at full-layer size.  Usage: bash scripts/profile_round.sh TAG
T=${1:-r1}
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_$T.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu_$T.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke_$T.log
timeout 900 python bench.py > gpurun_out/bench_$T.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench_$T.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --layers 2 --steps 2 --warmup 3 --parity-steps 0 --e2e-steps 1 > gpurun_out/ncu_launch_$T.log 2>&1; echo ncu_rc=$?
# lane-size launches: chain_phases.py 4 runs 3 engine steps (4 lanes x scan2/chain) then one scan + chain
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan2_kernel|chain_kernel" -s 24 -c 2 -o gpurun_out/prof_${T}_lane python scripts/chain_phases.py 4 > gpurun_out/ncu_full_${T}_lane.log 2>&1; echo ncufull_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan2_kernel|chain_kernel" --launch-skip-before-match 0 -c 2 -o gpurun_out/prof_${T}_layer python bench.py --layers 2 --steps 2 --warmup 3 --parity-steps 0 --e2e-steps 1 > gpurun_out/ncu_full_${T}_layer.log 2>&1; echo ncufull2_rc=$?
