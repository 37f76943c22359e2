# round-1 measurement set (d): gpu tests, smoke, default bench, ncu launch list + full captures
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench_default.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1d.csv python bench.py --layers 2 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_launch_r1d.log 2>&1; echo ncu_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan2_kernel|chain_kernel" -s 4 -c 2 -o gpurun_out/prof_r1d python bench.py --layers 2 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_full_r1d.log 2>&1; echo ncufull_rc=$?
