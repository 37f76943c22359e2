# round-1 measurement set: smoke, default bench, reference arm, ncu launch list + full captures
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench_default.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref_rc=$?; tail -1 gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1c.csv python bench.py --layers 2 --steps 2 --warmup 3 --no-graph --no-cpu --e2e-steps 1 > gpurun_out/ncu_launch_r1c.log 2>&1; echo ncu_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan2_kernel|chain_kernel|tail_wide" -s 12 -c 3 -o gpurun_out/prof_r1c python bench.py --layers 2 --steps 2 --warmup 3 --no-graph --no-cpu --e2e-steps 1 > gpurun_out/ncu_full_r1c.log 2>&1; echo ncufull_rc=$?
