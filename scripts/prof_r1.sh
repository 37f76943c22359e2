set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "kats or dot_scores" > gpurun_out/pytest_kats.log 2>&1; tail -2 gpurun_out/pytest_kats.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --layers 2 --seq 98304 --steps 2 --warmup 2 --no-graph --no-cpu --e2e-steps 1 > gpurun_out/ncu_launch_bench.log 2>&1; echo launches_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan_kernel|unit_kernel" -s 4 -c 2 -o gpurun_out/prof_decode_r1 python bench.py --layers 2 --seq 98304 --steps 2 --warmup 2 --no-graph --no-cpu --e2e-steps 1 > gpurun_out/ncu_decode.log 2>&1; echo decode_prof_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"scores_kernel|topk_rows" -c 2 -o gpurun_out/prof_build_r1 python bench.py --layers 1 --seq 98304 --steps 1 --warmup 1 --no-graph --no-cpu --e2e-steps 1 > gpurun_out/ncu_build.log 2>&1; echo build_prof_rc=$?
ls -la gpurun_out
