# GPU round trip: parity suite, then the default bench (cfg2)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench_rc=$?; tail -2 gpurun_out/bench_full.log | cut -c1-3000
