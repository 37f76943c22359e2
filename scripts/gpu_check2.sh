timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/phase_times.py 1 > gpurun_out/phase.log 2>&1; tail -24 gpurun_out/phase.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench_full.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench_full.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ['value','ms_per_step']}, d['kernels']['scan_kernel'], d['kernels']['unit_kernel'], d['build'], d['e2e'])"
