# phase breakdown of the v2 unit kernel, v4 A/B, ncu full of scan2 + unit2
CTKV_DECODE=2 timeout 600 python scripts/phase_times.py 2 > gpurun_out/phase_v2.log 2>&1; echo phase_rc=$?; cat gpurun_out/phase_v2.log | tail -30
CTKV_DECODE=4 timeout 900 python bench.py --no-cpu --steps 10 > gpurun_out/bench_d4.log 2>&1; echo "decode v4 rc=$?"; tail -1 gpurun_out/bench_d4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ['value','ms_per_step']})" || tail -5 gpurun_out/bench_d4.log
CTKV_DECODE=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan2_kernel|unit2_kernel" -s 4 -c 2 -o gpurun_out/prof_v2 python bench.py --layers 2 --steps 2 --warmup 3 --no-graph --no-cpu --e2e-steps 1 > gpurun_out/ncu_v2.log 2>&1; echo ncu_rc=$?
