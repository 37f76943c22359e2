# v2 decode kernels + tcgen05 build: ncu full captures (one GPU)
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -4 gpurun_out/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan2_kernel|unit2_kernel" -s 4 -c 2 -o gpurun_out/prof_decode_r1b python bench.py --layers 2 --steps 2 --warmup 2 --no-graph --no-cpu --e2e-steps 1 > gpurun_out/ncu_decode.log 2>&1; echo decode_prof_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scores_tc_kernel|select_kernel|kth_value" -c 4 -o gpurun_out/prof_build_r1b python bench.py --layers 1 --steps 1 --warmup 1 --no-graph --no-cpu --e2e-steps 1 > gpurun_out/ncu_build.log 2>&1; echo build_prof_rc=$?
