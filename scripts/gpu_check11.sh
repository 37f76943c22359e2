timeout 600 python scripts/chain_phases.py 4 > gpurun_out/chain_ph4.log 2>&1; echo rc=$?; tail -16 gpurun_out/chain_ph4.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"chain_kernel" -s 8 -c 1 -o gpurun_out/prof_chain python bench.py --layers 2 --steps 2 --warmup 3 --no-graph --no-cpu --e2e-steps 1 > gpurun_out/ncu_chain.log 2>&1; echo ncu_rc=$?
