timeout 600 python scripts/chain_phases.py 4 > gpurun_out/chain_ph4.log 2>&1; echo rc=$?; cat gpurun_out/chain_ph4.log | tail -16
timeout 600 python scripts/chain_phases.py 1 > gpurun_out/chain_ph1.log 2>&1; echo rc=$?; cat gpurun_out/chain_ph1.log | tail -16
