#!/bin/bash
# compute-sanitizer over the round-2 paths: 8-CTA chain clusters (small
# geometries), 4-CTA clusters at 24 units (engine, lanes), the kernel
# staging copies of the host-I/O graphs, the tensor-core build, the
# tensor-core static partitions over a ragged static window.
set -u
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool memcheck python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "geometries and 8-8-128" > gpurun_out/san_mem_geo.txt 2>&1
timeout 1200 compute-sanitizer --tool racecheck python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "geometries and 16-2-128" > gpurun_out/san_race_geo.txt 2>&1
timeout 1500 compute-sanitizer --tool memcheck python -m pytest tests/test_engine_gpu.py -q -p no:cacheprovider -k "host or stage_copy or 12" > gpurun_out/san_mem_eng.txt 2>&1
timeout 1500 compute-sanitizer --tool memcheck python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "cfg1_bf16_fast_build" > gpurun_out/san_mem_build.txt 2>&1
timeout 1200 compute-sanitizer --tool memcheck python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "ragged" > gpurun_out/san_mem_ragged.txt 2>&1
timeout 1500 compute-sanitizer --tool racecheck python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -k "ragged and (32-4-128 or 16-8-64)" > gpurun_out/san_race_ragged.txt 2>&1
for f in san_mem_geo san_race_geo san_mem_eng san_mem_build san_mem_ragged san_race_ragged; do echo "== $f"; grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/$f.txt | tail -3; done > gpurun_out/san_summary.txt
