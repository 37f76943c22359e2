#!/bin/bash
# BASELINE configs beyond the default bench line: cfg1 (8K fp32 parity
# config), cfg3 (Yi-9B geometry, capacity plan), cfg5 (128K, one GPU's slice
# of the 8-GPU kv-head x batch plan, global batch sweep), cfg2 no-rerank
# ablation (Fig. 11).  One bench JSON line per run in gpurun_out/cov_*.txt.
set -u
mkdir -p gpurun_out
run() { local tag=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/cov_$tag.txt 2>&1; echo "rc=$?" >> gpurun_out/cov_$tag.txt; }
run cfg1 --config cfg1
run cfg2_norerank --config cfg2 --no-rerank
run cfg3 --config cfg3
for B in 1 2 4 8 16 32; do run cfg5_b$B --config cfg5 --batch $B; done
run cfg5_b64 --config cfg5 --batch 64 --phys-layers 24
