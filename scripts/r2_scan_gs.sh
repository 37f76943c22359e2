#!/bin/bash
# scan2 at gs = 4 (cfg2) vs gs = 8 (cfg3): per-CTA timelines and one ncu
# --set full capture of a full-layer launch at each geometry
set -u
mkdir -p gpurun_out
for geo in "8 8" "16 4"; do
  tag=$(echo $geo | tr ' ' x)
  timeout 600 python scripts/scan2_timeline.py $geo > gpurun_out/scan_tl_$tag.txt 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan2 -s 12 -c 1 \
    -o /tmp/scan_$tag python scripts/scan2_timeline.py $geo > gpurun_out/scan_ncu_$tag.log 2>&1
  python scripts/ncu_summary.py /tmp/scan_$tag.ncu-rep > gpurun_out/scan_sum_$tag.txt 2>&1
  ncu -i /tmp/scan_$tag.ncu-rep --page source --print-source cuda,sass --csv > /tmp/src_$tag.csv 2>/dev/null
  python scripts/ncu_lines.py /tmp/src_$tag.csv 30 > gpurun_out/scan_lines_$tag.txt 2>&1
  cp /tmp/scan_$tag.ncu-rep gpurun_out/
done
