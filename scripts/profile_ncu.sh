# ncu part of the measurement set, summarised on the box so only small text
# files (and the lane-size report) come back.  Usage: bash scripts/profile_ncu.sh TAG
T=${1:-r1}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --layers 2 --steps 2 --warmup 3 --parity-steps 0 --e2e-steps 1 > gpurun_out/ncu_launch_$T.log 2>&1; echo ncu_rc=$?
python scripts/ncu_launches.py gpurun_out/launches_$T.csv > gpurun_out/launches_$T.md
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan2_kernel|chain_kernel" -s 24 -c 2 -o /tmp/prof_${T}_lane python scripts/chain_phases.py 4 > gpurun_out/ncu_full_${T}_lane.log 2>&1; echo ncufull_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan2_kernel|chain_kernel" -c 2 -o /tmp/prof_${T}_layer python bench.py --layers 2 --steps 2 --warmup 3 --parity-steps 0 --e2e-steps 1 > gpurun_out/ncu_full_${T}_layer.log 2>&1; echo ncufull2_rc=$?
for w in lane layer; do
  python scripts/ncu_summary.py /tmp/prof_${T}_$w.ncu-rep > gpurun_out/ncu_summary_${T}_$w.txt 2>&1
  ncu -i /tmp/prof_${T}_$w.ncu-rep --page raw --csv > gpurun_out/ncu_raw_${T}_$w.csv 2>/dev/null
  for k in scan2 chain; do
    ncu -i /tmp/prof_${T}_$w.ncu-rep -k regex:$k --page source --print-source cuda,sass --csv > /tmp/src_$k.csv 2>/dev/null
    python scripts/ncu_lines.py /tmp/src_$k.csv 25 > gpurun_out/ncu_lines_${T}_${w}_$k.txt 2>&1
    ncu -i /tmp/prof_${T}_$w.ncu-rep -k regex:$k --page source --print-source sass --csv > /tmp/sass_$k.csv 2>/dev/null
    python scripts/ncu_sass_top.py /tmp/sass_$k.csv 25 > gpurun_out/ncu_sass_${T}_${w}_$k.txt 2>&1
  done
done
python scripts/ncu_traffic.py /tmp/prof_${T}_layer.ncu-rep > gpurun_out/ncu_traffic_$T.log 2>&1; cp profiles/ncu_traffic.json gpurun_out/ncu_traffic_$T.json
cp /tmp/prof_${T}_lane.ncu-rep gpurun_out/ 2>/dev/null
gzip -f gpurun_out/ncu_raw_${T}_*.csv gpurun_out/launches_$T.csv
du -sh gpurun_out
