# Copy one measurement set (scripts/profile_ncu.sh TAG + a default bench run
# into gpurun_out/bench_TAG.log) into the tracked profiles/ summaries.
# Usage: bash scripts/update_profiles.sh TAG [ROUND]
T=${1:?tag}
R=${2:-r2}
grep '^{' gpurun_out/bench_$T.log | tail -1 > profiles/${R}_bench.json
cp gpurun_out/ncu_traffic_$T.json profiles/ncu_traffic.json
{
  echo "# $R launch list"' (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none; `bench.py --layers 2 --steps 2 --warmup 3 --parity-steps 0 --e2e-steps 1`)'
  echo
  echo "Measurement set \`$T\` (\`scripts/profile_ncu.sh $T\`). Cold-cache, serialised per-launch times (compare shares, not absolutes). Full-layer launches (scan2 grid 2624, chain 256, tail 64) come from the bench timing pass (lanes=1); grid 656 / 64 / 16 launches are the 4-lane engine's per-lane kernels (2 sequences = 16 (b, kv-head) units each). Only this repo's kernels are listed (ctkv:: decode, tc:: index build); the torch kernels in the raw list are the synthetic-data generator outside the timed region."
  echo
  echo '| kernel | grid | launches | mean us | mean DRAM MB/launch |'
  echo '|---|---|---|---|---|'
  grep -E "^\| (ctkv|tc)::" gpurun_out/launches_$T.md
} > profiles/${R}_launches.md
{
  echo "# $R decode kernels"': ncu --set full (B200, cfg2 geometry)'
  echo
  echo "Measurement set \`$T\` (\`scripts/profile_ncu.sh $T\`): lane-size launches (the 4-lane engine's per-lane scan2 + chain, \`scripts/chain_phases.py 4\`) and full-layer launches (bench timing pass). \`--clock-control none\`, serialised and cold-cache: shares, not absolute step time."
  echo
  echo '## full-layer launches (scan2 grid 2624, chain grid 256)'
  echo
  cat gpurun_out/ncu_summary_${T}_layer.txt
  echo
  echo 'DRAM traffic per full-layer launch: `profiles/ncu_traffic.json` (scan2 vs 176.4 MB algorithmic).'
  echo
  echo '## lane-size launches (scan2 grid 656, chain grid 64)'
  echo
  cat gpurun_out/ncu_summary_${T}_lane.txt
  for w in lane layer; do for k in chain scan2; do
    echo
    echo "## $k ($w): warp-stall samples by source line"
    echo
    sed 's/^/    /' gpurun_out/ncu_lines_${T}_${w}_$k.txt | head -20
    echo
    echo "## $k ($w): top SASS by warp-stall samples"
    echo
    sed 's/^/    /' gpurun_out/ncu_sass_${T}_${w}_$k.txt | head -14
  done; done
} > profiles/${R}_ncu_decode.md
echo updated
