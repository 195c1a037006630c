#!/bin/bash
# Writes the profiles/<tag>_* summaries from gpurun_out/<tag>_* (produced on a GPU box by
# tools/profile_round.sh <tag>).  Usage (here, no GPU needed): bash tools/profile_summary.sh <tag>
set -eu
TAG=$1
IN=gpurun_out
OUT=profiles
tail -n 1 $IN/${TAG}_bench.json > $OUT/${TAG}_bench.json
{
  echo "# ncu launch list of \`python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e\` (gpu__time_duration.sum, --clock-control none; cold-cache, serialised; first 400 launches)"
  echo
  python tools/summarize_ncu.py launches $IN/${TAG}_launches.csv
  echo
  echo "Per-step share (one bench step; medians x launches per step):"
  echo
  python tools/summarize_ncu.py share $IN/${TAG}_launches.csv
} > $OUT/${TAG}_launches.md
{
  echo "# ncu --set full (tools/profile_step.py, config 3, one step after the first forward; --clock-control none)"
  echo
  python tools/summarize_ncu.py full $IN/${TAG}_full_render.ncu-rep
  echo
  python tools/summarize_ncu.py full $IN/${TAG}_full_sort.ncu-rep
} > $OUT/${TAG}_full.md
python tools/summarize_ncu.py traffic $IN/${TAG}_full_render.ncu-rep $IN/${TAG}_full_sort.ncu-rep > $OUT/${TAG}_traffic.json
python tools/pipes.py $IN/${TAG}_full_render.ncu-rep --json $OUT/${TAG}_pipes_render.json --md $OUT/${TAG}_pipes_render.md > /dev/null
python tools/pipes.py $IN/${TAG}_full_sort.ncu-rep --json $OUT/${TAG}_pipes_sort.json --md $OUT/${TAG}_pipes_sort.md > /dev/null
ls -la $OUT/${TAG}_*
