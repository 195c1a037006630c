#!/bin/bash
# quick GPU check of the sort path: parity tests touching the lists, stage times, bin kernel times
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/stage_times.py 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 12 --csv python tools/profile_step.py --steps 2 > gpurun_out/kt_base.csv 2>/dev/null
shopt -s nullglob
for d in paper_2402_10128_b200/build/variants/*/; do
  v=$(basename $d)
  GES_LIB=$d/libges.so timeout 300 python tools/stage_times.py --tag $v 2>&1 | tail -1
  GES_LIB=$d/libges.so ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 12 --csv python tools/profile_step.py --steps 2 > gpurun_out/kt_$v.csv 2>/dev/null
done
