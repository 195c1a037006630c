#!/bin/bash
# stage_times for the base library and every variant under build/variants/
python tools/stage_times.py --tag base 2>&1 | tail -1
for d in paper_2402_10128_b200/build/variants/*/; do
  v=$(basename $d)
  GES_LIB=$d/libges.so python tools/stage_times.py --tag $v 2>&1 | tail -1
done
