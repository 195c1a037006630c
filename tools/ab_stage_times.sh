# A/B per-stage device times of build variants (tools/stage_times.py), interleaved:
# bash tools/ab_stage_times.sh "base head opq2" [rounds] [config]
VARS=${1:-"base"}; R=${2:-2}; CFG=${3:-3}
for r in $(seq $R); do for v in $VARS; do
  if [ $v = base ]; then unset GES_LIB; else export GES_LIB=paper_2402_10128_b200/build/variants/$v/libges.so; fi
  echo "$v $(python tools/stage_times.py --config $CFG --steps 30 --tag $v 2>&1 | tail -1)"
done; done
