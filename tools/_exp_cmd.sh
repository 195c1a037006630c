for v in chunk8192 "" chunk32768 chunk65536; do
  if [ -n "$v" ]; then export GES_LIB=exp/$v/libges.so; else unset GES_LIB; fi
  echo "== $v"
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bin_" -s 6 -c 3 python tools/profile_step.py --steps 3 2>&1 | grep -E "^  [a-z_]+kernel|duration" | paste - - | awk '{print $1, $NF}'
done
