for v in "" pb_t256 pb_s3 pb_s4 pb_t64s4; do
  if [ -n "$v" ]; then export GES_LIB=exp/$v/libges.so; else unset GES_LIB; fi
  echo "== $v"
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"particle_bwd" -s 1 -c 2 python tools/profile_step.py --steps 3 2>&1 | grep -E "duration" | awk '{print $NF}' | tr '\n' ' '; echo
done
