# Per-kernel ncu times (gpu__time_duration) of the default library and every build/variants/* library
# (kernels matching $KREGEX, default depth_sort): bash tools/variant_kernel_times.sh
for d in "" paper_2402_10128_b200/build/variants/*/; do
  if [ -n "$d" ]; then export GES_LIB=$d/libges.so; v=$(basename $d); else unset GES_LIB; v=base; fi
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"${KREGEX:-depth_sort}" --csv python tools/profile_step.py --steps 3 2>/dev/null > gpurun_out/kt_v.csv
  echo "== $v $(python tools/ktimes.py gpurun_out/kt_v.csv | tr '\n' ' ' | tr -s ' ')"
done
