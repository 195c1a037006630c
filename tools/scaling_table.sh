# Per-stage device times at config 3's distributions for several particle counts
# (DESIGN.md §9 "Scaling with the particle count"): bash tools/scaling_table.sh
for P in 250000 500000 1000000 1500000 3000000 6000000; do
  echo "P=$P $(python tools/stage_times.py --P $P --steps 20 --tag P$P 2>&1 | tail -1)"
done
