#!/bin/bash
# One GPU session of measurements for profiles/: bench line, ncu launch list of
# the bench command, ncu --set full captures of the hot kernels.
# Usage (on the GPU box): bash tools/profile_round.sh [tag]
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
python -m pytest tests -m gpu -x -q > $OUT/${TAG}_pytest.log 2>&1; tail -2 $OUT/${TAG}_pytest.log
python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err || { echo "bench failed"; tail -20 $OUT/${TAG}_bench.err; exit 1; }
tail -c 600 $OUT/${TAG}_bench.json
# launch list of the bench command (cold-cache, serialised per-launch times)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $OUT/${TAG}_ncu_launch.log 2>&1
# full captures: the hot kernels of one step (after the first forward)
ncu --set full --import-source on --clock-control none \
    -k regex:"render_bwd|render_fwd|preprocess_tma|particle_bwd_tma" -s 2 -c 4 \
    -o $OUT/${TAG}_full_render -f python tools/profile_step.py --steps 1 > $OUT/${TAG}_ncu_full1.log 2>&1
ncu --set full --import-source on --clock-control none \
    -k regex:"depth_sort|bin_" -s 4 -c 4 \
    -o $OUT/${TAG}_full_sort -f python tools/profile_step.py --steps 1 > $OUT/${TAG}_ncu_full2.log 2>&1
ls -la $OUT
