#!/bin/bash
# ncu --set full capture of the batch renderer (and k_fk_batch) on a short C4 bench run.
# Usage (under gpurun): bash scripts/prof_render.sh <tag>
T=${1:-cur}
B="python bench.py --steps 2 --warmup 1 --no-fit --no-cpu-baseline --frames 0 --clock-ramp 0"
$B > gpurun_out/plain_$T.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_render_persist|k_fk_batch' \
    -s 6 -c 3 -o gpurun_out/prof_$T $B > gpurun_out/ncu_$T.log 2>&1
