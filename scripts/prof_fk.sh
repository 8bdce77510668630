#!/bin/bash
# ncu --set full capture of k_fk_batch on a short C4 bench run.  Usage: bash scripts/prof_fk.sh <tag>
T=${1:-cur}
B="python bench.py --steps 2 --warmup 1 --no-fit --no-cpu-baseline --frames 0 --clock-ramp 0"
$B > gpurun_out/plainfk_$T.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_fk_batch' \
    -s 2 -c 1 -o gpurun_out/proffk_$T $B > gpurun_out/ncufk_$T.log 2>&1
