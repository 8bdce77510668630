#!/bin/bash
# ncu --set full capture of the persistent fit kernel k_fit (C3 fit) with source attribution.
# Usage (under gpurun): bash scripts/prof_fit.sh <tag>
T=${1:-cur}
python scripts/fit_time.py > gpurun_out/plainfit_$T.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_fit" -s 24 -c 1 \
    -o gpurun_out/proffit_$T python scripts/fit_time.py > gpurun_out/ncufit_$T.log 2>&1
ncu -i gpurun_out/proffit_$T.ncu-rep --page source --csv --kernel-name regex:k_fit \
    --launch-count 1 --print-source sass > gpurun_out/fit_src_sass_$T.csv 2>&1
ncu -i gpurun_out/proffit_$T.ncu-rep --page raw --csv > gpurun_out/fit_raw_$T.csv 2>&1
