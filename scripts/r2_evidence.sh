#!/bin/bash
# Round-2 evidence run (final build) (under gpurun): the full default bench line, the ncu launch list of a
# short bench run, one ncu --set full capture each of k_render_persist, k_fk_batch and k_fit,
# and the renderer-tail / fit-phase probes (their own instrumented builds in build_prof/).
set -x
python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
S="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --fit-seeds 2 --track-frames 5 --frames 4"
$S > gpurun_out/r2_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2_launches.csv $S > gpurun_out/r2_launches.log 2>&1
bash scripts/prof_render.sh r2
bash scripts/prof_fk.sh r2
ncu -i gpurun_out/prof_r2.ncu-rep --page source --csv --kernel-name regex:k_render_persist \
    --launch-count 1 --print-source sass > gpurun_out/r2_render_src_sass.csv 2>&1
bash scripts/prof_fit.sh r2
python scripts/fit_time.py > gpurun_out/r2_fit_time.txt 2>&1
[ -e build_prof/tail.so ] && HP_LIB=build_prof/tail.so timeout 120 python scripts/tail_prof.py > gpurun_out/r2_tail.txt 2>&1
[ -e build_prof/genprof.so ] && HP_LIB=build_prof/genprof.so timeout 120 python scripts/fit_prof.py > gpurun_out/r2_fit_phases.txt 2>&1
[ -e build_prof/fkb.so ] && HP_LIB=build_prof/fkb.so timeout 120 python scripts/fkb_prof.py > gpurun_out/r2_fk_phases.txt 2>&1
