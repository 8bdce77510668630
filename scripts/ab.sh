#!/bin/bash
# A/B kernel variants: the default build, then every build in build_variants/ (HP_LIB), each
# run twice in alternation to expose box-to-box drift.  Usage (under gpurun): bash scripts/ab.sh [reps]
R=${1:-2}
B="python bench.py --steps 100 --warmup 5 --no-fit --no-cpu-baseline --frames 0 --clock-ramp 0.3"
P='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("%.3fM hyp/s  step %.4f ms render %.4f ms fk %.4f ms  frac %.4f" % (d["value"]/1e6, d["ms_per_step"], r["kernel_ms"], r["fk_kernel_ms"], r["frac"]))'
for i in $(seq $R); do
  echo "default: $($B | python -c "$P")"
  for f in build_variants/*.so; do
    [ -e "$f" ] || continue
    echo "$f: $(HP_LIB=$f $B | python -c "$P")"
  done
done
