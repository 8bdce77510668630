#!/bin/bash
# A/B kernel variants: default build, env switches, and builds in build_variants/.
B="python bench.py --steps 100 --warmup 5 --no-fit --no-cpu-baseline --frames 0 --clock-ramp 0.3"
P='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("%.3fM hyp/s  step %.4f ms render %.4f ms fk %.4f ms  frac %.4f" % (d["value"]/1e6, d["ms_per_step"], r["kernel_ms"], r["fk_kernel_ms"], r["frac"]))'
echo "default:                $($B | python -c "$P")"
echo "HP_NO_PERSIST=1:        $(HP_NO_PERSIST=1 $B | python -c "$P")"
for f in build_variants/*.so; do
  [ -e "$f" ] || continue
  echo "$f: $(HP_LIB=$f $B | python -c "$P")"
done
