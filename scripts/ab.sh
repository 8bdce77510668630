#!/bin/bash
# A/B kernel variants: default build, env switches, and builds in build_variants/.
B="python bench.py --steps 100 --warmup 5 --no-fit --no-cpu-baseline --clock-ramp 0.3"
P='import json,sys; d=json.loads(sys.stdin.read()); print("%.3fM hyp/s  step %.4f ms kernel %.4f ms  frac %.4f" % (d["value"]/1e6, d["ms_per_step"], d["roofline"]["kernel_ms"], d["roofline"]["frac"]))'
echo "default:                $($B | python -c "$P")"
echo "HP_NO_PERSIST=1:        $(HP_NO_PERSIST=1 $B | python -c "$P")"
for f in build_variants/*.so; do
  [ -e "$f" ] || continue
  echo "$f: $(HP_LIB=$f $B | python -c "$P")"
done
