#!/bin/bash
# A/B of the library builds in paper_2005_07068_b200/variants/ against the default build.
B="python bench.py --steps 100 --warmup 5 --no-fit --no-cpu-baseline --frames 0 --clock-ramp 0.3"
P='import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("%.3fM hyp/s  step %.4f ms render %.4f ms fk %.4f ms  frac %.4f" % (d["value"]/1e6, d["ms_per_step"], r["kernel_ms"], r["fk_kernel_ms"], r["frac"]))'
echo "default: $($B | python -c "$P")"
for f in paper_2005_07068_b200/variants/*.so; do
  [ -e "$f" ] || continue
  echo "$f: $(HP_LIB=$f $B | python -c "$P")"
done
