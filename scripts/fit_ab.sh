#!/bin/bash
# A/B of the fit path (C3 ms/frame) for the default build and build_variants/*.so.
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --frames 0 --track-frames 20 --fit-seeds 10 --clock-ramp 0.3"
P='import json,sys; d=json.loads(sys.stdin.read()); print("%.3fM hyp/s  fit %.3f ms/frame  track %.3f ms/frame" % (d["value"]/1e6, d["pso_fit"]["ms_per_frame"], d["tracking"]["ms_per_frame"]))'
echo "default: $($B | python -c "$P")"
for f in build_variants/*.so; do
  [ -e "$f" ] || continue
  echo "$f: $(HP_LIB=$f $B | python -c "$P")"
done
