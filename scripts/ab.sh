#!/bin/bash
# A/B the kernel variants in build_variants/ against the default build (bench kernel time).
B="python bench.py --steps 100 --warmup 5 --no-fit --no-cpu-baseline --clock-ramp 0.3"
echo "default: $($B | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["kernel_ms"], d["roofline"]["frac"])')"
for f in build_variants/*.so; do
  echo "$f: $(HP_LIB=$f $B | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["kernel_ms"], d["roofline"]["frac"])')"
done
