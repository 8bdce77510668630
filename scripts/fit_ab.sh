#!/bin/bash
# A/B of the C3 fit across library builds: the default build and every build_variants/*.so
# (HP_LIB), run twice in alternation.  Usage (under gpurun): bash scripts/fit_ab.sh
for i in 1 2; do
  echo "default: $(python scripts/fit_time.py 2>&1 | grep C3)"
  for f in build_variants/*.so; do
    [ -e "$f" ] || continue
    echo "$f: $(HP_LIB=$f python scripts/fit_time.py 2>&1 | grep C3)"
  done
done
