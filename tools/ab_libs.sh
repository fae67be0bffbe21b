#!/bin/sh
# A/B of library builds on the SAME box (boxes differ by several % in HBM speed):
#   tools/ab_libs.sh libA.so libB.so ...   -> per-rank sweep times, interleaved twice
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $lib (rep $rep)"
    CAVI_LIB=$lib python tools/per_rank_sizes.py 2>&1 | head -4
  done
done
