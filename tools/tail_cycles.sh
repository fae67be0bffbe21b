#!/bin/sh
# clock64 phase stamps of the sweep tail (build: make BUILD=build/prof LIB=paper_2401_10068_b200/libcavi_prof.so
# EXTRA=-DCAVI_TAIL_PROF), one line per N
for n in ${@:-2 4 7 10 16}; do
  printf "N=%s: " $n
  CAVI_LIB=${PROF_LIB:-paper_2401_10068_b200/libcavi_prof.so} CAVI_TAIL_PROF_PRINT=1 timeout 300 python bench.py --networks $n \
    --genes 1e6 --steps 20 --warmup 5 --no-e2e --no-cpu --no-converge 2>&1 >/dev/null | grep "tail cycles"
done
