#!/bin/sh
# K sweep (V=1e8) of several library builds on the same box: tools/ksweep_ab.sh "N list" lib1 lib2 ...
NS=$1; shift
for lib in "$@"; do
  for N in $NS; do
    CAVI_LIB=$lib timeout 300 python bench.py --networks $N --steps 20 --warmup 5 --no-e2e --no-cpu --no-converge 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$lib N=$N', round(d['value'],1), 'sweeps/s pass', round(r['kernel_ms'],3), 'ms', round(r['achieved']), 'GB/s')"
  done
done
