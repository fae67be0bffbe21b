#!/bin/sh
# small-V sweep time of several library builds on the same box: tools/smallv_ab.sh "V list" lib1 lib2 ...
VS=$1; shift
for lib in "$@"; do
  for V in $VS; do
    CAVI_LIB=$lib timeout 300 python bench.py --genes $V --steps 200 --warmup 20 --no-e2e --no-cpu --no-converge 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib V=$V', round(d['value'],1), 'sweeps/s', round(d['ms_per_step']*1e3,2), 'us/sweep')"
  done
done
