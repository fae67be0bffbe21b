#!/bin/sh
# sustained-load sweep rate (400 timed sweeps at V=1e8: the power-capped regime of long fits)
# of several library builds on the same box: tools/sustained_ab.sh "N list" lib1 lib2 ...
NS=$1; shift
for rep in 1 2; do
  for lib in "$@"; do
    for N in $NS; do
      CAVI_LIB=$lib timeout 300 python bench.py --networks $N --steps 400 --warmup 40 --no-e2e --no-cpu --no-converge 2>/dev/null |
        python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib N=$N sustained', round(d['value'],1), 'sweeps/s', round(d['ms_per_step']*1e3,1), 'us/sweep, sm', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
    done
  done
done
