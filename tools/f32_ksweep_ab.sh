#!/bin/sh
# fp32-stream (fp64 math) sweep rate at V=1e8 for several N and library builds: tools/f32_ksweep_ab.sh "N list" lib1 lib2 ...
NS=$1; shift
for lib in "$@"; do
  for N in $NS; do
    CAVI_LIB=$lib timeout 300 python bench.py --storage f32 --networks $N --steps 20 --warmup 5 --no-e2e --no-cpu --no-converge 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$lib f32 N=$N', round(d['value'],1), 'sweeps/s pass', round(r['kernel_ms'],4), 'ms', round(r['achieved']), 'GB/s')"
  done
done
