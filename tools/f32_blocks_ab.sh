#!/bin/sh
# CTAs/SM on the fp32 streams (CAVI_F32_BLOCKS / CAVI_F32M_BLOCKS builds), V=1e8 N=4: f32 (fp64 math), f32m (fp32 math)
for lib in "$@"; do
  for st in f32 f32m; do
    CAVI_LIB=$lib python bench.py --storage $st --no-e2e --no-cpu --no-converge 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib $st', round(d['value'],1), 'sweeps/s, pass', round(d['roofline']['kernel_ms']*1e3,1), 'us =', round(d['roofline']['achieved']), 'GB/s')"
  done
done
