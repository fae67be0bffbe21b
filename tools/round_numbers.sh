#!/bin/sh
# The numbers DESIGN.md quotes, in one call: K sweep (V=1e8, fp64), the fp32 streams, small V,
# EM, batched fits, the posterior sampler
P=${1:-r02}
bash tools/ksweep_dmma.sh 2 3 4 5 6 7 8 9 10 11 12 13 14 15 16 > gpurun_out/${P}_ksweep.txt 2>&1
for st in f32 f32m; do
  python bench.py --storage $st --no-e2e --no-cpu --no-converge 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$st N=4', round(d['value'],1), 'sweeps/s pass', round(r['kernel_ms'],4), 'ms', round(r['achieved']), 'GB/s')"
done > gpurun_out/${P}_fp32.txt
for g in 1e6 1e7; do
  python bench.py --genes $g --steps 400 --warmup 40 --no-e2e --no-cpu --no-converge 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('V=$g', round(d['value'],1), 'sweeps/s', round(d['ms_per_step']*1e3,2), 'us/sweep')"
done > gpurun_out/${P}_small_v.txt
python tools/bench_em.py --genes 1e6 1e8 > gpurun_out/${P}_em.txt 2>&1
python tools/bench_batched.py --fits 1e4 1e5 > gpurun_out/${P}_batched.txt 2>&1
python tools/bench_posterior.py > gpurun_out/${P}_posterior.txt 2>&1
cat gpurun_out/${P}_ksweep.txt gpurun_out/${P}_fp32.txt gpurun_out/${P}_small_v.txt
tail -3 gpurun_out/${P}_em.txt; tail -2 gpurun_out/${P}_batched.txt; tail -4 gpurun_out/${P}_posterior.txt
