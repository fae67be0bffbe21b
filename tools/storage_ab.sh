# fp64 vs fp32 storage at V=1e8 and 1e6 (config 2 / 3), one line each
for st in f64 f32; do for g in 1e8 1e6; do
  timeout 300 python bench.py --genes $g --storage $st --steps 100 --warmup 10 --no-e2e --no-cpu --no-converge 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$st V=$g', round(d['value'],1), 'sweeps/s pass', round(d['roofline']['kernel_ms']*1e3,1), 'us frac', round(d['roofline']['frac'],3))"
done; done
