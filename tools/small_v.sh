# per-sweep time at small V (config 2) with and without programmatic dependent launch
for g in 1e6 1e7 1e8; do
  for pdl in 1 0; do
    if [ $pdl = 0 ]; then export CAVI_NO_PDL=1; else unset CAVI_NO_PDL; fi
    timeout 300 python bench.py --genes $g --steps 200 --warmup 20 --no-e2e --no-cpu --no-converge 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('V=$g pdl=$pdl', round(d['value'],1), 'sweeps/s', round(d['ms_per_step']*1e3,2), 'us/sweep, pass', round(d['roofline']['kernel_ms']*1e3,2), 'us')"
  done
done
unset CAVI_NO_PDL
