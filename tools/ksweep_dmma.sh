# K sweep of the fused pass at V=1e8 (config 5): one bench line per N
for N in "$@"; do
  timeout 300 python bench.py --networks $N --steps 30 --warmup 5 --no-e2e --no-cpu --no-converge > gpurun_out/ks_$N.json 2> gpurun_out/ks_$N.err
  python - "$N" <<'PY'
import json, sys
N = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ks_{N}.json").read().strip().splitlines()[-1])
    r = d["roofline"]
    print(f"N={N} sweeps/s={d['value']:.1f} ms/sweep={d['ms_per_step']:.3f} pass_ms={r['kernel_ms']:.3f} GB/s={r['achieved']:.0f} frac={r['frac']:.3f}")
except Exception as e:
    print("N", N, "failed", e, open(f"gpurun_out/ks_{N}.err").read()[-500:])
PY
done
