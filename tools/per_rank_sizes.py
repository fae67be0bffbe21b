"""One GPU at the per-rank sizes of the strong-scaling run (V = 1e8 over 8/4/2/1 GPUs): sweep
time against the HBM streaming floor (8(1+d) B/gene), i.e. the per-sweep fixed cost that caps
strong-scaling efficiency, and the efficiency it implies before any exchange cost:
eff(W) = t(1e8) / (W t(1e8 / W)).   python tools/per_rank_sizes.py [N]"""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N = int(sys.argv[1]) if len(sys.argv) > 1 else 4
peak = 6555.5
try:
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass
t = {}
for W in (8, 4, 2, 1):
    V = 1e8 / W
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--genes", str(V), "--networks", str(N),
                          "--steps", "400", "--warmup", "40", "--no-e2e", "--no-cpu", "--no-converge"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    d = json.loads(out.stdout.strip().splitlines()[-1])
    us = d["ms_per_step"] * 1e3
    floor = 8 * N * V / (peak * 1e9) * 1e6
    t[W] = us
    print(f"V={V:.3g} (rank of {W}): {us:.1f} us/sweep, pass alone {d['roofline']['kernel_ms'] * 1e3:.1f} us, "
          f"HBM floor {floor:.1f} us, fixed {us - floor:.1f} us", flush=True)
for W in (2, 4, 8):
    print(f"implied strong-scaling efficiency at {W} GPUs (no exchange cost): {t[1] / (W * t[W]):.3f}")
