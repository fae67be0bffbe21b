"""The CPU legs of bench.py (the cpu_baseline and the `--impl reference` arm) run here:
the reference algorithm on host processes over gene slices, scaled to the full V."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_cpu_reference_parallel_scales_a_bounded_sample():
    import bench

    per_sweep, cores, sample = bench.cpu_reference_parallel(10**8, 4, procs=2, steps=1, target_s=0.3)
    assert cores == 2 and per_sweep > 0
    assert "2 processes" in sample and "scaled by 100000000/" in sample


def test_reference_arm_prints_one_json_line():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--genes", "2e6"], capture_output=True, text=True, timeout=600, env=env,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0
