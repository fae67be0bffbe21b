"""The CPU legs of bench.py (the cpu_baseline and the `--impl reference` arm) run here:
the reference algorithm on host processes over slices of the same dataset."""

import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_generate_slice_is_the_dataset_slice():
    """Each reference-arm process sweeps its own genes of the one seed-2026 dataset."""
    from oracle import philox

    K, L = np.full(3, 0.2), 100.0 * np.eye(3)
    r, mu, D = philox.generate(2026, 60001, 4, K, L, 100.0)
    for lo, hi in [(0, 4096), (4096, 30000), (30000, 60001)]:
        a = philox.generate_slice(2026, lo, hi, 60001, 4, K, L, 100.0)
        assert np.array_equal(a[0], r[lo:hi]) and np.array_equal(a[1], mu[lo:hi]) and np.array_equal(a[2], D[lo:hi])


def test_cpu_reference_runs_the_sweeps_it_reports():
    import bench

    wall, Vs, cores, sample = bench.cpu_reference(10**6, 4, warmup=1, steps=2, budget_s=3.0, procs=2)
    assert cores == 2 and wall > 0 and 0 < Vs <= 10**6 and Vs % (2 * 4096) in (0, 10**6 % (2 * 4096))
    assert "2 processes" in sample and "1 warm-up + 2 timed steps" in sample


def test_reference_arm_prints_one_json_line_with_the_gpu_arms_config():
    import bench

    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--genes", "2e6"], capture_output=True, text=True, timeout=600, env=env,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["cores"] >= 1
    assert line["steps"] == 2 and line["warmup"] == 1
    assert line["config"] == bench.bench_config(2 * 10**6, 4, "f64")
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    # the value is what the timed steps ran: sample genes / V per wall second
    assert abs(line["value"] - line["sample_genes_per_step"] / 2e6 / (line["ms_per_step"] / 1e3)) < 1e-9 * line["value"]
