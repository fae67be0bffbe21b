"""Input recipes shared by tests/golden/make_kde_golden.py (run against the reference) and
tests/test_gpu_analysis.py (run against the drop-in).  Mirrors the reference's own
test_analysis.py cases (reference pkg/tests/test_analysis.py) plus posterior draws."""

import os

import numpy as np

CASES = {
    # name: recipe -> 1-d samples, optional bandwidth / grid / range
    "normal10k": {"seed": 0, "kind": "normal", "n": 10_000},
    "mixture5k": {"seed": 2, "kind": "mixture", "n": 5000, "grid": 2048},
    "oversmoothed100k": {"seed": 4, "kind": "shift2", "n": 100_000, "bw": 0.4},
    "perm400": {"seed": 5, "kind": "normal", "n": 400},
    "affine2k": {"seed": 6, "kind": "shift07", "n": 2000, "bw": 0.2, "grid": 1024},
    "bimodal2": {"kind": "fixed", "x": [-2.0, 2.0], "bw": 0.3, "grid": 1025, "lo": -4.0, "hi": 4.0},
    "constant4": {"kind": "fixed", "x": [3.25, 3.25, 3.25, 3.25], "bw": 0.5},
    "lognormal3k": {"seed": 12, "kind": "lognormal", "n": 3000},
}

SUMMARY_CASES = {
    "const_weights": {"kind": "const"},
    "std_normal100k": {"kind": "normal", "seed": 7, "n": 100_000},
    "lambda_mean": {"kind": "lambda", "seed": 8, "n": 300},
    "bw_explicit": {"kind": "normal", "seed": 9, "n": 5000, "d": 3, "bw": 0.05},
    "post_n3_v700k": {"kind": "post", "file": "post_n3_v700k.npz", "tile": 30},
    "post_n4_v200": {"kind": "post", "file": "post_n4_v200.npz", "tile": 1},
}


def inputs(c):
    if c["kind"] == "fixed":
        return np.array(c["x"], dtype=float)
    rng = np.random.default_rng(c["seed"])
    n = c["n"]
    if c["kind"] == "normal":
        return rng.standard_normal(n)
    if c["kind"] == "shift2":
        return 2.0 + rng.standard_normal(n)
    if c["kind"] == "shift07":
        return rng.standard_normal(n) + 0.7
    if c["kind"] == "mixture":
        return np.concatenate([rng.standard_normal(3000), 4 + 0.5 * rng.standard_normal(n - 3000)])
    if c["kind"] == "lognormal":
        return np.exp(0.5 * rng.standard_normal(n))
    raise ValueError(c)


def summary_inputs(c, golden_dir):
    if c["kind"] == "const":
        return {"K": np.tile([0.1, 0.3], (200, 1)), "rho": np.full(200, 7.0)}
    if c["kind"] == "normal":
        rng = np.random.default_rng(c["seed"])
        d = c.get("d", 1)
        return {"K": rng.standard_normal((c["n"], d)), "rho": np.abs(rng.standard_normal(c["n"])) + 0.5}
    if c["kind"] == "lambda":
        rng = np.random.default_rng(c["seed"])
        n = c["n"]
        return {"K": rng.standard_normal((n, 2)), "rho": np.abs(rng.standard_normal(n)) + 1.0,
                "Lambda": np.broadcast_to(np.eye(2), (n, 2, 2)).copy() + 0.01 * rng.standard_normal((n, 2, 2))}
    if c["kind"] == "post":
        z = np.load(os.path.join(golden_dir, c["file"]))
        t = c["tile"]
        # draws of the reference's own vb_posterior_sample (>= 100 needed): tiled
        return {"K": np.tile(z["K"], (t, 1)), "rho": np.tile(z["rho"], t), "Lambda": np.tile(z["Lambda"], (t, 1, 1))}
    raise ValueError(c)
