"""Time analysis.summarize on posterior-shaped draws.

    python tools/bench_analysis.py --draws 1e4 1e5 1e6 [--reference]

Draws: K ~ N(0.3, 0.05^2) (n, d), rho ~ |N| + 50, Lambda (n, d, d); one JSON line per n.
--reference also times the reference's tissuemix.analysis.summarize on the same draws
(only where the reference is importable: this container, not the GPU box).
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def draws(n, d, seed=1):
    rng = np.random.default_rng(seed)
    return {"K": 0.3 + 0.05 * rng.standard_normal((n, d)), "rho": np.abs(rng.standard_normal(n)) + 50.0,
            "Lambda": 100.0 * np.eye(d) + rng.standard_normal((n, d, d))}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--draws", type=float, nargs="+", default=[1e4, 1e5, 1e6])
    p.add_argument("--d", type=int, default=2)
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--reference", action="store_true")
    a = p.parse_args()
    for n in a.draws:
        n = int(n)
        s = draws(n, a.d)
        out = {"what": "analysis.summarize", "draws": n, "d": a.d}
        if a.reference:
            sys.path.insert(0, "/root/reference/pkg/src")
            from tissuemix import analysis as ref

            t0 = time.perf_counter()
            ref.summarize(s)
            out["reference_s"] = time.perf_counter() - t0
        else:
            from paper_2401_10068_b200 import analysis

            analysis.summarize(s)  # warm-up (context, module load)
            ts = []
            for _ in range(a.reps):
                t0 = time.perf_counter()
                analysis.summarize(s)
                ts.append(time.perf_counter() - t0)
            out["gpu_s_best"] = min(ts)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
