"""Time vb_posterior_sample at the reference's CLI default of 1e4 draws.

    python tools/bench_posterior.py --genes 1e6 1e8 --draws 1000 10000

Each Wishart draw sums nu = n0 + V outer products of d-vectors of Philox normals (the
reference's construction, vb.py:357-393), so the work is ~ draws x V x d normals.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--genes", type=float, nargs="+", default=[1e6])
    p.add_argument("--draws", type=int, nargs="+", default=[1000])
    p.add_argument("--networks", type=int, default=4)
    a = p.parse_args()
    from paper_2401_10068_b200 import model, samplers, vb

    N = a.networks
    hp = model.default_hyperparams(N)
    for V in a.genes:
        V = int(V)
        dd = model.regime(min(V, 1_000_000), 3, N)  # a fitted state (its V only enters through nu)
        st, _ = vb.vb_fit(dd, hp, max_iter=50)
        for n in a.draws:
            vb.vb_posterior_sample(samplers.RngStream(1), st, hp, V, 2)  # warm-up
            t0 = time.perf_counter()
            out = vb.vb_posterior_sample(samplers.RngStream(7), st, hp, V, n)
            dt = time.perf_counter() - t0
            normals = float(n) * (V + hp.n0) * (N - 1)
            print(json.dumps({"what": "vb_posterior_sample", "V": V, "N": N, "draws": n, "wall_s": dt,
                              "draws_per_s": n / dt, "normals_per_s": normals / dt,
                              "rho_mean": float(np.mean(out["rho"]))}), flush=True)


if __name__ == "__main__":
    main()
