"""Time EM point estimation: em.em_fit iterations/s on the GPU.

    python tools/bench_em.py --genes 1e6 1e8 [--reference-genes 1e5]

--reference-genes times the reference's tissuemix.em.em_fit per iteration on a host sample
(only where the reference is importable: this container, not the GPU box).
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
    p.add_argument("--networks", type=int, default=4)
    p.add_argument("--iters", type=int, default=200)
    p.add_argument("--reference-genes", type=float, default=0)
    a = p.parse_args()
    N = a.networks
    if a.reference_genes:
        sys.path.insert(0, "/root/reference/pkg/src")
        from tissuemix import em as rem
        from tissuemix import model as rmodel

        from oracle import philox  # the reference's own generator restated (input only)

        V = int(a.reference_genes)
        r, mu, D, _, _ = philox.make_regime(V, 2026, N)
        ds = rmodel.Dataset(r=r, mu=mu, D=D, n_networks=N)
        hp = rmodel.default_hyperparams(N)
        init = rmodel.ModelParams(K=hp.K0, Lam=hp.Lambda0, rho=1.0)
        t0 = time.perf_counter()
        _, tr = rem.em_fit(ds, init, max_iter=5, rel_tol=0.0)
        dt = (time.perf_counter() - t0) / len(tr)
        print(json.dumps({"what": "reference tissuemix.em.em_fit (1 core)", "V": V, "N": N, "s_per_iter": dt,
                          "iters_per_s_scaled_to_1e8": 1.0 / (dt * 1e8 / V)}))
        return
    from paper_2401_10068_b200 import em, model

    hp = model.default_hyperparams(N)
    for V in a.genes:
        V = int(V)
        dd = model.regime(V, 2026, N)
        init = model.ModelParams(K=hp.K0, Lam=hp.Lambda0, rho=1.0)
        em.em_fit(dd, init, max_iter=5, rel_tol=0.0)  # warm-up (graph capture)
        t0 = time.perf_counter()
        _, tr = em.em_fit(dd, init, max_iter=a.iters, rel_tol=0.0)
        dt = time.perf_counter() - t0
        print(json.dumps({"what": "em.em_fit (GPU, one fused pass per iteration)", "V": V, "N": N, "iters": len(tr),
                          "wall_s": dt, "iters_per_s": len(tr) / dt, "loglik": float(tr.loglik[-1])}), flush=True)


if __name__ == "__main__":
    main()
