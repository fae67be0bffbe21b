"""Time batched independent fits (BASELINE config 4: 1e4 fibroblast-shaped tissue samples,
V=56 genes, N=3 networks) through vb.vb_fit_many, one JSON line per batch size.

    python tools/bench_batched.py --fits 1e4 1e5
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
    p.add_argument("--fits", type=float, nargs="+", default=[1e4])
    p.add_argument("--genes", type=int, default=56)
    p.add_argument("--networks", type=int, default=3)
    p.add_argument("--reps", type=int, default=3)
    a = p.parse_args()
    from paper_2401_10068_b200 import model, vb

    hp = model.default_hyperparams(a.networks)
    for nf in a.fits:
        nf = int(nf)
        dd = model.regime(nf * a.genes, 56, a.networks)  # the reference test regime, generated on the GPU
        r, mu, D = dd.download()
        dd.close()
        dss = [model.Dataset(r=r[i * a.genes:(i + 1) * a.genes], mu=mu[i * a.genes:(i + 1) * a.genes],
                             D=D[i * a.genes:(i + 1) * a.genes], n_networks=a.networks) for i in range(nf)]
        vb.vb_fit_many(dss[: min(nf, 64)], hp)  # warm-up
        ts = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            out = vb.vb_fit_many(dss, hp)
            ts.append(time.perf_counter() - t0)
        iters = out.n_iter
        best = min(ts)
        # the device call alone (inputs pre-concatenated, outputs left in the C structs)
        import ctypes as C

        from paper_2401_10068_b200 import _lib

        offs = np.arange(nf + 1, dtype=np.int64) * a.genes
        rr, mm, DD = (np.ascontiguousarray(x[: nf * a.genes]) for x in (r, mu, D))
        states = (_lib.CvState * nf)()
        tr = np.empty((nf, 4, 300))
        hs, keep = _lib.hyper_struct(hp)
        tc = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            _lib.check(_lib.lib().cv_batched_fit(_lib.dptr(rr), _lib.dptr(mm), _lib.dptr(DD),
                                                 offs.ctypes.data_as(C.POINTER(C.c_int64)), nf, a.networks - 1,
                                                 C.byref(hs), 300, 1e-8, 1, 1e-10, 0, states, _lib.dptr(tr)))
            tc.append(time.perf_counter() - t0)
        print(json.dumps({"what": "vb_fit_many (config 4)", "fits": nf, "genes_per_fit": a.genes, "N": a.networks,
                          "wall_s": best, "fits_per_s": nf / best, "c_call_s": min(tc), "iters_mean": float(iters.mean()),
                          "iters_max": int(iters.max())}), flush=True)


if __name__ == "__main__":
    main()
