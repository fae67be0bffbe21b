"""Time batched independent fits (BASELINE config 4: 1e4 fibroblast-shaped tissue samples,
V=56 genes, N=3 networks), one JSON line per batch size:
  kernel_ms      the fit kernel alone (CUDA events, CAVI_BATCH_PROF)
  concat_wall_s  vb.vb_fit_concat on pre-concatenated host arrays (H2D + setup + kernel + n_iter)
  many_wall_s    vb.vb_fit_many on a list of Dataset objects (+ the concatenation)
  all_wall_s     vb_fit_many + copying every state and trace to the host

    python tools/bench_batched.py --fits 1e4 1e5
"""

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)


def kernel_ms(nf, genes, networks):
    """The fit kernel's event time, from a child process with CAVI_BATCH_PROF set."""
    code = (f"import sys; sys.path.insert(0, {ROOT!r})\n"
            "import numpy as np\nfrom paper_2401_10068_b200 import model, vb\n"
            f"dd = model.regime({nf} * {genes}, 56, {networks}); r, mu, D = dd.download()\n"
            f"off = np.arange({nf} + 1, dtype=np.int64) * {genes}\n"
            f"hp = model.default_hyperparams({networks})\n"
            "for _ in range(3): vb.vb_fit_concat(r, mu, D, off, hp)\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         env=dict(os.environ, CAVI_BATCH_PROF="1"))
    ms = [float(l.split(" in ")[1].split()[0]) for l in out.stderr.splitlines() if l.startswith("batched_fit_kernel")]
    return min(ms) if ms else None


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--fits", type=float, nargs="+", default=[1e4])
    p.add_argument("--genes", type=int, default=56)
    p.add_argument("--networks", type=int, default=3)
    p.add_argument("--reps", type=int, default=5)
    a = p.parse_args()
    from paper_2401_10068_b200 import model, vb

    hp = model.default_hyperparams(a.networks)
    for nf in a.fits:
        nf = int(nf)
        dd = model.regime(nf * a.genes, 56, a.networks)  # the reference test regime, generated on the GPU
        r, mu, D = dd.download()
        dd.close()
        off = np.arange(nf + 1, dtype=np.int64) * a.genes
        dss = [model.Dataset(r=r[i * a.genes:(i + 1) * a.genes], mu=mu[i * a.genes:(i + 1) * a.genes],
                             D=D[i * a.genes:(i + 1) * a.genes], n_networks=a.networks) for i in range(nf)]
        vb.vb_fit_many(dss[: min(nf, 64)], hp)  # warm-up

        def best(fn):
            ts = []
            for _ in range(a.reps):
                t0 = time.perf_counter()
                out = fn()
                ts.append(time.perf_counter() - t0)
                del out
            return min(ts)

        t_concat = best(lambda: vb.vb_fit_concat(r, mu, D, off, hp))
        t_many = best(lambda: vb.vb_fit_many(dss, hp))

        def everything():
            res = vb.vb_fit_many(dss, hp)
            return res.states(), res.traces()

        t_all = best(everything)
        res = vb.vb_fit_many(dss, hp)
        iters = res.n_iter
        print(json.dumps({"what": "batched independent fits (config 4)", "fits": nf, "genes_per_fit": a.genes,
                          "N": a.networks, "kernel_ms": kernel_ms(nf, a.genes, a.networks),
                          "concat_wall_s": t_concat, "many_wall_s": t_many, "all_wall_s": t_all,
                          "fits_per_s_many": nf / t_many, "iters_mean": float(iters.mean()),
                          "iters_max": int(iters.max()), "fit_sweeps": int(iters.sum())}), flush=True)


if __name__ == "__main__":
    main()
