"""Time the dataset file path: native writer and GPU reader.

    python tools/bench_ingest.py --rows 1e7 --networks 4 [--reference-rows 1e5]

Generates the config-3 regime on the GPU, writes it as the reference's CSV format
(ingest.write_dataset_csv), reads it back with ingest.load_dataset_csv (file -> HBM ->
parsed dataset), checks the round trip bit-exactly, and prints one JSON line.
--reference-rows times the reference's own reader (cli.read_dataset_csv) on a prefix
of the same file when the reference is importable (this container, not the GPU box).
"""

import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--rows", type=float, default=1e7)
    p.add_argument("--networks", type=int, default=4)
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--dir", default=None)
    p.add_argument("--reference-rows", type=float, default=0)
    a = p.parse_args()
    import torch

    from paper_2401_10068_b200 import ingest, model

    V, N = int(a.rows), a.networks
    dd = model.generate(2026, V, N, np.full(N - 1, 0.2), 100.0 * np.eye(N - 1), 100.0)
    r, mu, D = dd.download()
    dd.close()
    d = tempfile.mkdtemp(dir=a.dir)
    path = os.path.join(d, "ds.csv")
    t0 = time.perf_counter()
    ingest.write_dataset_csv(path, model.Dataset(r=r, mu=mu, D=D, n_networks=N))
    t_write = time.perf_counter() - t0
    size = os.path.getsize(path)
    times = []
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x = ingest.load_dataset_csv(path)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        if len(times) < a.reps:
            x.close()
    r2, mu2, D2 = x.download()
    ok = bool(np.array_equal(r2.view(np.uint64), r.view(np.uint64)) and np.array_equal(mu2, mu) and
              np.array_equal(D2.view(np.uint64), D.view(np.uint64)))
    best = min(times)
    out = {"what": "dataset CSV -> HBM dataset (ingest.load_dataset_csv)", "rows": V, "N": N, "file_bytes": size,
           "load_s_best": best, "load_s_all": times, "rows_per_s": V / best, "file_GB_per_s": size / best / 1e9,
           "write_s": t_write, "write_rows_per_s": V / t_write, "round_trip_bit_exact": ok,
           "host_cores": os.cpu_count()}
    if a.reference_rows:
        try:
            sys.path.insert(0, "/root/reference/pkg/src")
            from tissuemix import cli
        except ImportError:
            out["reference"] = "unavailable"
        else:
            n = int(a.reference_rows)
            sub = os.path.join(d, "sub.csv")
            with open(path) as src, open(sub, "w") as dst:
                for i, line in enumerate(src):
                    if i > n:
                        break
                    dst.write(line)
            t0 = time.perf_counter()
            cli.read_dataset_csv(sub)
            tr = time.perf_counter() - t0
            out["reference"] = {"rows": n, "s": tr, "rows_per_s": n / tr}
    print(json.dumps(out))
    os.remove(path)


if __name__ == "__main__":
    main()


def bench_npz(V=100_000_000, N=4):
    """Binary dataset file -> HBM (load_dataset_npz) at V genes."""
    import tempfile

    from paper_2401_10068_b200 import ingest, model

    dd = model.regime(V, 2026, N)
    with tempfile.TemporaryDirectory() as tmp:
        p = os.path.join(tmp, "ds.npz")
        t = time.time()
        ingest.write_dataset_npz(p, dd)
        tw = time.time() - t
        size = os.path.getsize(p)
        loads = []
        for _ in range(3):
            t = time.time()
            d2 = ingest.load_dataset_npz(p)
            loads.append(time.time() - t)
            same = np.array_equal(d2.stream_x(), dd.stream_x())
            d2.close()
    print(json.dumps({"what": "dataset .npz -> HBM dataset (ingest.load_dataset_npz)", "rows": V, "N": N,
                      "file_bytes": size, "write_s": tw, "load_s_best": min(loads), "load_s_all": loads,
                      "file_GB_per_s": size / min(loads) / 1e9, "stream_bit_exact": bool(same)}), flush=True)
