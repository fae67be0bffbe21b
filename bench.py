#!/usr/bin/env python
"""CAVI sweep throughput at the north-star configuration (BASELINE.json).

metric : CAVI iters/sec at N=1e8 measurements, K=4 subpopulations (d = 3), fp64
step   : one CAVI sweep (vb_step + vb_elbo) over the whole synthetic dataset:
         one fused streaming pass of the 1e8-gene measurement stream + the
         on-device tail (K/Lambda block, bound, stop rule)
value  : sweeps / s with the data resident in HBM, CUDA-event timed
e2e    : the same metric through the public API, vb_fit(host Dataset) with
         the H2D upload of r, mu, D (from pinned memory) and the D2H of the
         result inside the timed region: iters / s = sweeps / wall of the call
reference arm (--impl reference): the reference algorithm (oracle port of
         tissuemix.vb, numpy, host cores) timed on a bounded sample of the
         same workload and scaled to the full 1e8 genes.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CAVI iters/sec at N=1e8,K=4 (1/2/4/8 GPU, % HBM peak); time to ELBO convergence"
UNIT = "iters/s"
SEED = 2026


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--genes", type=float, default=1e8)
    p.add_argument("--networks", type=int, default=4)
    p.add_argument("--storage", choices=["f64", "f32"], default="f64")
    p.add_argument("--e2e-sweeps", type=int, default=0, help="0: the reference's vb_fit defaults")
    p.add_argument("--e2e-steps", type=int, default=2)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--profile", action="store_true", help="under ncu: no clock soak, no e2e/cpu legs")
    p.add_argument("--force-dist", action="store_true", help="use the sharded NCCL path even at N=1")
    p.add_argument("--converge", action="store_true", help="time vb_fit to ELBO convergence (default at N=1)")
    p.add_argument("--no-converge", action="store_true", help="skip the time-to-convergence leg")
    return p.parse_args()


def truth(N):
    return np.full(N - 1, 0.2), np.linalg.inv(0.01 * np.eye(N - 1)), 100.0  # conftest.py:18-22 regime


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi clocks/throttle sampler running during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def traffic_per_launch():
    """dram bytes per pass launch from the committed ncu --set full capture summary (or None)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_pass_kernel.json")) as fh:
            return json.load(fh).get("dram_bytes_per_launch")
    except Exception:
        return None


# ----------------------------------------------------------------------------- CPU side
def cpu_reference_sample(V_total, N, target_s=1.0, min_genes=20000):
    """One sweep (vb_step + vb_elbo) of the reference algorithm (oracle port) on a sample.

    Returns a closure timing one sweep, plus the sample description.
    """
    from oracle import cavi as ocavi  # the reference's algorithm restated (reported baseline only)
    from oracle import philox

    K, Lam, rho = truth(N)
    # probe: size the sample so one sweep takes ~target_s
    Vs = min_genes
    r, mu, D = philox.generate(SEED, Vs, N, K, Lam, rho)
    hp = ocavi.default_hyper(N)
    st = ocavi.init(r, mu, D, hp)
    t0 = time.perf_counter()
    ocavi.elbo(ocavi.step(st, r, mu, D, hp), r, mu, D, hp)
    per_gene = (time.perf_counter() - t0) / Vs
    Vs = int(min(V_total, max(min_genes, target_s / max(per_gene, 1e-9))))
    Vs = (Vs // 1024) * 1024 or min_genes
    r, mu, D = philox.generate(SEED, Vs, N, K, Lam, rho)
    state = {"st": ocavi.init(r, mu, D, hp)}

    def sweep():
        t = time.perf_counter()
        nw = ocavi.step(state["st"], r, mu, D, hp)
        ocavi.elbo(nw, r, mu, D, hp)
        state["st"] = nw
        return time.perf_counter() - t

    sample = (f"first {Vs} genes of the seed-{SEED} N={N} dataset; one vb_step+vb_elbo of the reference "
              f"algorithm (numpy oracle port of tissuemix.vb, 1024-gene chunks, 1 thread) per step, "
              f"scaled by {V_total}/{Vs}")
    return sweep, Vs, sample


def _cpu_worker(args):
    """One worker process: its own gene slice, barrier-started sweeps (see cpu_reference_parallel)."""
    V_slice, N, steps, barrier, out = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import cavi as ocavi
    from oracle import philox

    K, Lam, rho = truth(N)
    r, mu, D = philox.generate(SEED, V_slice, N, K, Lam, rho)
    hp = ocavi.default_hyper(N)
    st = ocavi.init(r, mu, D, hp)
    st = ocavi.step(st, r, mu, D, hp)  # warm-up
    barrier.wait()
    for _ in range(steps):
        nw = ocavi.step(st, r, mu, D, hp)
        ocavi.elbo(nw, r, mu, D, hp)
        st = nw
    barrier.wait()
    out.put(0)


def cpu_reference_parallel(V_total, N, procs=None, steps=2, target_s=2.0):
    """The reference algorithm on every host core: `procs` processes each sweep a 1/procs
    slice of a bounded sample (the work of one sweep is a sum over genes), started
    together; seconds per full-V sweep = wall per sweep x V_total / sample."""
    import multiprocessing as mp

    procs = procs or os.cpu_count() or 1
    sweep, Vs1, _ = cpu_reference_sample(V_total, N, target_s=target_s / 2)
    per_gene = statistics.median([sweep() for _ in range(2)]) / Vs1
    V_slice = max(1024, int(target_s / per_gene / 1024) * 1024)
    ctx = mp.get_context("fork")
    barrier = ctx.Barrier(procs + 1)
    q = ctx.Queue()
    ps = [ctx.Process(target=_cpu_worker, args=((V_slice, N, steps, barrier, q),)) for _ in range(procs)]
    for p_ in ps:
        p_.start()
    barrier.wait()
    t0 = time.perf_counter()
    barrier.wait()
    wall = (time.perf_counter() - t0) / steps
    for p_ in ps:
        q.get()
        p_.join()
    Vs = V_slice * procs
    sample = (f"{procs} processes x the first {V_slice} genes of the seed-{SEED} N={N} dataset; vb_step+vb_elbo "
              f"of the reference algorithm (numpy oracle port of tissuemix.vb), {steps} sweeps started together, "
              f"wall per sweep scaled by {V_total}/{Vs}; single core: {1.0 / (per_gene * V_total):.4g} sweeps/s")
    return wall * V_total / Vs, procs, sample


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    V = int(args.genes)
    per = []
    for _ in range(max(1, min(args.steps, 3))):
        t, cores, sample = cpu_reference_parallel(V, args.networks)
        per.append(t)
    per_sweep_full = statistics.median(per)
    value = 1.0 / per_sweep_full
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_sweep_full * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"CAVI sweep, V={V:.0e} genes, N={args.networks} networks (K={args.networks}), "
                               f"fp64, reference algorithm on host cores (bounded sample)",
                   "V": V, "N": args.networks},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU side
def run_ours(args):
    import ctypes as C

    from paper_2401_10068_b200 import _lib, model, vb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != 1 or args.gpus != 1 or args.force_dist:
        from paper_2401_10068_b200 import dist  # noqa: PLC0415

        return dist.bench_main(args, METRIC, UNIT, clocks_cls=Clocks)

    dev = _lib.default_device()
    V, N = int(args.genes), args.networks
    d = N - 1
    K, Lam, rho = truth(N)
    hp = model.default_hyperparams(N)
    t0 = time.time()
    dd = model.generate(SEED, V, N, K, Lam, rho, storage=args.storage, device=dev)
    gen_s = time.time() - t0
    st = vb.vb_init(dd, hp)
    hs, keep = _lib.hyper_struct(hp)
    ms_total, ms_kernel, nl = C.c_double(), C.c_double(), C.c_int32()
    with Clocks(dev) as clk:
        _lib.check(_lib.lib().cv_bench_sweeps(dd.handle, C.byref(hs), C.byref(st._cs), args.warmup, args.steps,
                                              C.byref(ms_total), C.byref(ms_kernel), C.byref(nl)))
        # keep sampling clocks for >=1 s of the same sweeps if the timed region was shorter
        soak = 0 if args.profile else max(0, int(1000.0 / max(ms_total.value / args.steps, 1e-3)) - args.steps)
        if soak:
            a, b, c = C.c_double(), C.c_double(), C.c_int32()
            _lib.check(_lib.lib().cv_bench_sweeps(dd.handle, C.byref(hs), C.byref(st._cs), 0, min(soak, 20000),
                                                  C.byref(a), C.byref(b), C.byref(c)))
    ms_step = ms_total.value / args.steps
    value = 1000.0 / ms_step
    esz = 8 if args.storage == "f64" else 4
    bytes_sweep = V * esz * (1 + d)  # x = r - mu and D: the stream one pass reads
    kern_s = ms_kernel.value / args.steps / 1e3
    achieved = bytes_sweep / kern_s / 1e9
    peak, peak_kind = peaks()
    # the committed ncu capture is of the default workload (V=1e8, d=3, fp64); other configs: no capture
    traffic = traffic_per_launch() if (V, N, args.storage) == (int(1e8), 4, "f64") else None

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if args.storage == "f64" else "f64 (fp32 storage)", "data": "synthetic",
        "config": {"workload": f"CAVI sweep (fused E-pass + on-device K/Lambda/rho tail + ELBO), V={V:.0e} genes, "
                               f"N={N} networks (d={d}), {args.storage} storage, inputs resident in HBM",
                   "V": V, "N": N, "seed": SEED, "storage": args.storage,
                   "l2": (f"inputs ({bytes_sweep / 1e9:.2f} GB) larger than L2 (126 MB); no flush needed"
                          if bytes_sweep > 126e6 else
                          f"inputs ({bytes_sweep / 1e6:.0f} MB) L2-resident by design (evict-last): the "
                          f"small-V latency regime, not an HBM measurement"),
                   "generate_s": round(gen_s, 3), "parallelism": "single GPU"},
        "gpu_launches": int(nl.value),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_kind": peak_kind,
                     "bytes_per_launch": bytes_sweep, "kernel_ms": kern_s * 1e3},
        "clocks": clk.summary(),
    }

    # the metric's second half: wall time of vb_fit to the reference's stop rule (rel_tol 1e-8)
    # on the resident dataset; on by default at N=1 (about 23 s at V=1e8)
    if (args.converge or args.gpus == 1) and not (args.no_converge or args.profile):
        t = time.time()
        s_conv, tr = vb.vb_fit(dd, hp, max_iter=100000, rel_tol=1e-8)
        line["converge"] = {"wall_s": time.time() - t, "iterations": len(tr), "final_elbo": float(tr.elbo[-1]),
                            "call": "vb.vb_fit(resident dataset, hp, max_iter=100000, rel_tol=1e-8)"}

    if not (args.no_e2e or args.profile):
        line["e2e"] = e2e(args, dd, hp)
    del dd
    if not (args.no_cpu or args.profile):
        t, cores, sample = cpu_reference_parallel(V, N)
        line["cpu_baseline"] = {"value": 1.0 / t, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}
    print(json.dumps(line), flush=True)
    return 0


def e2e(args, dd, hp):
    """The public call a user makes, on host data: vb.vb_fit(Dataset(host arrays), hp) with the
    reference's defaults (max_iter=300, rel_tol=1e-8; vb.py:312-320).  Timed per call: H2D of
    r, mu, D from pinned memory, the on-device transform, vb_init + every sweep to the stop
    rule, and the D2H of the state and trace.  iters/s = sweeps the call ran / wall time."""
    import ctypes as C
    import gc

    from paper_2401_10068_b200 import _lib, model, vb

    V, d = dd.V, dd.dim
    r = _lib.pinned_empty((V,))
    mu = _lib.pinned_empty((V,))
    D = _lib.pinned_empty((V, d))
    r0, mu0, D0 = dd.download()
    r[:], mu[:], D[:] = r0, mu0, D0
    del r0, mu0, D0
    kw = {} if args.e2e_sweeps <= 0 else {"max_iter": args.e2e_sweeps, "rel_tol": 0.0}
    times, sweeps = [], []
    for i in range(args.e2e_steps + 1):
        ds = model.Dataset(r=r, mu=mu, D=D, n_networks=dd.n_networks)  # a fresh object: uploaded again
        t = time.perf_counter()
        st, tr = vb.vb_fit(ds, hp, **kw)
        _ = (st.k0k, st.b_rho, tr.elbo[-1])
        dt = time.perf_counter() - t
        if i:
            times.append(dt)
            sweeps.append(len(tr))
        del ds, st, tr
        gc.collect()
    wall = statistics.median(times)
    M = int(statistics.median(sweeps))
    return {"value": M / wall, "unit": UNIT, "h2d_bytes_per_step": int(8 * V * (2 + d)),
            "d2h_bytes_per_step": int(C.sizeof(_lib.CvState) + 4 * 8 * M), "sweeps_per_call": M,
            "call": "paper_2401_10068_b200.vb.vb_fit(Dataset(host, pinned), hp" + (
                ")  [reference defaults: max_iter=300, rel_tol=1e-8]" if not kw else f", max_iter={M}, rel_tol=0)"),
            "wall_s": wall}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
