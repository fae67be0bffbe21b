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
         tissuemix.vb, numpy) on every host core, one process per core over its
         slice of the same dataset, W warm-up + K barrier-delimited timed sweeps
         (the whole 1e8 genes when that fits ~150 s, else a prefix, scaled).

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
NOMINAL_HBM_GBS = 7700.0  # B200 HBM3e, HGX figure (/opt/skills/guides/B200_PROFILING.md)
# pure-read ceiling measured on this GPU type: a bare 16-byte-load reduction over 3.2 GB
# (tools/read_bw.cu, profiles/r02f_read_bw_ceiling.txt) -- the bound a read stream can reach
READ_CEILING_GBS = 7251.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--genes", type=float, default=1e8)
    p.add_argument("--networks", type=int, default=4)
    p.add_argument("--storage", choices=["f64", "f32", "f32m"], default="f64",
                   help="f32: fp32 stream, fp64 math; f32m: fp32 stream and fp32 per-gene math (d <= 7)")
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


# ----------------------------------------------------------------------------- shared
def bench_config(V, N, storage, world=1):
    """The workload both arms report (identical dicts: the driver compares them)."""
    d = N - 1
    esz = 8 if storage == "f64" else 4
    nbytes = V * esz * (1 + d)
    return {"workload": f"CAVI sweep (vb_step + vb_elbo) over V={V:.0e} genes, N={N} networks (d={d}), "
                        f"seed-{SEED} synthetic dataset (K=0.2, Lambda=100 I, rho=100), {storage} "
                        + ("on 1 GPU" if world == 1 else f"sharded by octant over {world} GPUs"),
            "V": V, "N": N, "seed": SEED, "storage": storage,
            "l2": (f"inputs ({nbytes / 1e9:.2f} GB) larger than L2 (126 MB); no flush needed" if nbytes > 126e6 else
                   f"inputs ({nbytes / 1e6:.0f} MB) L2-resident by design (evict-last): the small-V latency "
                   f"regime, not an HBM measurement"),
            "parallelism": "single GPU" if world == 1 else f"dp{world} (gene shards)"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            names = [ln.split(":", 1)[1].strip() for ln in fh if ln.startswith("model name")]
        return f"{names[0]} x {len(names)} logical CPUs"
    except Exception:
        return "unknown"


# ----------------------------------------------------------------------------- CPU side
def _mem_available():
    try:
        with open("/proc/meminfo") as fh:
            for ln in fh:
                if ln.startswith("MemAvailable:"):
                    return int(ln.split()[1]) * 1024
    except Exception:
        pass
    return 16 << 30


def _ref_worker(args):
    """One host process: genes [lo, hi) of the seed-2026 dataset, the reference algorithm
    (oracle port of tissuemix.vb: vb_step then vb_elbo) once per barrier-delimited step."""
    lo, hi, V_total, N, n_steps, barrier, q = args
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:
        pass
    from oracle import cavi as ocavi  # the reference's algorithm restated (reported baseline only)
    from oracle import philox

    K, Lam, rho = truth(N)
    r, mu, D = philox.generate_slice(SEED, lo, hi, V_total, N, K, Lam, rho)
    hp = ocavi.default_hyper(N)
    st = ocavi.init(r, mu, D, hp)
    barrier.wait()
    for _ in range(n_steps):
        nw = ocavi.step(st, r, mu, D, hp)
        ocavi.elbo(nw, r, mu, D, hp)
        st = nw
        barrier.wait()
    q.put(0)


def cpu_reference(V_total, N, warmup, steps, budget_s, procs=None):
    """The reference's algorithm on every host core, one process per core (its own thread pool
    is slower than serial), each sweeping a contiguous slice of the dataset's
    first V_s genes; V_s = V_total unless (warmup + steps) full sweeps would exceed budget_s or
    40% of the host's free memory.  Every step is barrier-delimited; returns the mean wall
    time of the `steps` timed sweeps and V_s (full-V sweeps/s = V_s / V_total / wall)."""
    import multiprocessing as mp

    from oracle import cavi as ocavi
    from oracle import philox

    procs = procs or os.cpu_count() or 1
    K, Lam, rho = truth(N)
    Vp = 20480  # probe: per-gene cost of one sweep on one core
    r, mu, D = philox.generate(SEED, Vp, N, K, Lam, rho)
    hp = ocavi.default_hyper(N)
    st = ocavi.step(ocavi.init(r, mu, D, hp), r, mu, D, hp)
    t0 = time.perf_counter()
    ocavi.elbo(ocavi.step(st, r, mu, D, hp), r, mu, D, hp)
    per_gene = (time.perf_counter() - t0) / Vp
    unit = procs * 4096
    by_time = budget_s / max(1, warmup + steps) * procs / per_gene
    d = N - 1
    by_mem = 0.4 * _mem_available() / (12.0 * (2 * (2 * d * d + 2 * d) + 2 + d))  # two states + data, x1.5
    Vs = int(min(V_total, by_time, by_mem))
    Vs = V_total if Vs >= V_total else max(unit, Vs // unit * unit)
    bounds = [min(Vs, (Vs * k // procs) // 2 * 2) for k in range(procs + 1)]
    bounds[-1] = Vs
    ctx = mp.get_context("fork")
    barrier = ctx.Barrier(procs + 1)
    q = ctx.Queue()
    n_steps = warmup + steps
    ps = [ctx.Process(target=_ref_worker, args=((bounds[k], bounds[k + 1], V_total, N, n_steps, barrier, q),))
          for k in range(procs)]
    for p_ in ps:
        p_.start()
    barrier.wait()  # every slice generated and initialised
    marks = [time.perf_counter()]
    for _ in range(n_steps):
        barrier.wait()
        marks.append(time.perf_counter())
    for p_ in ps:
        q.get()
        p_.join()
    wall = (marks[-1] - marks[warmup]) / steps
    sample = (f"{'the whole dataset' if Vs == V_total else f'the first {Vs} of {V_total} genes'} split over "
              f"{procs} processes (one per core); per step every process runs vb_step + vb_elbo of the "
              f"reference algorithm (numpy oracle port of tissuemix.vb, 1024-gene chunks, 1 thread) on its "
              f"slice, steps barrier-delimited; {warmup} warm-up + {steps} timed steps"
              + ("" if Vs == V_total else f"; iters/s scaled by {Vs}/{V_total}")
              + f"; single core: {1.0 / (per_gene * V_total):.4g} full sweeps/s")
    return wall, Vs, procs, sample


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    V, N = int(args.genes), args.networks
    wall, Vs, cores, sample = cpu_reference(V, N, args.warmup, args.steps, budget_s=150.0)
    value = Vs / V / wall
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(V, N, args.storage, args.gpus),
        "sample_genes_per_step": Vs,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                         "cpu": cpu_model()},
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

        return dist.bench_main(args, METRIC, UNIT, clocks_cls=Clocks,
                               config=bench_config(int(args.genes), args.networks, args.storage, world))

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
        "dtype": {"f64": "f64", "f32": "f64 (fp32 storage)", "f32m": "f32 per gene, f64 sums (fp32 storage)"}[args.storage],
        "data": "synthetic",
        "config": bench_config(V, N, args.storage),
        "step": "one fused E-pass over the HBM-resident stream + the on-device K/Lambda/rho tail with the bound",
        "generate_s": round(gen_s, 3),
        "gpu_launches": int(nl.value),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_kind": peak_kind,
                     "peak_note": "MEASURED_PEAKS hbm_gbs is a copy (read+write) benchmark; this pass is a pure "
                                  "read stream, which the HBM serves faster: frac can exceed 1",
                     "peak_nominal": NOMINAL_HBM_GBS, "frac_nominal": achieved / NOMINAL_HBM_GBS,
                     "peak_read_measured": READ_CEILING_GBS, "frac_read": achieved / READ_CEILING_GBS,
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
        wall, Vs, cores, sample = cpu_reference(V, N, warmup=1, steps=2, budget_s=30.0)
        line["cpu_baseline"] = {"value": Vs / V / wall, "unit": UNIT, "cores": cores, "kind": "port",
                                "sample": sample, "cpu": cpu_model()}
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
    h2d, d2h = int(8 * V * (2 + d)), int(C.sizeof(_lib.CvState) + 4 * 8 * M)
    return {"value": M / wall, "unit": UNIT, "h2d_bytes_per_step": h2d // M, "d2h_bytes_per_step": d2h // M,
            "h2d_bytes_per_call": h2d, "d2h_bytes_per_call": d2h, "sweeps_per_call": M,
            "step": "one sweep; a call = H2D of r, mu, D + vb_init + the sweeps to the stop rule + D2H of the "
                    "state and trace, so the per-step bytes are the call's bytes / sweeps_per_call",
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
