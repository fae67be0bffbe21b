"""Multi-GPU CAVI: one process per GPU, genes sharded by octant, one NCCL
allgather of an n_stats(d)-double partial per sweep (96 bytes at d = 3).

The reference has no distributed mode (its "parallel" is a thread pool over
1024-gene chunks with a fixed-tree combine, reference linalg.py:238-255,
301-328); this module scales the same deterministic contract across GPUs:

* `plan` / `shard_ranges` -- the reduction plan every device shares:
  262144-gene groups (of 4096- or 8192-gene chunks, engine.cuh plan_chunk_genes),
  8 octants of whole groups.  Rank r of
  a world of 1/2/4/8 owns octants [8r/W, 8(r+1)/W), i.e. a contiguous gene
  range; its partial is the octant subtree the single-GPU tree would build,
  so totals -- and therefore every state, ELBO and stop decision -- are
  bit-identical for any world size.
* `Comm.bootstrap` -- NCCL communicator; the 128-byte unique id travels over
  torch.distributed (gloo is enough: plumbing, not the data path).
* `shard_generate` / `shard_upload` -- the rank's slice of a dataset in HBM.
* `bench_main` -- the N>1 leg of bench.py.

Launch: `python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N`.
"""

from __future__ import annotations

import ctypes as C
import json
import os
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib, model

CHUNK_GENES = 4096
GROUP_CHUNKS = 64
N_OCTANTS = 8
GROUP_GENES = CHUNK_GENES * GROUP_CHUNKS


@dataclass(frozen=True)
class Plan:
    V: int
    n_chunks: int
    n_groups: int
    groups_per_octant: int

    def octant_genes(self, o: int):
        per = self.groups_per_octant * GROUP_GENES
        lo = min(o * per, self.V)
        return lo, min(lo + per, self.V)


def plan(V: int) -> Plan:
    """The reduction plan of a V-gene dataset (same on every device and in csrc/cavi.cu)."""
    nc = max(1, -(-V // CHUNK_GENES))
    ng = -(-nc // GROUP_CHUNKS)
    return Plan(V, nc, ng, -(-ng // N_OCTANTS))


def shard_ranges(V: int, world: int):
    """[(gene_lo, gene_hi)] per rank: rank r owns octants [8r/world, 8(r+1)/world)."""
    if world not in (1, 2, 4, 8):
        raise ValueError("world size must be 1, 2, 4 or 8")
    p = plan(V)
    per = N_OCTANTS // world
    return [(p.octant_genes(r * per)[0], p.octant_genes(r * per + per - 1)[1]) for r in range(world)]


def world_info():
    """(rank, world, local_rank) from torchrun's environment (1 process if absent)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init_host_group():
    """torch.distributed process group for host-side plumbing (gloo; 127.0.0.1 rendezvous)."""
    import torch.distributed as td  # noqa: PLC0415

    if not td.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        td.init_process_group("gloo")
    return td


def share_unique_id(uid: bytes | None, td=None) -> bytes:
    """Rank 0's 128-byte NCCL unique id, delivered to every rank over the host group."""
    td = td or init_host_group()
    box = [uid if td.get_rank() == 0 else None]
    td.broadcast_object_list(box, src=0)
    return box[0]


class Comm:
    """An NCCL communicator over this process's GPU (handle to `cv_comm`)."""

    def __init__(self, handle: int, rank: int, world: int, device: int):
        self._h = C.c_void_p(handle)
        self.rank, self.world, self.device = rank, world, device
        self._fin = weakref.finalize(self, _lib.lib().cv_comm_destroy, self._h)

    @property
    def handle(self):
        return self._h

    @property
    def fused(self) -> bool:
        """True when the per-sweep exchange is fused into the pass (NVLink stores into the
        peers' NCCL symmetric windows); False: one ncclAllGather per sweep."""
        return bool(_lib.lib().cv_comm_fused(self._h))

    def drop_publish(self, ahead: int) -> None:
        """Fault injection for tests: skip this rank's publish `ahead` sweeps into the next
        shard call, so that call fails with PeerTimeoutError (cv_comm_drop_publish)."""
        _lib.check(_lib.lib().cv_comm_drop_publish(self._h, int(ahead)))

    @classmethod
    def bootstrap(cls, device: int | None = None, td=None) -> "Comm":
        td = td or init_host_group()
        rank, world = td.get_rank(), td.get_world_size()
        uid = None
        if rank == 0:
            buf = C.create_string_buffer(128)
            _lib.check(_lib.lib().cv_nccl_unique_id(buf))
            uid = buf.raw
        uid = share_unique_id(uid, td)
        device = _lib.default_device() if device is None else device
        h = C.c_void_p()
        _lib.check(_lib.lib().cv_comm_create(uid, rank, world, device, C.byref(h)))
        return cls(h.value, rank, world, device)


def attach(dd: model.DeviceDataset, comm: Comm) -> model.DeviceDataset:
    _lib.check(_lib.lib().cv_dataset_set_comm(dd.handle, comm.handle))
    dd.comm = comm  # keep the communicator alive as long as the shard
    return dd


def shard_generate(seed: int, V: int, N: int, K, Lam, rho: float, comm: Comm, storage: str = "f64"):
    """This rank's slice of generate(seed, V, N, K, Lam, rho), with the communicator attached."""
    lo, hi = shard_ranges(V, comm.world)[comm.rank]
    dd = model.generate(seed, hi - lo, N, K, Lam, rho, storage=storage, device=comm.device, gene_lo=lo, V_total=V)
    return attach(dd, comm)


def shard_upload(ds, comm: Comm, storage: str = "f64", V_total: int | None = None, gene_lo: int | None = None):
    """Upload this rank's slice of a host Dataset (the whole dataset, or just the slice with its gene_lo)."""
    if V_total is None:
        V_total = int(np.atleast_1d(ds.r).shape[0])
        lo, hi = shard_ranges(V_total, comm.world)[comm.rank]
        part = model.Dataset(r=ds.r[lo:hi], mu=ds.mu[lo:hi], D=np.atleast_2d(ds.D)[lo:hi], n_networks=ds.n_networks) \
            if hi > lo else None
    else:
        lo, part = gene_lo, ds
    if part is None:  # a rank without genes still takes part in every exchange
        d = np.atleast_2d(ds.D).shape[1]
        part = model.Dataset.__new__(model.Dataset)
        object.__setattr__(part, "r", np.zeros(0))
        object.__setattr__(part, "mu", np.zeros(0))
        object.__setattr__(part, "D", np.zeros((0, d)))
        object.__setattr__(part, "n_networks", ds.n_networks)
    dd = model.upload(part, storage=storage, device=comm.device, gene_lo=lo, V_total=V_total)
    return attach(dd, comm)


# ----------------------------------------------------------- independent fits (config 4)
def fit_ranges(n_fits: int, world: int):
    """Contiguous, balanced split of n_fits independent fits over `world` ranks."""
    return [(n_fits * r // world, n_fits * (r + 1) // world) for r in range(world)]


def fit_many_partitioned(datasets, hp, rank: int | None = None, world: int | None = None, **kw):
    """vb_fit_many over this rank's share of independent datasets (BASELINE config 4 across
    GPUs): no collective -- every fit is independent, so each rank fits its slice on its own
    GPU (LOCAL_RANK) and the caller gathers whatever it needs.  Returns (lo, hi, results)."""
    from . import vb  # noqa: PLC0415

    r0, w0, local = world_info()
    rank = r0 if rank is None else rank
    world = w0 if world is None else world
    datasets = list(datasets)
    lo, hi = fit_ranges(len(datasets), world)[rank]
    if hi == lo:
        return lo, hi, []
    return lo, hi, vb.vb_fit_many(datasets[lo:hi], hp, device=kw.pop("device", local), **kw)


# ---------------------------------------------------------------------------- bench leg
def bench_main(args, metric: str, unit: str, clocks_cls=None, config=None) -> int:
    """bench.py at N>1: strong scaling of the V-gene sweep over the ranks of torchrun.

    Device-timed sweeps (max over ranks), nvidia-smi clocks during them (rank 0's GPU),
    and the end-to-end public call at N GPUs: each rank uploads its shard from pinned
    host memory and runs vb.vb_fit on it with the communicator attached (max over ranks).
    """
    import torch  # noqa: PLC0415

    from . import vb  # noqa: PLC0415

    rank, world, local = world_info()
    os.environ["CAVI_DEVICE"] = str(local)
    if "MASTER_PORT" not in os.environ:  # not under torchrun: a world of one
        os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_PORT="29511")
    td = init_host_group()
    comm = Comm.bootstrap(device=local, td=td)
    V, N = int(args.genes), args.networks
    d = N - 1
    K, Lam, rho = np.full(d, 0.2), np.linalg.inv(0.01 * np.eye(d)), 100.0
    hp = model.default_hyperparams(N)
    shard = shard_generate(2026, V, N, K, Lam, rho, comm, storage=args.storage)
    st = vb.vb_init(shard, hp)
    hs, keep = _lib.hyper_struct(hp)
    ms_total, ms_kernel, nl = C.c_double(), C.c_double(), C.c_int32()
    td.barrier()
    clk = clocks_cls(local) if clocks_cls is not None else None
    if clk is not None:
        clk.__enter__()
    _lib.check(_lib.lib().cv_bench_sweeps(shard.handle, C.byref(hs), C.byref(st._cs), args.warmup, args.steps,
                                          C.byref(ms_total), C.byref(ms_kernel), C.byref(nl)))
    td.barrier()
    t = torch.tensor([ms_total.value, ms_kernel.value], dtype=torch.float64)
    td.all_reduce(t, op=td.ReduceOp.MAX)
    ms_step = float(t[0]) / args.steps
    if clk is not None:
        # keep the clocks sampler running over >= 1 s of the same sweeps (same count on every rank)
        soak = 0 if getattr(args, "profile", False) else max(0, int(1000.0 / max(ms_step, 1e-3)) - args.steps)
        if soak:
            a_, b_, c_ = C.c_double(), C.c_double(), C.c_int32()
            _lib.check(_lib.lib().cv_bench_sweeps(shard.handle, C.byref(hs), C.byref(st._cs), 0, min(soak, 20000),
                                                  C.byref(a_), C.byref(b_), C.byref(c_)))
        clk.__exit__(None, None, None)
    kern_s = float(t[1]) / args.steps / 1e3
    esz = 8 if args.storage == "f64" else 4
    peak = 6551.4
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as fh:
            peak = float(json.load(fh)["hbm_gbs"])
    except Exception:
        pass
    bytes_rank = max(hi - lo for lo, hi in shard_ranges(V, world)) * esz * (1 + d)
    achieved = bytes_rank / kern_s / 1e9
    e2e = None
    if not (getattr(args, "no_e2e", False) or getattr(args, "profile", False)):
        e2e = _e2e_sharded(args, shard, comm, td, hp, unit)
    if rank == 0:
        ns = d + d * (d + 1) // 2 + 3
        line = {
            "metric": metric, "value": 1000.0 / ms_step, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64" if args.storage == "f64" else "f64 (fp32 storage)",
            "data": "synthetic",
            "config": config or {"V": V, "N": N, "parallelism": f"dp{world} (gene shards)"},
            "exchange": f"per-sweep exchange of {ns} doubles: " + (
                "fused into the pass (NVLink stores into NCCL symmetric windows)" if comm.fused
                else "one ncclAllGather"),
            "gpu_launches": int(nl.value),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "per": "largest rank shard, max over ranks"},
        }
        if clk is not None:
            line["clocks"] = clk.summary()
        if e2e is not None:
            line["e2e"] = e2e
        print(json.dumps(line), flush=True)
    td.barrier()
    del shard
    return 0


def _e2e_sharded(args, shard, comm, td, hp, unit):
    """vb.vb_fit at N GPUs from host data: per call each rank uploads its pinned shard
    (H2D inside the timed region), fits with the communicator, reads the state back."""
    import gc  # noqa: PLC0415
    import statistics  # noqa: PLC0415
    import time  # noqa: PLC0415

    import torch  # noqa: PLC0415

    from . import vb  # noqa: PLC0415

    lo, _ = shard_ranges(shard.V_total, comm.world)[comm.rank]
    V, d = shard.V, shard.dim
    r, mu, D = _lib.pinned_empty((V,)), _lib.pinned_empty((V,)), _lib.pinned_empty((V, d))
    r0, mu0, D0 = shard.download()
    r[:], mu[:], D[:] = r0, mu0, D0
    del r0, mu0, D0
    kw = {} if args.e2e_sweeps <= 0 else {"max_iter": args.e2e_sweeps, "rel_tol": 0.0}
    times, sweeps = [], []
    for i in range(args.e2e_steps + 1):
        part = model.Dataset(r=r, mu=mu, D=D, n_networks=shard.n_networks)
        td.barrier()
        t0 = time.perf_counter()
        dd = shard_upload(part, comm, storage=args.storage, V_total=shard.V_total, gene_lo=lo)
        st, tr = vb.vb_fit(dd, hp, **kw)
        _ = (st.k0k, st.b_rho, tr.elbo[-1])
        wall = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
        td.all_reduce(wall, op=td.ReduceOp.MAX)
        if i:
            times.append(float(wall[0]))
            sweeps.append(len(tr))
        del dd, st, tr, part
        gc.collect()
    wall = statistics.median(times)
    M = int(statistics.median(sweeps))
    h2d, d2h = int(8 * shard.V_total * (2 + d)), int(comm.world * (C.sizeof(_lib.CvState) + 4 * 8 * M))
    return {"value": M / wall, "unit": unit, "h2d_bytes_per_step": h2d // M, "d2h_bytes_per_step": d2h // M,
            "h2d_bytes_per_call": h2d, "d2h_bytes_per_call": d2h, "sweeps_per_call": M,
            "call": "per rank: dist.shard_upload(Dataset(host shard, pinned)) + vb.vb_fit(shard, hp)"
                    + ("  [reference defaults]" if not kw else f", max_iter={M}, rel_tol=0"),
            "wall_s": wall}


__all__ = ["Comm", "Plan", "attach", "bench_main", "fit_many_partitioned", "fit_ranges", "init_host_group", "plan",
           "shard_generate", "shard_ranges", "shard_upload", "share_unique_id", "world_info"]
