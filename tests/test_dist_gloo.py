"""Multi-rank host logic on CPU (gloo, world_size 2): the shard planner, the NCCL-id
bootstrap over the host group, and the GPU-count invariance of the reduction plan
(rank partials combined by the top of the octant tree == the single-rank total, bit-exactly)."""

import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_planner_matches_oracle_plan():
    from oracle import fused
    from paper_2401_10068_b200 import dist

    for V in [1, 5, 4095, 4096, 4097, 262144, 262145, 3_000_001, 100_000_000, 1_000_000_000]:
        for world in (1, 2, 4, 8):
            assert dist.shard_ranges(V, world) == fused.shard_ranges(V, world)
        p, q = dist.plan(V), fused.make_plan(V)
        assert (p.n_chunks, p.n_groups, p.groups_per_octant) == (q.n_chunks, q.n_groups, q.groups_per_octant)
    spans = dist.shard_ranges(10**8, 8)
    assert spans[0][0] == 0 and spans[-1][1] == 10**8
    assert all(lo % dist.GROUP_GENES == 0 for lo, _ in spans)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as td

    from oracle import cavi, fused, philox
    from paper_2401_10068_b200 import dist

    td.init_process_group("gloo", rank=rank, world_size=world)
    # 1) NCCL unique-id bootstrap over the host group (bytes from rank 0 reach every rank)
    uid = bytes(range(128)) if rank == 0 else None
    got = dist.share_unique_id(uid, td)
    # 2) rank partials of one sweep's statistics on this rank's shard (planner of the product)
    V = 64 * 4096 * 3 + 12345  # several groups, ragged tail
    r, mu, D, _, _ = philox.make_regime(70000, 11, 4)
    x = np.resize(r - mu, V)
    Dx = np.resize(D, (V, 3))
    hp = cavi.default_hyper(4)
    gen, st = fused.init(hp, V)
    gen, a, b = fused.sweep_generator(st, 321.0, hp, V)
    lo, hi = dist.shard_ranges(V, world)[rank]
    octs = fused.local_stats(x[lo:hi], Dx[lo:hi], gen, lo, V)
    per = fused.N_OCTANTS // world
    part = fused.tree8(octs[rank * per:(rank + 1) * per])
    parts = [None] * world
    td.all_gather_object(parts, part)
    combined = fused.combine(parts)
    whole = fused.full_stats(x, Dx, gen)
    np.save(os.path.join(out_dir, f"r{rank}.npy"),
            np.array([got == bytes(range(128)), np.array_equal(combined, whole)], dtype=bool))
    td.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_gloo_exchange_is_bit_identical(tmp_path, world):
    import torch.multiprocessing as mp

    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    for rk in range(world):
        ok = np.load(tmp_path / f"r{rk}.npy")
        assert ok[0], "NCCL unique id did not reach every rank"
        assert ok[1], "rank partials combined by the octant tree differ from the single-rank total"


@pytest.mark.parametrize("n,world", [(10000, 8), (7, 8), (1, 2), (12345, 3)])
def test_fit_ranges_partition_all_fits(n, world):
    """config 4 across GPUs: every fit on exactly one rank, balanced to within one fit."""
    from paper_2401_10068_b200 import dist

    spans = dist.fit_ranges(n, world)
    assert spans[0][0] == 0 and spans[-1][1] == n
    assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
    sizes = [hi - lo for lo, hi in spans]
    assert max(sizes) - min(sizes) <= 1
