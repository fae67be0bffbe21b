"""The fused multi-GPU exchange protocol (csrc/lsa.cuh), modelled on the CPU: W ranks as
threads with random delays run pass -> publish(s) / tail -> wait(s) -> read for many
sweeps over the same two-parity window layout (the device tags every word with its
sequence number, LL-style; the model keeps one tag per rank slot, which is the same
validity rule).  Asserts that every tail reads exactly
sweep s's partials from every rank (the double-buffer argument in lsa.cuh) and that the
sequence numbers stay in lock step.  (The device code itself is exercised by the GPU
tests; a world of >1 GPU is not available in this environment.)"""

import random
import threading
import time

import pytest


class Window:
    def __init__(self, world):
        self.data = [[[None] for _ in range(world)] for _ in range(2)]  # [parity][rank]
        self.flags = [[0] * world for _ in range(2)]
        self.lock = threading.Lock()


def run(world, sweeps, seed):
    rng = random.Random(seed)
    wins = [Window(world) for _ in range(world)]
    errors = []
    start_seq = 1  # the self-test consumed sequence 1

    def rank_main(r):
        seq = start_seq
        lrng = random.Random(seed * 31 + r)
        for _ in range(sweeps):
            s = seq + 1
            par = s & 1
            time.sleep(lrng.random() * 1e-4)  # the pass
            payload = (s, r)
            for p in range(world):  # data stores into every peer, then the flags
                with wins[p].lock:
                    wins[p].data[par][r][0] = payload
            for p in range(world):
                with wins[p].lock:
                    wins[p].flags[par][r] = s
            t0 = time.time()  # the tail: bounded wait on every flag, then read
            while True:
                with wins[r].lock:
                    if all(wins[r].flags[par][q] >= s for q in range(world)):
                        got = [wins[r].data[par][q][0] for q in range(world)]
                        break
                if time.time() - t0 > 5:
                    errors.append(f"rank {r} timed out at {s}")
                    return
                time.sleep(lrng.random() * 2e-5)
            if got != [(s, q) for q in range(world)]:
                errors.append(f"rank {r} sweep {s} read {got}")
                return
            seq = s

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return errors


@pytest.mark.parametrize("world", [2, 4, 8])
def test_two_parity_window_never_serves_a_stale_or_future_sweep(world):
    assert run(world, sweeps=200, seed=world) == []


def test_model_detects_a_single_buffer_race():
    """The model has teeth: with one slot per rank (no parity), fast ranks overwrite."""
    import inspect

    src = inspect.getsource(run).replace("par = s & 1", "par = 0")
    ns = dict(globals())
    exec(compile(src, "single_buffer", "exec"), ns)
    assert any(ns["run"](8, 200, seed) for seed in range(5))
