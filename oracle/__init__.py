"""CPU oracle for the CAVI hot path -- TEST INFRASTRUCTURE ONLY.

This package is a plain-numpy restatement of the reference `tissuemix`
algorithm for the coordinate-ascent VB path (vb.py / linalg.py / model.py /
samplers.py under /root/reference/pkg/src/tissuemix).  It exists to *check*
the CUDA engine, never to stand in for it:

* only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu-baseline /
  `--impl reference` leg may import it;
* the product package `paper_2401_10068_b200` never imports it and fails
  loudly when its CUDA library is missing.

Parity pin: the restatement is checked bit-for-bit / to <=1e-12 against
golden vectors produced by running the reference itself in the build
container (`tests/golden/make_golden.py`, fixtures in `tests/golden/`), and
against the reference's own Philox known-answer vectors
(tests/test_samplers.py:24-36 in the reference).

Modules
-------
philox   -- Philox4x32-10 streams and the synthetic generator (a16/a17).
cavi     -- direct per-gene restatement of vb_init/vb_step/vb_elbo/vb_fit.
fused    -- the single-pass rank-1 restatement with the
            exact chunk/group/octant reduction plan the device kernel uses;
            the executable spec of the kernel and of the multi-rank combine.
"""
