"""Pin the CPU oracle against the reference's own known answers and golden fixtures (no GPU)."""

import numpy as np
import pytest

from oracle import cavi, fused, philox
from golden_io import Golden, names

# Random123 philox4x32-10 known-answer vectors, as the reference's tests hold them
# (reference tests/test_samplers.py:24-36).
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


def test_philox_known_answers():
    for ctr, key, want in KAT:
        got = philox.philox_block(np.array(ctr, dtype=np.uint64), np.array(key, dtype=np.uint64))
        assert tuple(int(v) for v in got) == want


def test_stream_consumes_whole_blocks():
    # reference tests/test_samplers.py:62-68
    s = philox.Stream(5, 0)
    first = np.concatenate([s.uniforms(3), s.uniforms(5)])
    joined = philox.Stream(5, 0).uniforms(8)
    np.testing.assert_array_equal(first[:3], joined[:3])
    assert s.block == 2 + 3
    u = philox.Stream(1, 2).uniforms(10_000)
    assert np.all(u > 0.0) and np.all(u <= 1.0)


@pytest.mark.parametrize("name", names())
def test_golden_dataset_rebuilds_bit_exact(name):
    Golden(name).data(check=True)


FAST_FITS = [n for n in names("fit_") if n != "fit_n3_v4000_t1"]


def _cmp_fit(g, st, trace_elbo, n_iter, rtol):
    assert n_iter == int(g["n_iter"])
    ref = g["elbo"]
    if np.all(np.isnan(ref)):
        assert np.all(np.isnan(trace_elbo))
    else:
        np.testing.assert_allclose(trace_elbo, ref, rtol=rtol, atol=0)
    np.testing.assert_allclose(st.k0k, g["k0k"], rtol=rtol, atol=0)
    np.testing.assert_allclose(st.b_rho, g["b_rho"], rtol=rtol, atol=0)
    np.testing.assert_allclose(st.lam0l_inv, g["lam0l_inv"], rtol=rtol, atol=rtol * np.abs(g["lam0l_inv"]).max())
    np.testing.assert_allclose(st.e_lam, g["e_lam"], rtol=rtol, atol=rtol * np.abs(g["e_lam"]).max())


@pytest.mark.parametrize("name", FAST_FITS)
def test_direct_oracle_matches_reference_bit_exact(name):
    g = Golden(name)
    r, mu, D = g.data()
    st, tr = cavi.fit(r, mu, D, g.hyper, **g.fit_kw)
    _cmp_fit(g, st, tr.elbo, len(tr.elbo), rtol=0)
    idx = g["idx"]
    np.testing.assert_array_equal(st.mu_beta[idx], g["mu_beta"])
    np.testing.assert_array_equal(st.lam_beta[idx], g["lam_beta"])
    np.testing.assert_array_equal(st.e_bbt[idx], g["e_bbt"])


@pytest.mark.parametrize("name", names("fit_"))
def test_fused_restatement_matches_reference(name):
    """The kernel's executable spec: 1e-9 relative and the same iteration count."""
    g = Golden(name)
    r, mu, D = g.data()
    st, tr, n = fused.fit(r, mu, D, g.hyper, **g.fit_kw)
    _cmp_fit(g, st, tr["elbo"], n, rtol=1e-9)
    for k in ("delta_k0k", "delta_rho", "delta_lam"):
        np.testing.assert_allclose(tr[k], g[k], rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("name", names("steps_"))
def test_direct_oracle_steps_bit_exact(name):
    g = Golden(name)
    r, mu, D = g.data()
    st = cavi.init(r, mu, D, g.hyper)
    idx = g["idx"]
    for i in range(len(g["elbo"])):
        if i:
            st = cavi.step(st, r, mu, D, g.hyper)
        assert cavi.elbo(st, r, mu, D, g.hyper) == g["elbo"][i]
        assert st.b_rho == g["b_rho"][i]
        np.testing.assert_array_equal(st.k0k, g["k0k"][i])
        np.testing.assert_array_equal(st.mu_beta[idx], g["mu_beta"][i])


@pytest.mark.parametrize("name", names("post_"))
def test_posterior_oracle_bit_exact(name):
    """vb_posterior_sample restated (vb.py:357-393, samplers.py:220-261): same draws, same stream end."""
    g = Golden(name)
    s = philox.Stream(int(g["seed"]), int(g["stream_id"]), int(g["pre_block"]))
    out = cavi.posterior_sample(s, float(g["a_rho"]), float(g["b_rho"]), g["k0k"], g["lam0l_inv"], g.hyper,
                                int(g["V"]), int(g["n"]))
    assert s.block == int(g["end_block"])
    for k in ("K", "Lambda", "rho"):
        np.testing.assert_array_equal(out[k], g[k])


@pytest.mark.parametrize("name", names("em_"))
def test_em_oracle_bit_exact(name):
    """em_fit / em_step restated (em.py:44-124, model.py:273-287) == the reference's own numbers."""
    from oracle import em

    g = Golden(name)
    r, mu, D = g.data()
    (K, Lam, rho), ll, ks, rhos = em.em_fit(r, mu, D, g["init_K"], g["init_Lam"], float(g["init_rho"]), **g.fit_kw)
    assert len(ll) == int(g["n_iter"])
    np.testing.assert_array_equal(ll, g["loglik"])
    np.testing.assert_array_equal(K, g["K"])
    np.testing.assert_array_equal(Lam, g["Lam"])
    assert rho == float(g["rho"])
    K1, L1, r1, Sig, M, S = em.em_step(r, mu, D, g["init_K"], g["init_Lam"], float(g["init_rho"]))
    np.testing.assert_array_equal(K1, g["step_K"])
    np.testing.assert_array_equal(S[g["idx"]], g["step_S"])


@pytest.mark.parametrize("world", [2, 4, 8])
def test_octant_plan_is_world_size_invariant(world):
    r, mu, D, _, _ = philox.make_regime(5000, 3, 4)
    # stretch the plan so every octant holds genes: 300 chunks of 4096 genes would be 1.2M genes;
    # instead exercise it by tiling the small dataset.
    reps = 1 + (fused.CHUNK_GENES * fused.GROUP_CHUNKS * 9) // 5000
    x = np.tile(r - mu, reps)[: fused.CHUNK_GENES * fused.GROUP_CHUNKS * 9 + 777]
    Dx = np.tile(D, (reps, 1))[: x.shape[0]]
    hp = cavi.default_hyper(4)
    gen, st = fused.init(hp, x.shape[0])
    gen, a, b = fused.sweep_generator(st, 123.0, hp, x.shape[0])
    whole = fused.full_stats(x, Dx, gen)
    parts = [fused.rank_partial(x, Dx, gen, rk, world) for rk in range(world)]
    assert np.array_equal(fused.combine(parts), whole)
    spans = fused.shard_ranges(x.shape[0], world)
    assert spans[0][0] == 0 and spans[-1][1] == x.shape[0]
    assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
