"""Parity of the CUDA engine with the reference (goldens) and the oracle -- needs a B200.

Tolerances (BASELINE.json north_star): fp64 path within 1e-9 relative with the
same iteration count; fp32-storage path within 1e-4.
"""

import numpy as np
import pytest

from golden_io import Golden, names
from oracle import cavi as ocavi
from oracle import philox

pytestmark = pytest.mark.gpu

RTOL = 1e-9


@pytest.fixture(scope="module")
def eng():
    from paper_2401_10068_b200 import model, vb

    return vb, model


def host_ds(model, g):
    r, mu, D = g.data()
    return model.Dataset(r=r, mu=mu, D=D, n_networks=D.shape[1] + 1)


def hyper(model, g):
    h = g.hyper
    return model.HyperParams(a0=h.a0, b0=h.b0, q0=h.q0, n0=h.n0, K0=h.K0, Lambda0=h.Lambda0)


def close(got, want, rtol=RTOL, what=""):
    got, want = np.asarray(got, float), np.asarray(want, float)
    scale = np.max(np.abs(want)) if want.size else 1.0
    np.testing.assert_allclose(got, want, rtol=rtol, atol=rtol * scale, err_msg=what)


@pytest.mark.parametrize("name", names("fit_"))
def test_fit_matches_reference_golden(eng, name):
    vb, model = eng
    g = Golden(name)
    ds, hp = host_ds(model, g), hyper(model, g)
    st, tr = vb.vb_fit(ds, hp, **g.fit_kw)
    assert len(tr) == int(g["n_iter"]), "iteration count to convergence must match the reference"
    if np.all(np.isnan(g["elbo"])):
        assert np.all(np.isnan(tr.elbo))
    else:
        np.testing.assert_allclose(tr.elbo, g["elbo"], rtol=RTOL, atol=0)
    for k in ("delta_k0k", "delta_rho", "delta_lam"):
        np.testing.assert_allclose(getattr(tr, k), g[k], rtol=RTOL, atol=1e-12, err_msg=k)
    assert st.a_rho == float(g["a_rho"])
    close(st.b_rho, g["b_rho"], what="b_rho")
    close(st.k0k, g["k0k"], what="k0k")
    close(st.lam0l_inv, g["lam0l_inv"], what="lam0l_inv")
    close(st.e_lam, g["e_lam"], what="e_lam")
    close(st.e_rho, g["e_rho"], what="e_rho")
    close(st.e_lamk, g["e_lamk"], what="e_lamk")
    idx = g["idx"]
    close(st.mu_beta[idx], g["mu_beta"], what="mu_beta")
    close(st.lam_beta[idx], g["lam_beta"], what="lam_beta")
    close(st.e_bbt[idx], g["e_bbt"], what="e_bbt")


@pytest.mark.parametrize("name", names("steps_"))
def test_steps_match_reference_golden(eng, name):
    vb, model = eng
    g = Golden(name)
    ds, hp = host_ds(model, g), hyper(model, g)
    st = vb.vb_init(ds, hp)
    idx = g["idx"]
    for i in range(len(g["elbo"])):
        if i:
            st = vb.vb_step(st, ds, hp)
        close(vb.vb_elbo(st, ds, hp), g["elbo"][i], what=f"elbo[{i}]")
        assert st.a_rho == g["a_rho"][i]
        close(st.b_rho, g["b_rho"][i], what=f"b_rho[{i}]")
        close(st.k0k, g["k0k"][i], what=f"k0k[{i}]")
        close(st.lam0l_inv, g["lam0l_inv"][i], what=f"lam0l_inv[{i}]")
        close(st.e_lam, g["e_lam"][i], what=f"e_lam[{i}]")
        close(st.mu_beta[idx], g["mu_beta"][i], what=f"mu_beta[{i}]")
        close(st.lam_beta[idx], g["lam_beta"][i], what=f"lam_beta[{i}]")
        close(st.e_bbt[idx], g["e_bbt"][i], what=f"e_bbt[{i}]")


@pytest.mark.parametrize("V,N,seed", [(5000, 3, 1), (20000, 4, 2026), (777, 2, 5), (3001, 9, 3), (1000, 16, 16)])
def test_generator_matches_oracle(eng, V, N, seed):
    vb, model = eng
    r0, mu0, D0, K, lam = philox.make_regime(V, seed, N)
    dd = model.regime(V, seed, N)
    r, mu, D = dd.download()
    np.testing.assert_array_equal(mu, mu0)  # profile codes are integer-exact
    np.testing.assert_array_equal(D, D0)
    np.testing.assert_allclose(r, r0, rtol=0, atol=4e-15 * max(1.0, np.abs(r0).max()))
    # shards of the same stream are the same genes
    lo = 64 * 4096 if V > 64 * 4096 else 0
    part = model.generate(seed, V - lo, N, K, lam, 100.0, gene_lo=lo, V_total=V)
    r2, mu2, D2 = part.download()
    np.testing.assert_array_equal(r2, r[lo:])


@pytest.mark.parametrize("N,V,iters", [(3, 4000, 40), (4, 50000, 25), (2, 10000, 30), (6, 3000, 15),
                                       (7, 40000, 10), (8, 3000, 10), (9, 2000, 8),  # register/DMMA boundary
                                       (12, 2000, 8), (16, 3000, 6)])
def test_fit_matches_direct_oracle(eng, N, V, iters):
    vb, model = eng
    r, mu, D, K, lam = philox.make_regime(V, 7, N)
    ds = model.Dataset(r=r, mu=mu, D=D, n_networks=N)
    st, tr = vb.vb_fit(ds, model.default_hyperparams(N), max_iter=iters)
    so, to = ocavi.fit(r, mu, D, ocavi.default_hyper(N), max_iter=iters)
    assert len(tr) == len(to.elbo)
    np.testing.assert_allclose(tr.elbo, to.elbo, rtol=RTOL, atol=0)
    close(st.k0k, so.k0k)
    close(st.lam0l_inv, so.lam0l_inv)
    close(st.b_rho, so.b_rho)


def test_device_dataset_equals_uploaded(eng):
    vb, model = eng
    dd = model.regime(30000, 11, 4)
    host = dd.to_host()
    hp = model.default_hyperparams(4)
    s1, t1 = vb.vb_fit(dd, hp, max_iter=20)
    s2, t2 = vb.vb_fit(host, hp, max_iter=20)
    assert np.array_equal(t1.elbo, t2.elbo)
    assert np.array_equal(s1.k0k, s2.k0k)


@pytest.mark.parametrize("N", [4, 7, 8])
def test_fp32_storage_within_1e4(eng, N):
    vb, model = eng
    dd64 = model.regime(200000, 3, N)
    dd32 = model.regime(200000, 3, N, storage="f32")
    hp = model.default_hyperparams(N)
    s64, t64 = vb.vb_fit(dd64, hp, max_iter=40, rel_tol=0.0)
    s32, t32 = vb.vb_fit(dd32, hp, max_iter=40, rel_tol=0.0)
    np.testing.assert_allclose(t32.elbo, t64.elbo, rtol=1e-4)
    close(s32.k0k, s64.k0k, rtol=1e-4)
    close(s32.lam0l_inv, s64.lam0l_inv, rtol=1e-4)
    close(s32.b_rho, s64.b_rho, rtol=1e-4)


@pytest.mark.parametrize("V,N", [(1_000_003, 4), (9_000_001, 4), (9_000_001, 8), (9_000_001, 13)])
def test_run_to_run_bit_identical(eng, V, N):
    """Dynamic chunk tickets, the reducer warp and the LL / acquire-release cascades never change a
    bit: every sum is the plan's fixed tree (4096- and 8192-gene chunks)."""
    vb, model = eng
    dd = model.regime(V, 5, N)
    hp = model.default_hyperparams(N)
    a, ta = vb.vb_fit(dd, hp, max_iter=10)
    b, tb = vb.vb_fit(dd, hp, max_iter=10)
    assert np.array_equal(ta.elbo, tb.elbo) and np.array_equal(a.lam0l_inv, b.lam0l_inv)


def test_batched_fits_match_reference_goldens(eng):
    """Config 4: many fibroblast-shaped fits in one launch == per-fit reference vb_fit."""
    vb, model = eng
    gs = [Golden(n) for n in names("fit_fibro56_")]
    datasets = [host_ds(model, g) for g in gs]
    hp = hyper(model, gs[0])
    res = vb.vb_fit_many(datasets * 3, hp)  # repeated datasets: independent warps, identical answers
    for i, (st, tr) in enumerate(res):
        g = gs[i % len(gs)]
        assert len(tr) == int(g["n_iter"])
        np.testing.assert_allclose(tr.elbo, g["elbo"], rtol=RTOL, atol=0)
        np.testing.assert_allclose(tr.delta_k0k, g["delta_k0k"], rtol=RTOL, atol=1e-12)
        close(st.k0k, g["k0k"])
        close(st.lam0l_inv, g["lam0l_inv"])
        close(st.b_rho, g["b_rho"])
        close(st.mu_beta[g["idx"]], g["mu_beta"])
    first, again = res[0], res[len(gs)]
    assert np.array_equal(first[1].elbo, again[1].elbo)


def test_batched_fits_mixed_sizes_match_single_fits(eng):
    vb, model = eng
    datasets, hp = [], model.default_hyperparams(3)
    for s, V in enumerate([56, 1, 5, 200, 33, 1000]):
        r, mu, D, _, _ = philox.make_regime(V, 100 + s, 3)
        datasets.append(model.Dataset(r=r, mu=mu, D=D, n_networks=3))
    res = vb.vb_fit_many(datasets, hp, max_iter=150)
    for ds, (st, tr) in zip(datasets, res):
        s1, t1 = vb.vb_fit(ds, hp, max_iter=150)
        assert len(tr) == len(t1)
        np.testing.assert_allclose(tr.elbo, t1.elbo, rtol=RTOL, atol=0)
        close(st.k0k, s1.k0k)
        close(st.lam0l_inv, s1.lam0l_inv)


def test_batched_result_sequence_semantics(eng):
    """vb_fit_many returns a lazy sequence: len, indexing (incl. negative), slices, n_iter."""
    vb, model = eng
    datasets = []
    for s in range(5):
        r, mu, D, _, _ = philox.make_regime(56, 100 + s, 3)
        datasets.append(model.Dataset(r=r, mu=mu, D=D, n_networks=3))
    res = vb.vb_fit_many(datasets, model.default_hyperparams(3), max_iter=40)
    assert len(res) == 5
    st_last, tr_last = res[-1]
    st4, tr4 = res[4]
    assert np.array_equal(st_last.k0k, st4.k0k) and np.array_equal(tr_last.elbo, tr4.elbo)
    assert [len(t) for _, t in res[1:3]] == [int(n) for n in res.n_iter[1:3]]
    with pytest.raises(IndexError):
        res[5]
    # per-gene fields materialise from the fit's own dataset
    assert res[2][0].mu_beta.shape == (56, 2)


def test_partitioned_fits_equal_one_batch(eng):
    """config 4 split over ranks (no collective): the ranks' slices reproduce one batch."""
    from paper_2401_10068_b200 import dist

    vb, model = eng
    datasets = []
    for s in range(11):
        r, mu, D, _, _ = philox.make_regime(56, 300 + s, 3)
        datasets.append(model.Dataset(r=r, mu=mu, D=D, n_networks=3))
    hp = model.default_hyperparams(3)
    whole = vb.vb_fit_many(datasets, hp, max_iter=60)
    for rank in range(4):
        lo, hi, part = dist.fit_many_partitioned(datasets, hp, rank=rank, world=4, device=0, max_iter=60)
        for i, (st, tr) in enumerate(part):
            sw, tw = whole[lo + i]
            assert np.array_equal(tr.elbo, tw.elbo) and np.array_equal(st.k0k, sw.k0k)


def test_dimension_limit_is_a_value_error(eng):
    """N <= 16 networks (d <= 15) on the device path; beyond that a clean ValueError."""
    vb, model = eng
    rng = np.random.default_rng(0)
    V, N = 50, 17
    D = rng.integers(0, 2, (V, N - 1)).astype(float)
    ds = model.Dataset(r=rng.standard_normal(V), mu=np.zeros(V), D=D, n_networks=N)
    hp = model.HyperParams(a0=0.5, b0=0.5, q0=0.001, n0=1, K0=np.full(N - 1, 1 / 3), Lambda0=100.0 * np.eye(N - 1))
    with pytest.raises(ValueError):
        vb.vb_fit(ds, hp, max_iter=3)


def test_em_on_fp32_storage_within_1e4(eng):
    """EM through the optional fp32 stream agrees with the fp64 stream to 1e-4."""
    from paper_2401_10068_b200 import em

    vb, model = eng
    hp = model.default_hyperparams(4)
    init = model.ModelParams(K=hp.K0, Lam=hp.Lambda0, rho=1.0)
    p64, t64 = em.em_fit(model.regime(200_000, 9, 4), init, max_iter=30, rel_tol=0.0)
    p32, t32 = em.em_fit(model.regime(200_000, 9, 4, storage="f32"), init, max_iter=30, rel_tol=0.0)
    np.testing.assert_allclose(t32.loglik, t64.loglik, rtol=1e-4)
    np.testing.assert_allclose(p32.K, p64.K, rtol=1e-4)
