"""The reference's own VB test suite (reference pkg/tests/test_vb.py), run against the drop-in.

Each test cites the reference test it restates.  Datasets come from the
oracle's bit-exact restatement of the reference generator.
"""

import numpy as np
import pytest

from oracle import philox

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    from paper_2401_10068_b200 import linalg, model, vb

    class NS:
        pass

    ns = NS()
    ns.vb, ns.model, ns.linalg = vb, model, linalg
    return ns


def make_dataset(E, V, seed=0, N=3):
    r, mu, D, K, lam = philox.make_regime(V, seed, N)
    return E.model.Dataset(r=r, mu=mu, D=D, n_networks=N)


def fit_small(E, V=120, seed=21, **kw):
    ds = make_dataset(E, V, seed)
    hp = E.model.default_hyperparams(3)
    st, tr = E.vb.vb_fit(ds, hp, **kw)
    return ds, hp, st, tr


def test_means_start_at_k0(E):  # test_vb.py:17-22
    ds = make_dataset(E, 50, 1)
    st = E.vb.vb_init(ds, E.model.default_hyperparams(3))
    np.testing.assert_allclose(st.mu_beta, np.full((50, 2), 1.0 / 3.0))
    np.testing.assert_allclose(st.k0k, [1.0 / 3.0, 1.0 / 3.0])
    assert st.a_rho == 0.5 and st.b_rho == 0.5  # test_vb.py:24-28


def test_precisions_start_at_lambda0(E):  # test_vb.py:30-36
    ds = make_dataset(E, 5, 2)
    hp = E.model.default_hyperparams(3)
    st = E.vb.vb_init(ds, hp)
    for i in range(5):
        np.testing.assert_array_equal(st.lam_beta[i], hp.Lambda0)
    np.testing.assert_array_equal(st.lam0l_inv, hp.Lambda0)


def test_dim_mismatch_rejected(E):  # test_vb.py:38-41
    ds = make_dataset(E, 5, 2)
    with pytest.raises(ValueError, match="dim"):
        E.vb.vb_init(ds, E.model.default_hyperparams(4))


def test_a_rho_is_data_size_only(E):  # test_vb.py:45-52
    ds = make_dataset(E, 4000, 3)
    hp = E.model.default_hyperparams(3)
    st = E.vb.vb_init(ds, hp)
    for _ in range(3):
        st = E.vb.vb_step(st, ds, hp)
        assert st.a_rho == 0.5 + 2000.0


def test_beta_precision_formula(E):  # test_vb.py:54-72
    ds = make_dataset(E, 30, 4)
    hp = E.model.default_hyperparams(3)
    st = E.vb.vb_init(ds, hp)
    e_lam_used = (hp.n0 + ds.V) * np.linalg.inv(st.lam0l_inv)
    sigma = np.linalg.inv(st.lam_beta)
    e_bbt = np.einsum("vi,vj->vij", st.mu_beta, st.mu_beta) + sigma
    rm = ds.r - ds.mu
    b_rho = hp.b0 + 0.5 * float(np.sum(rm ** 2 - 2 * rm * (ds.D @ hp.K0) + np.einsum("vi,vij,vj->v", ds.D, e_bbt, ds.D)))
    e_rho_used = (hp.a0 + 0.5 * ds.V) / b_rho
    new = E.vb.vb_step(st, ds, hp)
    want = e_lam_used + e_rho_used * np.einsum("vi,vj->vij", ds.D, ds.D)
    np.testing.assert_allclose(new.lam_beta, want, rtol=1e-12)
    assert new.b_rho == pytest.approx(b_rho, rel=1e-12)


def test_weight_mean_update_arithmetic(E):  # test_vb.py:74-81
    ds = make_dataset(E, 1, 5)
    hp = E.model.default_hyperparams(3)
    new = E.vb.vb_step(E.vb.vb_init(ds, hp), ds, hp)
    want = (new.mu_beta[0] + hp.q0 * hp.K0) / (1 + hp.q0)
    np.testing.assert_allclose(new.k0k, want, rtol=1e-12)


def test_posterior_beta_covariance_spd(E):  # test_vb.py:90-95
    ds, hp, st, _ = fit_small(E, max_iter=20)
    sigma = np.linalg.inv(st.lam_beta)
    cov = st.e_bbt - np.einsum("vi,vj->vij", st.e_beta, st.e_beta)
    np.testing.assert_allclose(cov, sigma, atol=1e-10)
    np.linalg.cholesky(cov + 1e-13 * np.eye(2))


def test_permutation_invariance(E):  # test_vb.py:97-107
    ds = make_dataset(E, 257, 6)
    hp = E.model.default_hyperparams(3)
    perm = np.random.default_rng(0).permutation(ds.V)
    ds_p = E.model.Dataset(r=ds.r[perm], mu=ds.mu[perm], D=ds.D[perm], n_networks=3)
    s1, _ = E.vb.vb_fit(ds, hp, max_iter=40)
    s2, _ = E.vb.vb_fit(ds_p, hp, max_iter=40)
    np.testing.assert_allclose(s1.k0k, s2.k0k, rtol=1e-9)
    np.testing.assert_allclose(s1.b_rho, s2.b_rho, rtol=1e-9)
    np.testing.assert_allclose(s1.lam0l_inv, s2.lam0l_inv, rtol=1e-9)


def test_monotone_along_fit(E):  # test_vb.py:110-113
    _, _, _, tr = fit_small(E, V=300, seed=7, max_iter=150)
    e = tr.elbo
    assert np.all(np.diff(e) >= -1e-9 * np.abs(e[1:]))


def test_converged_state_is_fixed_point(E):  # test_vb.py:146-152
    ds, hp, st, _ = fit_small(E, V=150, seed=11, max_iter=2500, rel_tol=1e-12)
    e0 = E.vb.vb_elbo(st, ds, hp)
    st2 = E.vb.vb_step(st, ds, hp)
    e1 = E.vb.vb_elbo(st2, ds, hp)
    assert abs(e1 - e0) < 1e-10 * abs(e0)


def test_max_iter_one(E):  # test_vb.py:155-157
    _, _, _, tr = fit_small(E, max_iter=1)
    assert len(tr) == 1
    with pytest.raises(ValueError):
        fit_small(E, max_iter=0)


def test_decoupled_flat_profile_limit(E):  # test_vb.py:159-171
    V = 80
    mu = np.ones(V)
    D = np.zeros((V, 2))
    r = philox.synth(philox.Stream(12), [0.1, 0.3], np.linalg.inv(E.model.REFERENCE_LAMBDA_INV), 100.0, mu, D)
    ds = E.model.Dataset(r=r, mu=mu, D=D, n_networks=3)
    hp = E.model.default_hyperparams(3)
    st, _ = E.vb.vb_fit(ds, hp, max_iter=500, rel_tol=1e-12)
    np.testing.assert_allclose(st.k0k, hp.K0, atol=1e-6)
    np.testing.assert_allclose(st.mu_beta, np.broadcast_to(hp.K0, (V, 2)), atol=1e-6)
    want_b = hp.b0 + 0.5 * float(np.sum((ds.r - ds.mu) ** 2))
    assert st.b_rho == pytest.approx(want_b, rel=1e-9)


def test_param_delta_fallback_stopping(E):  # test_vb.py:173-178
    ds = make_dataset(E, 60, 13)
    hp = E.model.default_hyperparams(3)
    st, tr = E.vb.vb_fit(ds, hp, max_iter=4000, compute_elbo=False, param_tol=1e-11)
    assert len(tr) < 4000
    assert np.all(np.isnan(tr.elbo))


def test_serial_parallel_bit_identical(E):  # test_vb.py:180-188
    ds = make_dataset(E, 1500, 14)
    hp = E.model.default_hyperparams(3)
    s1, t1 = E.vb.vb_fit(ds, hp, max_iter=30, plan=E.linalg.ExecPlan(workers=1))
    s2, t2 = E.vb.vb_fit(ds, hp, max_iter=30, plan=E.linalg.ExecPlan(workers=3))
    assert np.array_equal(s1.k0k, s2.k0k)
    assert np.array_equal(s1.lam0l_inv, s2.lam0l_inv)
    assert np.array_equal(np.asarray(t1.elbo), np.asarray(t2.elbo))
    assert s1.b_rho == s2.b_rho


def test_improper_q_lambda_raises_numeric_error(E):  # vb.py:299-301
    # d = 15 with V = 3 genes: nu = n0 + V = 4 <= d - 1
    ds = make_dataset(E, 3, 1, N=16)
    hp = E.model.default_hyperparams(16)
    st = E.vb.vb_step(E.vb.vb_init(ds, hp), ds, hp)  # a sweep itself is fine
    with pytest.raises(E.linalg.NumericError, match="improper"):
        E.vb.vb_elbo(st, ds, hp)
    with pytest.raises(E.linalg.NumericError, match="improper"):
        E.vb.vb_fit(ds, hp, max_iter=5)
    st, tr = E.vb.vb_fit(ds, hp, max_iter=5, compute_elbo=False)  # no bound, no error (vb.py:344-347)
    assert len(tr) == 5


def test_nonfinite_profile_raises(E):  # linalg.py:67-69 via gemm_batched (vb.py:150)
    ds = make_dataset(E, 10, 1)
    D = ds.D.copy()
    D[3, 1] = np.nan
    bad = E.model.Dataset(r=ds.r, mu=ds.mu, D=D, n_networks=3)
    with pytest.raises(FloatingPointError):
        E.vb.vb_fit(bad, E.model.default_hyperparams(3), max_iter=3)


def test_install_is_importable(E):
    assert callable(E.vb.install)
