"""EM on the fused pass (paper_2401_10068_b200.em) against the reference's em_* goldens and
the reference's own EM test suite (reference pkg/tests/test_em.py), restated.

Goldens: the log-likelihood trace to 1e-9 relative with the same iteration count, the
final (K, Lambda, rho), and one em_step's Sigma / M / S on a fixed gene subset.
"""

import numpy as np
import pytest

from golden_io import Golden, names
from oracle import em as oracle_em
from oracle import philox

pytestmark = pytest.mark.gpu

RTOL = 1e-9


@pytest.fixture(scope="module")
def E():
    from paper_2401_10068_b200 import em, linalg, model

    class NS:
        pass

    ns = NS()
    ns.em, ns.model, ns.linalg = em, model, linalg
    return ns


def host_ds(E, r, mu, D):
    return E.model.Dataset(r=r, mu=mu, D=D, n_networks=D.shape[1] + 1)


def make_dataset(E, V, seed=0, N=3):
    r, mu, D, K, lam = philox.make_regime(V, seed, N)
    return host_ds(E, r, mu, D), E.model.ModelParams(K=K, Lam=lam, rho=100.0)


def init_params(E, hp):  # test_em.py:11-12
    return E.model.ModelParams(K=hp.K0, Lam=hp.Lambda0, rho=hp.a0 / hp.b0)


def state(E, p):
    return E.em.EmState(params=p, Sigma=None, M=None, S=None)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("name", names("em_"))
def test_em_fit_matches_reference_golden(E, name):
    g = Golden(name)
    ds = host_ds(E, *g.data())
    init = E.model.ModelParams(K=g["init_K"], Lam=g["init_Lam"], rho=float(g["init_rho"]))
    p, tr = E.em.em_fit(ds, init, **g.fit_kw)
    assert len(tr) == int(g["n_iter"])
    np.testing.assert_allclose(tr.loglik, g["loglik"], rtol=RTOL, atol=0)
    # parameters drift along long flat ridges (Lambda is weakly identified); the
    # log-likelihood pins the iteration, the parameters are checked more loosely.
    assert rel(p.K, g["K"]) < 1e-6
    assert abs(p.rho - float(g["rho"])) < 1e-6 * float(g["rho"])
    assert rel(p.Lam, g["Lam"]) < 1e-5
    assert rel(tr.K, g["tr_K"]) < 1e-6
    np.testing.assert_allclose(tr.rho, g["tr_rho"], rtol=1e-6)


@pytest.mark.parametrize("name", names("em_"))
def test_em_step_matches_reference_golden(E, name):
    g = Golden(name)
    ds = host_ds(E, *g.data())
    init = E.model.ModelParams(K=g["init_K"], Lam=g["init_Lam"], rho=float(g["init_rho"]))
    new = E.em.em_step(state(E, init), ds)
    np.testing.assert_allclose(new.params.K, g["step_K"], rtol=RTOL)
    assert rel(new.params.Lam, g["step_Lam"]) < 1e-9
    assert new.params.rho == pytest.approx(float(g["step_rho"]), rel=RTOL)
    idx = g["idx"]
    assert rel(new.Sigma[idx], g["step_Sigma"]) < 1e-12
    np.testing.assert_allclose(new.M[idx], g["step_M"], rtol=1e-12)
    np.testing.assert_allclose(new.S[idx], g["step_S"], rtol=1e-10)


def test_marginal_loglik_matches_oracle(E):
    r, mu, D, K, lam = philox.make_regime(3000, 11, 4)
    ds = host_ds(E, r, mu, D)
    p = E.model.ModelParams(K=K + 0.01, Lam=lam * 0.7, rho=55.0)
    want = oracle_em.marginal_loglik(r, mu, D, p.K, p.Lam, p.rho)
    assert E.em.marginal_loglik(ds, p) == pytest.approx(want, rel=1e-11)


# ---- the reference's test_em.py, restated ---------------------------------------


def test_vanishing_rho_leaves_prior_covariance(E):  # test_em.py:16-22
    ds, truth = make_dataset(E, 20, seed=30)
    p = E.model.ModelParams(K=truth.K, Lam=truth.Lam, rho=1e-300)
    new = E.em.em_step(state(E, p), ds)
    lam_inv = np.linalg.inv(truth.Lam)
    np.testing.assert_allclose(new.Sigma, np.broadcast_to(lam_inv, (20, 2, 2)), rtol=1e-9)


def test_flat_profiles_fixed_point_of_k(E):  # test_em.py:24-38
    V = 60
    mu, D = np.ones(V), np.zeros((V, 2))
    r = philox.synth(philox.Stream(31), [0.1, 0.3], np.linalg.inv(E.model.REFERENCE_LAMBDA_INV), 100.0, mu, D)
    ds = host_ds(E, r, mu, D)
    p0 = E.model.ModelParams(K=np.array([0.2, 0.2]), Lam=np.linalg.inv(E.model.REFERENCE_LAMBDA_INV), rho=5.0)
    new = E.em.em_step(state(E, p0), ds)
    np.testing.assert_allclose(new.params.K, p0.K, rtol=1e-12)
    np.testing.assert_allclose(new.M, np.broadcast_to(p0.K, (V, 2)), rtol=1e-12)
    want_rho = V / float(np.sum((ds.r - ds.mu) ** 2))
    assert new.params.rho == pytest.approx(want_rho, rel=1e-12)


def test_equal_s_gives_reciprocal_rho(E):  # test_em.py:40-44
    ds, truth = make_dataset(E, 25, seed=32)
    new = E.em.em_step(state(E, truth), ds)
    assert new.params.rho == pytest.approx(ds.V / float(np.sum(new.S)), rel=1e-12)


def test_sigma_spd_for_every_gene(E):  # test_em.py:46-50
    ds, truth = make_dataset(E, 150, seed=33)
    new = E.em.em_step(state(E, truth), ds)
    np.linalg.cholesky(new.Sigma)
    assert new.Sigma.shape == (150, 2, 2) and new.M.shape == (150, 2) and new.S.shape == (150,)


def test_ascent_on_random_small_instances(E):  # test_em.py:54-60
    for seed in range(37, 57):
        ds, _ = make_dataset(E, 50, seed=seed)
        hp = E.model.default_hyperparams(3)
        _, trace = E.em.em_fit(ds, init_params(E, hp), max_iter=150)
        ll = trace.loglik
        assert np.all(np.diff(ll) >= -1e-9 * np.abs(ll[1:])), f"seed {seed}"


def test_fixed_point_after_convergence(E):  # test_em.py:62-76
    s = philox.Stream(34)
    raw = s.uniforms(120 * 3).reshape(120, 3)
    mu = raw[:, -1].copy()
    D = raw[:, :-1] - mu[:, None]
    lam = np.linalg.inv(E.model.REFERENCE_LAMBDA_INV)
    r = philox.synth(s, [0.1, 0.3], lam, 100.0, mu, D)
    ds = host_ds(E, r, mu, D)
    hp = E.model.default_hyperparams(3)
    params, _ = E.em.em_fit(ds, init_params(E, hp), max_iter=5000, rel_tol=1e-15)
    after = E.em.em_step(state(E, params), ds).params
    assert np.max(np.abs(after.K - params.K)) < 1e-6
    assert abs(after.rho - params.rho) < 1e-5 * params.rho
    assert np.max(np.abs(after.Lam - params.Lam)) < 1e-4 * np.max(np.abs(params.Lam))


def test_noiseless_data_keeps_k_exact(E):  # test_em.py:78-90
    codes = philox.profile_codes(philox.Stream(35), 40, 3)
    mu, D = philox.codes_to_working(codes, 3)
    K = np.array([0.1, 0.3])
    r = D @ K + mu  # ZeroStream: beta = K, eps = 0
    ds = host_ds(E, r, mu, D)
    p0 = E.model.ModelParams(K=K, Lam=np.linalg.inv(E.model.REFERENCE_LAMBDA_INV), rho=1e9)
    new = E.em.em_step(state(E, p0), ds)
    np.testing.assert_allclose(new.params.K, K, atol=1e-10)
    assert new.params.rho > p0.rho


def test_matches_direct_maximization_on_tiny_instance(E):  # test_em.py:92-110
    scipy_opt = pytest.importorskip("scipy.optimize")
    r, mu, D, _, _ = philox.make_regime(40, 36, 2)
    ds = host_ds(E, r, mu, D)
    hp = E.model.default_hyperparams(2)
    params, _ = E.em.em_fit(ds, init_params(E, hp), max_iter=5000, rel_tol=1e-14)

    def neg_ll(theta):
        k, log_lam, log_rho = theta
        return -oracle_em.marginal_loglik(r, mu, D, np.array([k]), np.array([[np.exp(log_lam)]]), np.exp(log_rho))

    best = None
    for k in np.linspace(-0.5, 1.0, 16):
        for ll_ in np.linspace(0, 8, 9):
            for lr in np.linspace(0, 8, 9):
                v = neg_ll([k, ll_, lr])
                if best is None or v < best[1]:
                    best = ([k, ll_, lr], v)
    res = scipy_opt.minimize(neg_ll, best[0], method="Nelder-Mead",
                             options={"xatol": 1e-10, "fatol": 1e-12, "maxiter": 4000})
    assert abs(params.K[0] - res.x[0]) < 1e-3


def test_permutation_invariance(E):  # test_em.py:112-121
    ds, _ = make_dataset(E, 200, seed=38)
    hp = E.model.default_hyperparams(3)
    perm = np.random.default_rng(1).permutation(ds.V)
    ds_p = E.model.Dataset(r=ds.r[perm], mu=ds.mu[perm], D=ds.D[perm], n_networks=3)
    p1, _ = E.em.em_fit(ds, init_params(E, hp), max_iter=60)
    p2, _ = E.em.em_fit(ds_p, init_params(E, hp), max_iter=60)
    np.testing.assert_allclose(p1.K, p2.K, rtol=1e-9)
    np.testing.assert_allclose(p1.rho, p2.rho, rtol=1e-9)


def test_serial_parallel_bit_identical(E):  # test_em.py:123-131
    ds, _ = make_dataset(E, 1500, seed=39)
    hp = E.model.default_hyperparams(3)
    p1, t1 = E.em.em_fit(ds, init_params(E, hp), max_iter=25, plan=E.linalg.ExecPlan(workers=1))
    p2, t2 = E.em.em_fit(ds, init_params(E, hp), max_iter=25, plan=E.linalg.ExecPlan(workers=3))
    assert np.array_equal(p1.K, p2.K)
    assert p1.rho == p2.rho
    assert np.array_equal(t1.loglik, t2.loglik)


def test_max_iter_validated(E):  # test_em.py:133-137
    ds, _ = make_dataset(E, 10, seed=40)
    with pytest.raises(ValueError):
        E.em.em_fit(ds, init_params(E, E.model.default_hyperparams(3)), max_iter=0)


@pytest.mark.parametrize("V", [1_000_000, 9_000_001])
def test_em_at_scale_matches_fused_oracle_step(E, V):
    """One em_step on device-generated genes vs the oracle's float64 step on the same data
    (9_000_001 genes: the 8192-gene chunk plan and the reducer warp)."""
    from paper_2401_10068_b200 import model

    N = 4
    r, mu, D, K, lam = philox.make_regime(V, 77, N)
    ds = host_ds(E, r, mu, D)
    p = model.ModelParams(K=K, Lam=lam, rho=100.0)
    new = E.em.em_step(state(E, p), ds)
    K1, L1, r1, _, _, _ = oracle_em.em_step(r, mu, D, K, lam, 100.0)
    np.testing.assert_allclose(new.params.K, K1, rtol=1e-10)
    assert new.params.rho == pytest.approx(r1, rel=1e-10)
    assert rel(new.params.Lam, L1) < 1e-8
