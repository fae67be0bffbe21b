"""vb_posterior_sample on the GPU vs the reference's own draws (goldens) and the
reference test suite's moment checks (reference tests/test_vb.py:237-258)."""

from types import SimpleNamespace

import numpy as np
import pytest

from golden_io import Golden, names
from oracle import philox

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    from paper_2401_10068_b200 import model, samplers, vb

    return SimpleNamespace(vb=vb, model=model, samplers=samplers)


@pytest.mark.parametrize("name", names("post_"))
def test_draws_match_reference_stream(E, name):
    g = Golden(name)
    st = SimpleNamespace(a_rho=float(g["a_rho"]), b_rho=float(g["b_rho"]), k0k=g["k0k"], lam0l_inv=g["lam0l_inv"])
    h = g.hyper
    hp = E.model.HyperParams(a0=h.a0, b0=h.b0, q0=h.q0, n0=h.n0, K0=h.K0, Lambda0=h.Lambda0)
    rng = E.samplers.RngStream(int(g["seed"]), int(g["stream_id"]), int(g["pre_block"]))
    out = E.vb.vb_posterior_sample(rng, st, hp, int(g["V"]), int(g["n"]))
    assert rng._block == int(g["end_block"]), "stream cursor must advance exactly like the reference's"
    for k in ("Lambda", "K", "rho"):
        np.testing.assert_allclose(out[k], g[k], rtol=1e-9, atol=1e-12 * np.abs(g[k]).max(), err_msg=k)


def _fit_small(E, V, seed, max_iter):
    r, mu, D, _, _ = philox.make_regime(V, seed, 3)
    ds = E.model.Dataset(r=r, mu=mu, D=D, n_networks=3)
    hp = E.model.default_hyperparams(3)
    st, _ = E.vb.vb_fit(ds, hp, max_iter=max_iter)
    return ds, hp, st


def test_moment_recovery(E):  # reference tests/test_vb.py:238-246
    ds, hp, st = _fit_small(E, 200, 15, 120)
    draws = E.vb.vb_posterior_sample(E.samplers.RngStream(90), st, hp, ds.V, 100_000)
    nu = hp.n0 + ds.V
    np.testing.assert_allclose(draws["rho"].mean(), st.a_rho / st.b_rho, rtol=0.01)
    np.testing.assert_allclose(draws["K"].mean(0), st.k0k, atol=5e-3)
    want = nu * np.linalg.inv(st.lam0l_inv)
    assert np.linalg.norm(draws["Lambda"].mean(0) - want) < 0.05 * np.linalg.norm(want)


def test_reproducible_and_validated(E):  # reference tests/test_vb.py:248-258
    ds, hp, st = _fit_small(E, 50, 16, 40)
    a = E.vb.vb_posterior_sample(E.samplers.RngStream(91), st, hp, ds.V, 500)
    b = E.vb.vb_posterior_sample(E.samplers.RngStream(91), st, hp, ds.V, 500)
    np.testing.assert_array_equal(a["K"], b["K"])
    np.testing.assert_array_equal(a["rho"], b["rho"])
    with pytest.raises(ValueError):
        E.vb.vb_posterior_sample(E.samplers.RngStream(92), st, hp, ds.V, 0)
