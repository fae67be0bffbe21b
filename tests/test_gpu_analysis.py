"""Posterior summaries on the GPU (paper_2401_10068_b200.analysis) against what the
reference's tissuemix.analysis returned on the same inputs (tests/golden/kde/expected.npz,
made by tests/golden/make_kde_golden.py), plus the reference's own test_analysis.py cases.

Tolerances (fp64): bandwidth, means and densities 1e-12 relative (compensated device sums
vs numpy's pairwise sums); central-interval bounds bit-exact (same order statistics, same
interpolation arithmetic); modes within 1e-9 of the grid span (the golden-section path is
the reference's, evaluated on densities that agree to ~1e-15).
"""

import json
import os

import numpy as np
import pytest

from kde_cases import CASES, SUMMARY_CASES, inputs, summary_inputs

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
EXP = np.load(os.path.join(GOLD, "kde", "expected.npz"))


@pytest.fixture(scope="module")
def an():
    from paper_2401_10068_b200 import analysis

    return analysis


@pytest.mark.parametrize("name", sorted(CASES))
def test_kde_matches_reference(an, name):
    c = CASES[name]
    x = inputs(c)
    kde = an.kde_fit(x, c.get("bw"))
    assert kde.bandwidth == pytest.approx(float(EXP[f"{name}/bandwidth"]), rel=1e-12)
    n = c.get("grid", 512)
    g = an.kde_grid(kde, lo=c.get("lo"), hi=c.get("hi"), n=n)
    if c.get("bw"):  # same bandwidth bits -> the same linspace
        np.testing.assert_array_equal(g.x, EXP[f"{name}/grid_x"])
    np.testing.assert_allclose(g.density, EXP[f"{name}/grid_density"], rtol=1e-12, atol=1e-300)
    span = float(EXP[f"{name}/grid_x"][-1] - EXP[f"{name}/grid_x"][0])
    mode, multi = an.kde_mode(kde, n=n, lo=c.get("lo"), hi=c.get("hi"))
    assert abs(mode - float(EXP[f"{name}/mode"])) <= 1e-9 * span
    assert multi == bool(EXP[f"{name}/multimodal"])
    assert abs(g.mode - mode) <= 1e-9 * span
    q = np.linspace(float(x.min()) - 1.0, float(x.max()) + 1.0, 97)
    np.testing.assert_allclose(an.kde_density(kde, q), EXP[f"{name}/density_q"], rtol=1e-12, atol=1e-300)


def _cmp_entry(got, want, span):
    assert got["mean"] == pytest.approx(want["mean"], rel=1e-12, abs=1e-15)
    assert got["ci95"] == want["ci95"]  # bit-exact order statistics + lerp
    assert abs(got["mode"] - want["mode"]) <= 1e-9 * max(span, 1e-300) + 1e-15


@pytest.mark.parametrize("name", sorted(SUMMARY_CASES))
def test_summarize_matches_reference(an, name):
    c = SUMMARY_CASES[name]
    s = summary_inputs(c, GOLD)
    want = json.loads(str(EXP[f"{name}/report"]))
    got = an.summarize(s, c.get("bw"))
    assert set(got["parameters"]) == set(want["parameters"])
    assert set(got["full_weights"]) == set(want["full_weights"])
    for sec in ("parameters", "full_weights"):
        for k, w in want[sec].items():
            if k == "mode_vector":
                continue
            if k == "Lambda_mean":
                np.testing.assert_allclose(got[sec][k], w, rtol=1e-12, atol=1e-15)
                continue
            span = max(abs(w["ci95"][1] - w["ci95"][0]), abs(w["mean"]) * 1e-3)
            _cmp_entry(got[sec][k], w, span)
    np.testing.assert_allclose(got["full_weights"]["mode_vector"], want["full_weights"]["mode_vector"],
                               rtol=1e-9, atol=1e-12)


# ---- the reference's test_analysis.py, restated --------------------------------


def test_scott_bandwidth_formula(an):  # test_analysis.py:10-16
    x = np.random.default_rng(0).standard_normal(10_000)
    kde = an.kde_fit(x)
    assert kde.bandwidth == pytest.approx(np.std(x, ddof=1) * 10_000 ** (-0.2), rel=1e-12)
    assert kde.bandwidth == pytest.approx(0.158, abs=0.02)


def test_explicit_bandwidth_and_errors(an):  # test_analysis.py:18-30
    assert an.kde_fit([0.0, 1.0, 2.0], bandwidth=0.37).bandwidth == 0.37
    with pytest.raises(ValueError, match="bandwidth"):
        an.kde_fit([2.0, 2.0, 2.0])
    an.kde_fit([2.0, 2.0, 2.0], bandwidth=0.1)
    with pytest.raises(ValueError):
        an.kde_fit([1.0])


def test_close_to_normal_density(an):  # test_analysis.py:34-40
    from scipy.stats import norm

    x = np.random.default_rng(1).standard_normal(100_000)
    kde = an.kde_fit(x)
    grid = np.linspace(-4, 4, 401)
    assert np.max(np.abs(an.kde_density(kde, grid) - norm.pdf(grid))) < 0.01


def test_integrates_to_one(an):  # test_analysis.py:42-48
    rng = np.random.default_rng(2)
    x = np.concatenate([rng.standard_normal(3000), 4 + 0.5 * rng.standard_normal(2000)])
    kde = an.kde_fit(x)
    grid = an.kde_grid(kde, lo=x.min() - 5 * kde.bandwidth, hi=x.max() + 5 * kde.bandwidth, n=2048)
    assert np.all(grid.density >= 0)
    assert 0.98 <= grid.integral <= 1.02


def test_resolution_floor_and_summary_minimum(an):  # test_analysis.py:88-91, 111-113
    kde = an.kde_fit([0.0, 1.0], bandwidth=1.0)
    with pytest.raises(ValueError, match="256"):
        an.kde_mode(kde, n=100)
    with pytest.raises(ValueError, match="100"):
        an.summarize({"K": np.zeros((50, 2)), "rho": np.ones(50)})


def test_constant_weight_samples(an):  # test_analysis.py:95-100
    report = an.summarize({"K": np.tile([0.1, 0.3], (200, 1)), "rho": np.full(200, 7.0)})
    np.testing.assert_allclose(report["full_weights"]["mode_vector"], [0.1, 0.3, 0.6], atol=1e-12)
    assert report["parameters"]["rho"]["mode"] == 7.0


def test_summarize_posterior_draws_from_the_gpu_sampler(an):
    """End to end on the device path: fit -> vb_posterior_sample -> summarize."""
    from oracle import philox
    from paper_2401_10068_b200 import model, samplers, vb

    r, mu, D, K, lam = philox.make_regime(5000, 3, 3)
    ds = model.Dataset(r=r, mu=mu, D=D, n_networks=3)
    hp = model.default_hyperparams(3)
    st, _ = vb.vb_fit(ds, hp)
    draws = vb.vb_posterior_sample(samplers.RngStream(4), st, hp, ds.V, 2000)
    rep = an.summarize(draws)
    w = rep["full_weights"]["mode_vector"]
    assert abs(sum(w) - 1.0) < 0.05
    np.testing.assert_allclose(w[:2], K, atol=0.05)
