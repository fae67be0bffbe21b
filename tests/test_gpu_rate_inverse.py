"""The sweep tail's rate inversion against the reference's semantics (row a11: linalg.py:111-192
inverse_batched wrapped by spd_jitter_retry, linalg.py:279-298, at vb.py:137 / 183 and em.py):
adjugate with the |det| >= 1e-300 guard for d <= 3, LU-class pivoted elimination for d >= 4,
one retry with 1e-10 tr/d on the diagonal, NumericError after it -- and, like the reference,
no positive-definiteness test (an indefinite rate is inverted).  Checked against the oracle's
restatement (oracle/cavi.py inv_retry, pinned to the reference) on the device routine itself
(cv_test_rate_inverse runs tail_inverse as a sweep does)."""

import ctypes as C

import numpy as np
import pytest

from oracle import cavi as ocavi

pytestmark = pytest.mark.gpu


def device_inverse(A):
    from paper_2401_10068_b200 import _lib

    A = np.ascontiguousarray(A, dtype=np.float64)
    d = A.shape[0]
    out, ld, ok = np.empty((d, d)), np.empty(1), C.c_int32()
    _lib.check(_lib.lib().cv_test_rate_inverse(_lib.dptr(A), d, 0, _lib.dptr(out), _lib.dptr(ld), C.byref(ok)))
    return out, float(ld[0]), bool(ok.value)


def reference(A):
    try:
        S = ocavi.inv_retry(A.copy(), "Q(Lambda) rate inversion")
    except ocavi.NumericFailure:
        return None
    return S


@pytest.mark.parametrize("d", range(1, 16))
def test_spd_rates(d):
    rng = np.random.default_rng(d)
    X = rng.standard_normal((d, 3 * d))
    A = X @ X.T / d + 0.1 * np.eye(d)
    S, ld, ok = device_inverse(A)
    assert ok
    np.testing.assert_allclose(S, reference(A), rtol=1e-10, atol=1e-12 * np.abs(S).max())
    assert abs(ld - np.linalg.slogdet(A)[1]) < 1e-10 * max(1.0, abs(ld))


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 9, 15])
def test_indefinite_rates_are_inverted_like_the_reference(d):
    """The reference never tests positive definiteness here (adjugate / LU): neither does the tail."""
    rng = np.random.default_rng(100 + d)
    Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    ev = np.linspace(-2.0, 3.0, d) + 0.37  # no zero eigenvalue
    A = (Q * ev) @ Q.T
    A = 0.5 * (A + A.T)
    S, ld, ok = device_inverse(A)
    want = reference(A)
    assert ok and want is not None
    np.testing.assert_allclose(S, want, rtol=1e-9, atol=1e-11 * np.abs(want).max())
    assert abs(ld - np.linalg.slogdet(A)[1]) < 1e-10 * max(1.0, abs(ld))


@pytest.mark.parametrize("d", [4, 5, 8, 15])
def test_exactly_singular_rate_takes_the_jitter_retry(d):
    """Rank-deficient rate: the elimination hits an exact zero pivot (the reference's LinAlgError),
    the retry inverts A + 1e-10 tr(A)/d I -- the reference's result."""
    A = np.ones((d, d))
    want = reference(A)
    assert want is not None  # the reference's retry succeeds
    S, ld, ok = device_inverse(A)
    assert ok
    np.testing.assert_allclose(S, want, rtol=1e-6, atol=1e-6 * np.abs(want).max())  # cond ~ 1e10


@pytest.mark.parametrize("d", [1, 2, 3])
def test_tiny_determinant_fails_after_the_retry(d):
    """|det| < 1e-300 (the adjugate's guard) before and after the 1e-10 relative jitter: the
    reference raises NumericError; the tail reports failure (CV_ERR_NUMERIC for the fit)."""
    A = 10.0 ** (-310 / d) * np.eye(d)
    assert reference(A) is None
    _, _, ok = device_inverse(A)
    assert not ok


def _errors():
    import json
    import os

    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "errors.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("name", sorted(_errors()))
def test_vb_fit_raises_what_the_reference_raises(name):
    """Reference-made error goldens (tests/golden/make_error_golden.py): a Lambda0 whose
    determinant is under the adjugate's 1e-300 guard makes the reference's vb_init raise
    BatchItemError over every gene; the drop-in raises the same class and message."""
    from oracle import philox
    from paper_2401_10068_b200 import linalg, model, vb

    g = _errors()[name]
    rc = g["recipe"]
    r, mu, D = philox.generate(rc["seed"], rc["V"], rc["N"], rc["K"], np.array(rc["Lam"]), rc["rho"])
    ds = model.Dataset(r=r, mu=mu, D=D, n_networks=rc["N"])
    d = rc["N"] - 1
    hp = model.HyperParams(a0=0.5, b0=0.5, q0=0.001, n0=1, K0=np.full(d, 1 / 3),
                           Lambda0=rc["lambda0_scale"] * np.eye(d))
    assert g["error"] == "BatchItemError"
    with pytest.raises(linalg.BatchItemError) as info:
        vb.vb_fit(ds, hp)
    assert str(info.value) == g["message"]
