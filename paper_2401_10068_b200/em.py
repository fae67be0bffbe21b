"""Point-estimate EM on the GPU: drop-in for the reference's `tissuemix.em`
(reference em.py:19: EmState, EmTrace, em_step, em_fit), SURVEY §8(f) row 3.

EM's E-step has the CAVI β-block's structure exactly -- per gene
(Λ + ρ D Dᵀ)⁻¹ with shared (Λ, ρ) -- so it runs on the same fused streaming
pass: with the generator (c, A, e_ρ) = (K, Λ, ρ) one pass yields the E-step
sums (Σ M_i, Σ E[ββᵀ]_i, Σ S_i) for the M-step AND the β-marginalised
log-likelihood of (K, Λ, ρ) (model.py:278-287) that em_fit ascends -- the
reference needs two passes per iteration (em.py:116-117).  The joint M-step
(em.py:84-93) runs on the device in centred, cancellation-free form, and the
em_fit loop (em.py:97-124) is a CUDA graph with the stop rule on the device.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib, linalg, model
from .vb import _dims, device_dataset

__all__ = ["EmState", "EmTrace", "em_fit", "em_step", "marginal_loglik"]


class EmState:
    """Current point estimate with the E-step cache (reference em.py:22-29).

    Sigma (V, d, d), M (V, d), S (V,) are the E-step quantities of the parameters
    that ENTERED the step; they are produced on first access by the materialise kernel.
    """

    def __init__(self, params, Sigma=None, M=None, S=None, _src=None):
        self.params = params
        self._arrays = {"Sigma": Sigma, "M": M, "S": S}
        self._src = _src  # (device dataset, K, Lam, Lam^-1, rho) of the E-step

    def _fill(self):
        dds, K, Lam, Li, rho = self._src
        V, d = dds.V, dds.dim
        cs = _lib.CvState()
        cs.d, cs.V = d, dds.V_total
        for j in range(d):
            cs.gen_c[j] = K[j]
        for i in range(d * d):
            cs.gen_A[i] = Lam.flat[i]
            cs.gen_Ainv[i] = Li.flat[i]
        cs.gen_e_rho = rho
        M, Sig, S = np.empty((V, d)), np.empty((V, d, d)), np.empty(V)
        _lib.check(_lib.lib().cv_materialize(dds.handle, None, C.byref(cs), 0, V, _lib.dptr(M), None, None,
                                             _lib.dptr(Sig), _lib.dptr(S)))
        self._arrays.update(Sigma=Sig, M=M, S=S)

    def _get(self, k):
        if self._arrays[k] is None:
            if self._src is None:
                return np.empty(0)
            self._fill()
        return self._arrays[k]

    @property
    def Sigma(self):
        return self._get("Sigma")

    @property
    def M(self):
        return self._get("M")

    @property
    def S(self):
        return self._get("S")


@dataclass
class EmTrace:
    """Per-iteration log-likelihood and parameter path (reference em.py:32-41)."""

    loglik: np.ndarray
    K: np.ndarray
    rho: np.ndarray

    def __len__(self) -> int:
        return len(self.loglik)


def _theta(p, d):
    K = np.ascontiguousarray(np.atleast_1d(p.K), dtype=np.float64)
    Lam = np.ascontiguousarray(np.atleast_2d(p.Lam), dtype=np.float64)
    if K.shape[0] != d or Lam.shape != (d, d):
        raise ValueError(f"parameters of dimension {K.shape[0]} for a dataset of dimension {d}")
    return K, Lam, float(p.rho)


def _step(ds, params):
    """theta -> (theta', Lambda^-1, marginal loglik of theta): one fused pass + device M-step."""
    dds = device_dataset(ds)
    d = _dims(ds)[1]
    K, Lam, rho = _theta(params, d)
    Ko, Lo, Li = np.empty(d), np.empty((d, d)), np.empty((d, d))
    ro, ll = C.c_double(), C.c_double()
    _lib.check(_lib.lib().cv_em_step(dds.handle, _lib.dptr(K), _lib.dptr(Lam), rho, _lib.dptr(Ko), _lib.dptr(Lo),
                                     C.byref(ro), _lib.dptr(Li), C.byref(ll)))
    new = model.ModelParams(K=Ko, Lam=Lo, rho=float(ro.value))
    return new, (dds, K, Lam, Li, rho), float(ll.value)


def em_step(state: EmState, ds, plan: linalg.ExecPlan | None = None) -> EmState:
    """One E-step plus joint M-step (reference em.py:80-94)."""
    new, src, _ = _step(ds, state.params)
    return EmState(new, _src=src)


def marginal_loglik(ds, p) -> float:
    """beta-marginalised log-likelihood of p (reference model.py:278-287), from the same pass."""
    return _step(ds, p)[2]


def em_fit(ds, init, max_iter: int = 1000, rel_tol: float = 1e-10, plan: linalg.ExecPlan | None = None):
    """Iterate until the marginal log-likelihood settles (reference em.py:97-124)."""
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    dds = device_dataset(ds)
    d = _dims(ds)[1]
    K, Lam, rho = _theta(init, d)
    Ko, Lo, ro = np.empty(d), np.empty((d, d)), C.c_double()
    ll, tk, tr = np.empty(max_iter), np.empty((max_iter, d)), np.empty(max_iter)
    n = C.c_int32()
    _lib.check(_lib.lib().cv_em_fit(dds.handle, _lib.dptr(K), _lib.dptr(Lam), rho, int(max_iter), float(rel_tol),
                                    _lib.dptr(Ko), _lib.dptr(Lo), C.byref(ro), _lib.dptr(ll), _lib.dptr(tk),
                                    _lib.dptr(tr), C.byref(n)))
    k = n.value
    params = model.ModelParams(K=Ko, Lam=Lo, rho=float(ro.value))
    return params, EmTrace(loglik=ll[:k].copy(), K=tk[:k].copy(), rho=tr[:k].copy())
