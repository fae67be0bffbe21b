"""Direct per-gene CAVI restatement (oracle) -- TEST INFRASTRUCTURE ONLY.

Restates the reference's variational engine operation-for-operation so
that, on the same numpy/scipy, it reproduces the reference's numbers
bit-for-bit (pinned against goldens made by the reference itself,
tests/golden/make_golden.py):

  state init            reference vb.py:82-111
  residual moment sum   reference vb.py:114-126
  one sweep             reference vb.py:129-198
  Wishart log-normaliser / E ln|Lambda|   reference vb.py:201-213
  closed-form bound     reference vb.py:216-304
  fit loop + stop rule  reference vb.py:307-354
  1024-gene chunk map + fixed pairwise tree   reference linalg.py:238-276, 301-328
  jitter-once retry     reference linalg.py:279-298
  hyperparameter defaults   reference model.py:200-215

Per-gene state is materialised (V, d, d) exactly as the reference does; this
is the slow, obviously-faithful statement the CUDA engine is checked
against, not a design to imitate.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.special import digamma, gammaln, multigammaln

from .philox import SingularItem, chol_lower, inv_small

CHUNK = 1024  # linalg.py:43
LN2PI = np.log(2.0 * np.pi)


class NumericFailure(RuntimeError):
    """Mirror of linalg.NumericError (linalg.py:63-64)."""


@dataclass(frozen=True)
class Hyper:
    a0: float
    b0: float
    q0: float
    n0: int
    K0: np.ndarray
    Lambda0: np.ndarray

    @property
    def dim(self) -> int:
        return self.K0.shape[0]


def default_hyper(N: int) -> Hyper:
    """model.py:200-215 (K0 = 1/3 for every N; Lambda0 = inv(REF) for N=3 else 100 I)."""
    if N < 2:
        raise ValueError("need at least 2 networks")
    dim = N - 1
    ref = np.array([[0.01, 0.005], [0.005, 0.008]])
    lam0 = np.linalg.inv(ref) if N == 3 else np.linalg.inv(0.01 * np.eye(dim))
    return Hyper(0.5, 0.5, 0.001, 1, np.full(dim, 1.0 / 3.0), lam0)


@dataclass(frozen=True)
class State:
    a_rho: float
    b_rho: float
    mu_beta: np.ndarray
    lam_beta: np.ndarray
    k0k: np.ndarray
    lam0l_inv: np.ndarray
    e_beta: np.ndarray
    e_bbt: np.ndarray
    e_lam: np.ndarray
    e_rho: float
    e_k: np.ndarray
    e_lamk: np.ndarray


@dataclass
class Trace:
    elbo: np.ndarray
    delta_k0k: np.ndarray
    delta_rho: np.ndarray
    delta_lam: np.ndarray


# ------------------------------------------------------------ reduction plan
def spans(V: int):
    return [(lo, min(lo + CHUNK, V)) for lo in range(0, V, CHUNK)]


def pairwise(parts):
    """Fixed pairwise tree; odd tail carried up (linalg.py:238-255)."""
    parts = list(parts)
    while len(parts) > 1:
        nxt = [parts[i] + parts[i + 1] for i in range(0, len(parts) - 1, 2)]
        if len(parts) % 2:
            nxt.append(parts[-1])
        parts = nxt
    return parts[0]


def chunk_total(a):
    """reduce_sum on one <=1024-item chunk (linalg.py:258-276)."""
    out = np.sum(np.asarray(a, dtype=np.float64), axis=0)
    return float(out) if np.ndim(out) == 0 else out


def inv_retry(A, what):
    """spd_jitter_retry(inverse_batched, A) (linalg.py:279-298)."""
    try:
        return inv_small(A)
    except SingularItem as first:
        n = A.shape[-1]
        jit = 1e-10 * np.trace(A, axis1=-2, axis2=-1) / n
        J = A + (np.atleast_1d(jit)[..., None, None] if A.ndim == 3 else jit) * np.eye(n)
        try:
            return inv_small(J)
        except SingularItem as second:
            raise NumericFailure(f"{what} failed after jitter retry: {second}") from first


def _finite(a, name):
    if not np.all(np.isfinite(a)):
        raise FloatingPointError(f"non-finite values in {name}")


# ------------------------------------------------------------ the engine
def init(r, mu, D, hp: Hyper) -> State:
    V, d = D.shape
    if hp.dim != d:
        raise ValueError(f"hyperparams dim {hp.dim} != dataset dim {d}")
    lamb = np.broadcast_to(hp.Lambda0, (V, d, d)).copy()
    mub = np.broadcast_to(hp.K0, (V, d)).copy()
    sig = inv_small(lamb)
    elam = (hp.n0 + V) * inv_small(hp.Lambda0.copy())
    return State(
        a_rho=hp.a0, b_rho=hp.b0, mu_beta=mub, lam_beta=lamb, k0k=hp.K0.copy(),
        lam0l_inv=hp.Lambda0.copy(), e_beta=mub.copy(),
        e_bbt=np.einsum("vi,vj->vij", mub, mub) + sig, e_lam=elam,
        e_rho=hp.a0 / hp.b0, e_k=hp.K0.copy(), e_lamk=elam @ hp.K0,
    )


def resid_sum(st: State, r, mu, D) -> float:
    """sum_i (r-mu)^2 - 2(r-mu) D.E[b] + D.E[bb^T].D under st's moments (vb.py:114-126)."""
    parts = []
    for lo, hi in spans(D.shape[0]):
        x = r[lo:hi] - mu[lo:hi]
        Dc = D[lo:hi]
        sig = inv_small(st.lam_beta[lo:hi])
        m2 = np.einsum("vi,vj->vij", st.mu_beta[lo:hi], st.mu_beta[lo:hi]) + sig
        q = np.einsum("vi,vij,vj->v", Dc, m2, Dc)
        lin = np.einsum("vi,vi->v", Dc, st.e_beta[lo:hi])
        parts.append(chunk_total(x ** 2 - 2.0 * x * lin + q))
    return float(pairwise(parts))


def step(st: State, r, mu, D, hp: Hyper) -> State:
    """One sweep: expectations -> rho -> beta -> (K, Lambda) (vb.py:129-198)."""
    V, d = D.shape
    nu, qv = hp.n0 + V, hp.q0 + V
    elam = nu * inv_retry(st.lam0l_inv, "Q(Lambda) rate inversion")
    elamk = elam @ st.k0k
    a_rho = hp.a0 + 0.5 * V
    b_rho = hp.b0 + 0.5 * resid_sum(st, r, mu, D)
    e_rho = a_rho / b_rho
    lam_parts, mu_parts, m2_parts, smu, sm2 = [], [], [], [], []
    for lo, hi in spans(V):
        Dc = D[lo:hi]
        x = r[lo:hi] - mu[lo:hi]
        _finite(Dc, "A")
        _finite(elam, "C")
        lb = np.matmul(Dc[:, :, None], np.swapaxes(Dc[:, :, None], -1, -2))
        if e_rho != 1.0:
            lb *= e_rho
        lb = lb + 1.0 * elam[None]
        sb = inv_retry(lb, "beta precision inversion")
        rhs = elamk[None, :] + e_rho * Dc * x[:, None]
        mb = np.einsum("vij,vj->vi", sb, rhs)
        m2 = np.einsum("vi,vj->vij", mb, mb) + sb
        lam_parts.append(lb)
        mu_parts.append(mb)
        m2_parts.append(m2)
        smu.append(chunk_total(mb))
        sm2.append(chunk_total(m2))
    sum_mu, sum_m2 = pairwise(smu), pairwise(sm2)
    k0k = (sum_mu + hp.q0 * hp.K0) / qv
    L = inv_small(hp.Lambda0) + sum_m2 + hp.q0 * np.outer(hp.K0, hp.K0) - qv * np.outer(k0k, k0k)
    L = 0.5 * (L + L.T)
    elam_new = nu * inv_retry(L, "Q(Lambda) rate inversion")
    mub = np.concatenate(mu_parts)
    return State(
        a_rho=a_rho, b_rho=b_rho, mu_beta=mub, lam_beta=np.concatenate(lam_parts), k0k=k0k,
        lam0l_inv=L, e_beta=mub, e_bbt=np.concatenate(m2_parts), e_lam=elam_new,
        e_rho=e_rho, e_k=k0k, e_lamk=elam_new @ k0k,
    )


def wishart_log_z(dof, scale):
    """vb.py:201-207; None when improper (dof <= d-1)."""
    d = scale.shape[0]
    if dof <= d - 1:
        return None
    _, ld = np.linalg.slogdet(scale)
    return 0.5 * dof * d * np.log(2.0) + 0.5 * dof * ld + multigammaln(0.5 * dof, d)


def e_ln_det(dof, scale):
    """E ln|Lambda| under Wishart(dof, scale) (vb.py:210-213)."""
    d = scale.shape[0]
    _, ld = np.linalg.slogdet(scale)
    return float(np.sum(digamma(0.5 * (dof + 1 - np.arange(1, d + 1)))) + d * np.log(2.0) + ld)


def elbo(st: State, r, mu, D, hp: Hyper) -> float:
    """Closed-form bound (vb.py:216-304)."""
    V, d = D.shape
    nu, qv = hp.n0 + V, hp.q0 + V
    S = inv_small(st.lam0l_inv)
    e_rho = st.a_rho / st.b_rho
    e_lnrho = float(digamma(st.a_rho) - np.log(st.b_rho))
    e_lnlam = e_ln_det(nu, S)
    rp, sp, lp = [], [], []
    for lo, hi in spans(V):
        Dc = D[lo:hi]
        x = r[lo:hi] - mu[lo:hi]
        mb = st.mu_beta[lo:hi]
        sig = inv_small(st.lam_beta[lo:hi])
        m2 = np.einsum("vi,vj->vij", mb, mb) + sig
        rp.append(chunk_total(x ** 2 - 2.0 * x * np.einsum("vi,vi->v", Dc, mb)
                              + np.einsum("vi,vij,vj->v", Dc, m2, Dc)))
        dev = mb - st.k0k
        sp.append(chunk_total(sig + np.einsum("vi,vj->vij", dev, dev)))
        sgn, ld = np.linalg.slogdet(st.lam_beta[lo:hi])
        if np.any(sgn <= 0):
            raise NumericFailure("non-PD beta precision in bound evaluation")
        lp.append(chunk_total(-ld))
    resid, scat, ldsig = pairwise(rp), pairwise(sp), pairwise(lp)

    lik = 0.5 * V * (e_lnrho - LN2PI) - 0.5 * e_rho * resid
    tb = 0.5 * V * e_lnlam - 0.5 * V * d * LN2PI - 0.5 * (nu * float(np.trace(S @ scat)) + V * d / qv)
    dk = st.k0k - hp.K0
    tk = 0.5 * d * np.log(hp.q0) - 0.5 * d * LN2PI + 0.5 * e_lnlam - 0.5 * hp.q0 * (nu * float(dk @ S @ dk) + d / qv)
    tl = 0.5 * (hp.n0 - d - 1) * e_lnlam - 0.5 * nu * float(np.trace(inv_small(hp.Lambda0) @ S))
    zp = wishart_log_z(hp.n0, hp.Lambda0)
    if zp is not None:
        tl -= zp
    tr = hp.a0 * np.log(hp.b0) - gammaln(hp.a0) + (hp.a0 - 1.0) * e_lnrho - hp.b0 * e_rho
    hb = 0.5 * ldsig + 0.5 * V * d * (1.0 + LN2PI)
    hr = st.a_rho - np.log(st.b_rho) + gammaln(st.a_rho) + (1.0 - st.a_rho) * digamma(st.a_rho)
    qk = 0.5 * d * np.log(qv) - 0.5 * d * LN2PI + 0.5 * e_lnlam - 0.5 * d
    zq = wishart_log_z(nu, S)
    if zq is None:
        raise NumericFailure("Q(Lambda) is improper; dataset too small")
    ql = 0.5 * (nu - d - 1) * e_lnlam - 0.5 * nu * d - zq
    return float(lik + tb + tk + tl + tr + hb + hr - qk - ql)


def rel_delta(new, old) -> float:
    """vb.py:307-309."""
    den = max(float(np.max(np.abs(old))), 1e-300)
    return float(np.max(np.abs(np.asarray(new) - np.asarray(old)))) / den


def fit(r, mu, D, hp: Hyper, max_iter=300, rel_tol=1e-8, compute_elbo=True, param_tol=1e-10):
    """Sweep until the bound (or parameters) settle (vb.py:312-354)."""
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    st = init(r, mu, D, hp)
    es, dk, dr, dl = [], [], [], []
    prev = None
    for _ in range(max_iter):
        nw = step(st, r, mu, D, hp)
        dk.append(rel_delta(nw.k0k, st.k0k))
        dr.append(rel_delta(nw.a_rho / nw.b_rho, st.a_rho / st.b_rho))
        dl.append(rel_delta(nw.lam0l_inv, st.lam0l_inv))
        st = nw
        if compute_elbo:
            e = elbo(st, r, mu, D, hp)
            es.append(e)
            if prev is not None and abs(e - prev) < rel_tol * abs(e):
                break
            prev = e
        else:
            es.append(np.nan)
            if max(dk[-1], dr[-1], dl[-1]) < param_tol:
                break
    return st, Trace(np.array(es), np.array(dk), np.array(dr), np.array(dl))


__all__ = [
    "CHUNK", "Hyper", "NumericFailure", "State", "Trace", "chol_lower", "default_hyper",
    "e_ln_det", "elbo", "fit", "init", "inv_retry", "pairwise", "rel_delta", "resid_sum",
    "spans", "step", "wishart_log_z",
]


# ------------------------------------------------------------ posterior draws
def _gamma_ge1_many(stream, a: float, n: int) -> np.ndarray:
    """Cubed-normal rejection, vectorised rounds (reference samplers.py:220-237)."""
    d = a - 1.0 / 3.0
    c = 1.0 / np.sqrt(9.0 * d)
    out = np.empty(n)
    filled = 0
    while filled < n:
        todo = n - filled
        u = stream.uniforms(todo)
        x = stream.normals(todo)
        v = (1.0 + c * x) ** 3
        pos = v > 0.0
        logv = np.full_like(v, -np.inf)
        np.log(v, out=logv, where=pos)
        ok = pos & (np.log(u) < 0.5 * x * x + d - d * v + d * logv)
        k = int(np.count_nonzero(ok))
        out[filled:filled + k] = d * v[ok]
        filled += k
    return out


def gamma_many(stream, a: float, b: float, n: int) -> np.ndarray:
    """sample_gamma(rng, GammaParams(a, b), size=n) (reference samplers.py:240-261)."""
    if a >= 1.0:
        raw = _gamma_ge1_many(stream, a, n)
    else:
        boost = _gamma_ge1_many(stream, a + 1.0, n)
        u = stream.uniforms(n)
        raw = boost * u ** (1.0 / a)
    return raw / b


def posterior_sample(stream, a_rho, b_rho, k0k, lam0l_inv, hp: Hyper, V: int, n: int):
    """Joint (K, Lambda, rho) draws from the fitted Q (reference vb.py:357-393)."""
    if n < 1:
        raise ValueError("n_samples must be >= 1")
    d = k0k.shape[0]
    nu, qv = hp.n0 + V, hp.q0 + V
    R = chol_lower(inv_small(lam0l_inv))
    kd = np.empty((n, d))
    ld = np.empty((n, d, d))
    chunk = max(1, min(n, 4_000_000 // max(nu * d, 1)))
    done = 0
    while done < n:
        m = min(chunk, n - done)
        u = stream.normals(m * nu * d).reshape(m, nu, d)
        S = u @ R.T
        lam = np.einsum("mnd,mne->mde", S, S)
        ld[done:done + m] = lam
        Lk = chol_lower(inv_small(qv * lam))
        uk = stream.normals(m * d).reshape(m, d)
        kd[done:done + m] = k0k + np.einsum("mij,mj->mi", Lk, uk)
        done += m
    return {"K": kd, "Lambda": ld, "rho": np.asarray(gamma_many(stream, a_rho, b_rho, n))}
