"""Point-estimate EM restated (oracle) -- TEST INFRASTRUCTURE ONLY.

Restates reference em.py:44-124 (E-step, joint M-step, em_fit loop) and
model.py:273-287 (the beta-marginalised log-likelihood EM ascends) with the
reference's operations in the reference's order (1024-gene chunks, fixed
pairwise tree), pinned bit-for-bit against goldens the reference produced.
"""

from __future__ import annotations

import numpy as np

from .cavi import NumericFailure, chunk_total, inv_retry, pairwise, spans
from .philox import inv_small


def marginal_loglik(r, mu, D, K, Lam, rho) -> float:
    """model.py:273-287 (reduce_sum over 1024-item chunks + pairwise tree)."""
    lam_inv = inv_small(Lam)
    s2 = 1.0 / rho + np.einsum("vd,de,ve->v", D, lam_inv, D)
    resid = r - mu - D @ K
    terms = -0.5 * (np.log(2.0 * np.pi * s2) + resid ** 2 / s2)
    parts = [np.sum(terms[lo:lo + 1024], axis=0) for lo in range(0, terms.shape[0], 1024)]
    return float(pairwise(parts))


def em_step(r, mu, D, K, Lam, rho):
    """One E-step + joint M-step (em.py:44-94); returns (K', Lam', rho', Sigma, M, S)."""
    V = D.shape[0]
    lam_k = Lam @ K
    sig_p, m_p, s_p, sm, ss, sq = [], [], [], [], [], []
    for lo, hi in spans(V):
        Dc = D[lo:hi]
        x = r[lo:hi] - mu[lo:hi]
        prec = np.matmul(Dc[:, :, None], np.swapaxes(Dc[:, :, None], -1, -2))
        if rho != 1.0:
            prec *= rho
        prec = prec + 1.0 * Lam[None]
        sig = inv_retry(prec, "E-step covariance")
        m = np.einsum("vij,vj->vi", sig, lam_k[None, :] + rho * x[:, None] * Dc)
        second = np.einsum("vi,vj->vij", m, m) + sig
        s = x ** 2 - 2.0 * x * np.einsum("vi,vi->v", Dc, m) + np.einsum("vi,vij,vj->v", Dc, second, Dc)
        sig_p.append(sig)
        m_p.append(m)
        s_p.append(s)
        sm.append(chunk_total(m))
        ss.append(chunk_total(second))
        sq.append(chunk_total(s))
    sum_m, sum_second, sum_s = pairwise(sm), pairwise(ss), float(pairwise(sq))
    if sum_s <= 0.0:
        raise NumericFailure("non-positive residual sum in M-step")
    rho_new = V / sum_s
    k_new = sum_m / V
    lam_inv = sum_second / V - np.outer(k_new, k_new)
    lam_inv = 0.5 * (lam_inv + lam_inv.T)
    lam_new = inv_retry(lam_inv, "M-step precision")
    lam_new = 0.5 * (lam_new + lam_new.T)
    return k_new, lam_new, float(rho_new), np.concatenate(sig_p), np.concatenate(m_p), np.concatenate(s_p)


def em_fit(r, mu, D, K, Lam, rho, max_iter=1000, rel_tol=1e-10):
    """em.py:97-124; returns ((K, Lam, rho), loglik trace, K trace, rho trace)."""
    if max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    lls, ks, rhos = [], [], []
    prev = marginal_loglik(r, mu, D, K, Lam, rho)
    for _ in range(max_iter):
        K, Lam, rho, _, _, _ = em_step(r, mu, D, K, Lam, rho)
        ll = marginal_loglik(r, mu, D, K, Lam, rho)
        lls.append(ll)
        ks.append(K)
        rhos.append(rho)
        if abs(ll - prev) < rel_tol * abs(ll):
            break
        prev = ll
    return (K, Lam, rho), np.array(lls), np.stack(ks), np.array(rhos)
