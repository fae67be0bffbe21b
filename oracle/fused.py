"""Single-pass rank-1 CAVI restatement with the device reduction plan (oracle).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

This is the executable specification of the CUDA engine
(paper_2401_10068_b200/csrc): the same algebra and the
same deterministic reduction plan, in numpy.  It is checked against the
direct restatement `oracle.cavi` (itself pinned to the reference) and is
what the multi-rank gloo tests run.

Algebra (reference vb.py:129-198 and vb.py:216-304 rewritten):
  every VB state's per-gene moments come from a "generator" (c, A, e_rho):
      Lambda_beta_i = A + e_rho D_i D_i^T          (vb.py:150-152)
      u = A^-1 D_i, s = D_i^T u, t = D_i^T c, den = 1 + e_rho s
      w = e_rho (x_i - t) / den,  x_i = r_i - mu_i
      mu_beta_i = c + w u,  Sigma_i = A^-1 - (e_rho/den) u u^T   (Sherman-Morrison)
  vb_init's state is the generator (K0, Lambda0, 0); the state produced by a
  sweep is (k0k_prev, E[Lambda]_prev, e_rho_new).  One streaming pass per
  state accumulates
      g = sum w D,  G = sum (w^2 - e_rho/den) D D^T,
      R = sum (x - t - s w)^2 + s/den    (= the residual moment sum, vb.py:114-126)
      Ld = sum ln den                    (ln|Lambda_beta_i| = ln|A| + ln den)
  from which the (K, Lambda) block, the next b_rho and the bound follow in
  O(d^3) with centred (cancellation-free) formulas.

Reduction plan (GPU-count invariant, deterministic):
  chunk  = plan_chunk_genes(V, d) consecutive genes (4096, or 8192 for d >= 3 and
           V >= 2^23: engine.cuh plan_chunk_genes)  -> one partial
  group  = GROUP_GENES (262144) consecutive genes = its chunks, summed by warp_rows_sum
           (strided lanes + butterfly)
  octant = ceil(n_groups/8) consecutive groups, summed by warp_rows_sum
  total  = pairwise tree over the 8 octants ((o0+o1)+(o2+o3))+((o4+o5)+(o6+o7))
A rank of a power-of-two world G<=8 owns 8/G consecutive octants, reduces
them with its subtree, and the G rank partials are combined by the top of
the same tree -- bit-identical totals for G = 1, 2, 4, 8.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.special import digamma, gammaln, multigammaln

from .cavi import Hyper, NumericFailure

CHUNK_GENES = 4096  # the smallest chunk
GROUP_CHUNKS = 64   # chunks of CHUNK_GENES per group
GROUP_GENES = CHUNK_GENES * GROUP_CHUNKS


def plan_chunk_genes(V_total: int, d: int) -> int:
    """Genes per chunk of a dataset (engine.cuh plan_chunk_genes)."""
    return 8192 if d >= 3 and V_total >= (1 << 23) else CHUNK_GENES
N_OCTANTS = 8
LN2PI = np.log(2.0 * np.pi)


def n_stats(d: int) -> int:
    """[g (d) | G upper | R | Q | Ld] -- the device statistic vector."""
    return d + d * (d + 1) // 2 + 3


def triu_index(d: int):
    return [(j, k) for j in range(d) for k in range(j, d)]


# ------------------------------------------------------------------ plan
@dataclass(frozen=True)
class Plan:
    V: int
    n_chunks: int
    n_groups: int
    groups_per_octant: int

    def octant_genes(self, o: int):
        per = self.groups_per_octant * GROUP_GENES
        lo = min(o * per, self.V)
        return lo, min(lo + per, self.V)


def make_plan(V: int) -> Plan:
    nc = max(1, -(-V // CHUNK_GENES))
    ng = -(-nc // GROUP_CHUNKS)
    return Plan(V, nc, ng, -(-ng // N_OCTANTS))


def shard_ranges(V: int, world: int):
    """Gene range [lo, hi) per rank; ranks own 8/world consecutive octants."""
    if world not in (1, 2, 4, 8):
        raise ValueError("world size must be 1, 2, 4 or 8")
    p = make_plan(V)
    per = N_OCTANTS // world
    return [(p.octant_genes(r * per)[0], p.octant_genes(r * per + per - 1)[1]) for r in range(world)]


def tree8(parts):
    """Pairwise tree over a power-of-two list (top of the octant tree)."""
    parts = list(parts)
    while len(parts) > 1:
        parts = [parts[i] + parts[i + 1] for i in range(0, len(parts), 2)]
    return parts[0]


# ------------------------------------------------------------------ the pass
@dataclass(frozen=True)
class Generator:
    c: np.ndarray      # (d,) mean shift: k0k of the previous state (K0 at init)
    A: np.ndarray      # (d,d) shared precision E[Lambda] used (Lambda0 at init)
    Ainv: np.ndarray   # (d,d) its inverse
    lnA: float         # ln|A|
    e_rho: float       # E[rho] used (0 at init)


def gene_terms(x, D, gen: Generator):
    """Per-gene contributions (V, n_stats)."""
    d = D.shape[1]
    u = D @ gen.Ainv
    s = np.einsum("vi,vi->v", u, D)
    t = D @ gen.c
    den = 1.0 + gen.e_rho * s
    w = gen.e_rho * (x - t) / den
    gam = w * w - gen.e_rho / den
    res = (x - t - s * w) ** 2 + s / den
    cols = [w * D[:, j] for j in range(d)]
    cols += [gam * D[:, j] * D[:, k] for j, k in triu_index(d)]
    cols += [res, w * (x - t), np.log(den)]
    return np.stack(cols, axis=1)


def local_stats(x, D, gen: Generator, gene_lo: int, V_total: int):
    """Per-octant sums of genes [gene_lo, gene_lo+len(x)) (zeros outside the range)."""
    p = make_plan(V_total)
    ns = n_stats(D.shape[1])
    cg = plan_chunk_genes(V_total, D.shape[1])
    terms = gene_terms(x, D, gen) if x.shape[0] else np.zeros((0, ns))
    octs = []
    for o in range(N_OCTANTS):
        lo, hi = p.octant_genes(o)
        lo_l, hi_l = max(lo, gene_lo), min(hi, gene_lo + x.shape[0])
        if (lo, hi) != (lo_l, hi_l) and lo_l < hi_l:
            raise ValueError("shard boundary does not align with octants")
        acc = np.zeros(ns)
        if lo_l < hi_l:
            gsums = []
            for g0 in range(lo_l, hi_l, GROUP_GENES):
                csums = [terms[c0 - gene_lo: min(c0 + cg, hi_l) - gene_lo].sum(axis=0)
                         for c0 in range(g0, min(g0 + GROUP_GENES, hi_l), cg)]
                gsums.append(warp_rows_sum(csums))
            acc = warp_rows_sum(gsums)
        octs.append(acc)
    return octs


def warp_rows_sum(rows):
    """The device's row reduction (pass.cuh warp_sum_rows): lane l adds rows l, l+32, ... in
    index order from 0.0, then an xor butterfly over 32 lanes; lane 0's value."""
    ns = rows[0].shape[0]
    lanes = [np.zeros(ns) for _ in range(32)]
    for i, r in enumerate(rows):
        lanes[i % 32] = lanes[i % 32] + r
    for off in (16, 8, 4, 2, 1):
        lanes = [lanes[l] + lanes[l ^ off] for l in range(32)]
    return lanes[0]


def combine(rank_partials):
    """Top of the octant tree over the ranks' subtree partials."""
    return tree8(rank_partials)


def full_stats(x, D, gen: Generator):
    octs = local_stats(x, D, gen, 0, x.shape[0])
    return tree8(octs)


def streamed_stats(x, D, gen: Generator):
    """full_stats with memory bounded by one group: the per-gene terms are formed one group
    (GROUP_CHUNKS chunks) at a time, so the plan runs at V = 1e8-1e9 on a host (the same
    chunk -> group -> octant -> tree8 sums as local_stats)."""
    V = x.shape[0]
    p = make_plan(V)
    ns = n_stats(D.shape[1])
    step = GROUP_GENES
    cg = plan_chunk_genes(V, D.shape[1])
    gsums = []
    for g0 in range(0, V, step):
        hi = min(g0 + step, V)
        t = gene_terms(x[g0:hi], D[g0:hi], gen)
        gsums.append(warp_rows_sum([t[c0:c0 + cg].sum(axis=0) for c0 in range(0, hi - g0, cg)]))
    octs = []
    for o in range(N_OCTANTS):
        a, b = o * p.groups_per_octant, min((o + 1) * p.groups_per_octant, p.n_groups)
        octs.append(warp_rows_sum(gsums[a:b]) if b > a else np.zeros(ns))
    return tree8(octs)


def rank_partial(x_all, D_all, gen: Generator, rank: int, world: int):
    """The partial rank `rank` of `world` contributes (its octant subtree)."""
    V = x_all.shape[0]
    lo, hi = shard_ranges(V, world)[rank]
    octs = local_stats(x_all[lo:hi], D_all[lo:hi], gen, lo, V)
    per = N_OCTANTS // world
    return tree8(octs[rank * per:(rank + 1) * per])


# ------------------------------------------------------------------ tail
@dataclass(frozen=True)
class Globals:
    a_rho: float
    b_rho: float
    k0k: np.ndarray
    lam0l_inv: np.ndarray
    ln_det_l: float       # ln|lam0l_inv|
    e_lam: np.ndarray     # (n0+V) inv(lam0l_inv)
    e_rho: float          # a_rho / b_rho


def chol_inv_logdet(M):
    L = np.linalg.cholesky(M)
    Li = np.linalg.inv(L)
    return Li.T @ Li, 2.0 * np.sum(np.log(np.diag(L)))


def unpack(stats, d):
    g = stats[:d]
    G = np.zeros((d, d))
    for idx, (j, k) in enumerate(triu_index(d)):
        G[j, k] = G[k, j] = stats[d + idx]
    return g, G, float(stats[-3]), float(stats[-1])


def elbo(stats, gen: Generator, st: Globals, hp: Hyper, V: int) -> float:
    d = hp.dim
    nu, qv = hp.n0 + V, hp.q0 + V
    g, G, R, Ld = unpack(stats, d)
    S, ln_s = chol_inv_logdet(st.lam0l_inv)
    ln_s = -st.ln_det_l
    e_rho = st.a_rho / st.b_rho
    e_lnrho = float(digamma(st.a_rho) - np.log(st.b_rho))
    e_lnlam = float(np.sum(digamma(0.5 * (nu + 1 - np.arange(1, d + 1))))) + d * np.log(2.0) + ln_s
    h = gen.Ainv @ g
    dlt = st.k0k - gen.c
    scat = V * gen.Ainv + gen.Ainv @ G @ gen.Ainv - np.outer(dlt, h) - np.outer(h, dlt) + V * np.outer(dlt, dlt)
    ldsig = -(V * gen.lnA + Ld)
    lik = 0.5 * V * (e_lnrho - LN2PI) - 0.5 * e_rho * R
    tb = 0.5 * V * e_lnlam - 0.5 * V * d * LN2PI - 0.5 * (nu * float(np.sum(S * scat)) + V * d / qv)
    dk = st.k0k - hp.K0
    tk = 0.5 * d * np.log(hp.q0) - 0.5 * d * LN2PI + 0.5 * e_lnlam - 0.5 * hp.q0 * (nu * float(dk @ S @ dk) + d / qv)
    L0i = np.linalg.inv(hp.Lambda0)
    tl = 0.5 * (hp.n0 - d - 1) * e_lnlam - 0.5 * nu * float(np.sum(L0i * S))
    if hp.n0 > d - 1:
        ld0 = np.linalg.slogdet(hp.Lambda0)[1]
        tl -= 0.5 * hp.n0 * d * np.log(2.0) + 0.5 * hp.n0 * ld0 + multigammaln(0.5 * hp.n0, d)
    tr = hp.a0 * np.log(hp.b0) - gammaln(hp.a0) + (hp.a0 - 1.0) * e_lnrho - hp.b0 * e_rho
    hb = 0.5 * ldsig + 0.5 * V * d * (1.0 + LN2PI)
    hr = st.a_rho - np.log(st.b_rho) + gammaln(st.a_rho) + (1.0 - st.a_rho) * digamma(st.a_rho)
    qk = 0.5 * d * np.log(qv) - 0.5 * d * LN2PI + 0.5 * e_lnlam - 0.5 * d
    if nu <= d - 1:
        raise NumericFailure("Q(Lambda) is improper; dataset too small")
    zq = 0.5 * nu * d * np.log(2.0) + 0.5 * nu * ln_s + multigammaln(0.5 * nu, d)
    ql = 0.5 * (nu - d - 1) * e_lnlam - 0.5 * nu * d - zq
    return float(lik + tb + tk + tl + tr + hb + hr - qk - ql)


def init(hp: Hyper, V: int):
    nu = hp.n0 + V
    L0i, ld0 = chol_inv_logdet(hp.Lambda0)
    gen = Generator(hp.K0.copy(), hp.Lambda0.copy(), L0i, ld0, 0.0)
    st = Globals(hp.a0, hp.b0, hp.K0.copy(), hp.Lambda0.copy(), ld0, nu * L0i, hp.a0 / hp.b0)
    return gen, st


def sweep_generator(st: Globals, resid: float, hp: Hyper, V: int):
    """Expectations + rho block entering a sweep (vb.py:136-144)."""
    nu = hp.n0 + V
    a = hp.a0 + 0.5 * V
    b = hp.b0 + 0.5 * resid
    e_rho = a / b
    gen = Generator(st.k0k.copy(), st.e_lam, st.lam0l_inv / nu, d_lnnu(hp.dim, nu) - st.ln_det_l, e_rho)
    return gen, a, b


def d_lnnu(d, nu):
    return d * np.log(nu)


def sweep_tail(stats, gen: Generator, a: float, b: float, hp: Hyper, V: int) -> Globals:
    """(K, Lambda) block from the pass statistics, centred form (vb.py:172-197)."""
    d = hp.dim
    nu, qv = hp.n0 + V, hp.q0 + V
    g, G, _, _ = unpack(stats, d)
    h = gen.Ainv @ g
    k0c = hp.K0 - gen.c
    dlt = (h + hp.q0 * k0c) / qv
    k_new = gen.c + dlt
    L0i = np.linalg.inv(hp.Lambda0)
    L = L0i + V * gen.Ainv + gen.Ainv @ G @ gen.Ainv + hp.q0 * np.outer(k0c, k0c) - qv * np.outer(dlt, dlt)
    L = 0.5 * (L + L.T)
    S, ldl = chol_inv_logdet(L)
    return Globals(a, b, k_new, L, ldl, nu * S, a / b)


def rel_delta(new, old):
    den = max(float(np.max(np.abs(old))), 1e-300)
    return float(np.max(np.abs(np.asarray(new) - np.asarray(old)))) / den


def fit(r, mu, D, hp: Hyper, max_iter=300, rel_tol=1e-8, compute_elbo=True, param_tol=1e-10, x=None,
        stats_fn=None):
    """Single-pass CAVI fit; returns (Globals, trace dict, n_iter).  `x` = r - mu if already
    formed; `stats_fn` = streamed_stats for datasets too large to hold the per-gene terms."""
    V = D.shape[0]
    x = r - mu if x is None else x
    full_stats = stats_fn or globals()["full_stats"]
    gen, st = init(hp, V)
    resid = float(full_stats(x, D, gen)[-3])
    es, dk, dr, dl = [], [], [], []
    prev = None
    for _ in range(max_iter):
        gen, a, b = sweep_generator(st, resid, hp, V)
        stats = full_stats(x, D, gen)
        new = sweep_tail(stats, gen, a, b, hp, V)
        dk.append(rel_delta(new.k0k, st.k0k))
        dr.append(rel_delta(new.e_rho, st.e_rho))
        dl.append(rel_delta(new.lam0l_inv, st.lam0l_inv))
        st = new
        resid = float(stats[-3])
        if compute_elbo:
            e = elbo(stats, gen, st, hp, V)
            es.append(e)
            if prev is not None and abs(e - prev) < rel_tol * abs(e):
                break
            prev = e
        else:
            es.append(np.nan)
            if max(dk[-1], dr[-1], dl[-1]) < param_tol:
                break
    return st, {"elbo": np.array(es), "delta_k0k": np.array(dk), "delta_rho": np.array(dr),
                "delta_lam": np.array(dl)}, len(es)
