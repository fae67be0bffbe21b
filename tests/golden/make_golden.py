"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (the reference is importable there, not on the GPU
box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/<case>.npz.  Each file holds
  * `recipe`   -- JSON describing how the dataset is built (oracle.philox can
                  rebuild it bit-exactly) plus sha256 of r, mu, D,
  * the reference `vb_fit` outputs: ELBO trace, parameter deltas, iteration
    count, final globals (a_rho, b_rho, k0k, lam0l_inv, e_lam, e_rho, e_lamk),
    per-gene moments (mu_beta, lam_beta, e_bbt) on a fixed gene subset,
  * for `step_*` cases, the state after vb_init and after each of 3 vb_step
    calls, with vb_elbo of each.
The reference path: tissuemix.vb.vb_fit / vb_init / vb_step / vb_elbo
(reference vb.py:82-354), data from tissuemix.model.random_profiles +
synth_generate (model.py:224-270).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

from tissuemix import model, vb  # the reference
from tissuemix.samplers import RngStream

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LAM = np.linalg.inv(model.REFERENCE_LAMBDA_INV)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def regime(V, seed, N, K=None, rho=100.0):
    """reference tests/conftest.py:15-26."""
    if N == 3:
        lam = REF_LAM
        K = np.array([0.1, 0.3]) if K is None else np.asarray(K, float)
    else:
        lam = np.linalg.inv(0.01 * np.eye(N - 1))
        K = np.full(N - 1, 0.2) if K is None or len(K) != N - 1 else np.asarray(K, float)
    truth = model.ModelParams(K=K, Lam=lam, rho=rho)
    rng = RngStream(seed)
    ds = model.synth_generate(rng, truth, model.random_profiles(rng, V, N))
    recipe = {"kind": "random", "V": V, "seed": seed, "N": N, "K": list(map(float, K)),
              "Lam": lam.tolist(), "rho": rho}
    return ds, recipe


def fixed_profiles(codes_bits, seed, K, lam, rho):
    profs = [model.ExpressionProfile(np.array(b, dtype=float)) for b in codes_bits]
    truth = model.ModelParams(K=np.asarray(K, float), Lam=np.asarray(lam, float), rho=rho)
    ds = model.synth_generate(RngStream(seed), truth, profs)
    recipe = {"kind": "fixed", "profiles": [list(map(float, b)) for b in codes_bits], "seed": seed,
              "K": list(map(float, np.atleast_1d(K))), "Lam": np.atleast_2d(lam).tolist(), "rho": rho}
    return ds, recipe


def hyper_recipe(hp):
    return {"a0": hp.a0, "b0": hp.b0, "q0": hp.q0, "n0": hp.n0, "K0": hp.K0.tolist(),
            "Lambda0": hp.Lambda0.tolist()}


def subset(V):
    return np.unique(np.array([0, 1, 2, V // 3, V // 2, V - 2, V - 1]).clip(0, V - 1))


def save_fit(name, ds, recipe, hp, kw):
    state, tr = vb.vb_fit(ds, hp, **kw)
    idx = subset(ds.V)
    recipe = dict(recipe, sha_r=sha(ds.r), sha_mu=sha(ds.mu), sha_D=sha(ds.D))
    out = dict(
        recipe=json.dumps(recipe), hyper=json.dumps(hyper_recipe(hp)), fit_kw=json.dumps(kw),
        elbo=tr.elbo, delta_k0k=tr.delta_k0k, delta_rho=tr.delta_rho, delta_lam=tr.delta_lam,
        n_iter=len(tr), a_rho=state.a_rho, b_rho=state.b_rho, k0k=state.k0k,
        lam0l_inv=state.lam0l_inv, e_lam=state.e_lam, e_rho=state.e_rho, e_lamk=state.e_lamk,
        idx=idx, mu_beta=state.mu_beta[idx], lam_beta=state.lam_beta[idx], e_bbt=state.e_bbt[idx],
    )
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(f"{name}: V={ds.V} N={ds.n_networks} iters={len(tr)} elbo={tr.elbo[-1]!r}")


def save_steps(name, ds, recipe, hp, n_steps=3):
    idx = subset(ds.V)
    recipe = dict(recipe, sha_r=sha(ds.r), sha_mu=sha(ds.mu), sha_D=sha(ds.D))
    st = vb.vb_init(ds, hp)
    rows = {k: [] for k in ("a_rho", "b_rho", "k0k", "lam0l_inv", "e_lam", "e_rho", "e_lamk",
                            "elbo", "mu_beta", "lam_beta", "e_bbt")}
    for i in range(n_steps + 1):
        if i:
            st = vb.vb_step(st, ds, hp)
        for k in rows:
            if k == "elbo":
                rows[k].append(vb.vb_elbo(st, ds, hp))
            elif k in ("mu_beta", "lam_beta", "e_bbt"):
                rows[k].append(getattr(st, k)[idx])
            else:
                rows[k].append(getattr(st, k))
    out = {k: np.array(v) for k, v in rows.items()}
    np.savez_compressed(os.path.join(HERE, name + ".npz"), recipe=json.dumps(recipe),
                        hyper=json.dumps(hyper_recipe(hp)), idx=idx, **out)
    print(f"{name}: V={ds.V} steps={n_steps} elbo={out['elbo'][-1]!r}")


def save_posterior(name, ds, recipe, hp, fit_kw, seed, n, stream_id=0, pre_block=0):
    """vb_posterior_sample (vb.py:357-393) of the reference's own fitted state."""
    state, _ = vb.vb_fit(ds, hp, **fit_kw)
    rng = RngStream(seed, stream_id, pre_block)
    draws = vb.vb_posterior_sample(rng, state, hp, ds.V, n)
    recipe = dict(recipe, sha_r=sha(ds.r), sha_mu=sha(ds.mu), sha_D=sha(ds.D))
    np.savez_compressed(os.path.join(HERE, name + ".npz"), recipe=json.dumps(recipe),
                        hyper=json.dumps(hyper_recipe(hp)), fit_kw=json.dumps(fit_kw), seed=seed,
                        stream_id=stream_id, pre_block=pre_block, n=n, end_block=rng._block, V=ds.V,
                        a_rho=state.a_rho, b_rho=state.b_rho, k0k=state.k0k, lam0l_inv=state.lam0l_inv,
                        K=draws["K"], Lambda=draws["Lambda"], rho=draws["rho"])
    print(f"{name}: V={ds.V} n={n} end_block={rng._block}")


def save_em(name, ds, recipe, hp, kw):
    """em.em_fit from the reference CLI's init (K0, Lambda0, rho=1; test_acceptance.py:60)."""
    from tissuemix import em  # the reference

    init = model.ModelParams(K=hp.K0, Lam=hp.Lambda0, rho=1.0)
    params, tr = em.em_fit(ds, init, **kw)
    st = em.em_step(em.EmState(params=init, Sigma=np.empty(0), M=np.empty(0), S=np.empty(0)), ds)
    idx = subset(ds.V)
    recipe = dict(recipe, sha_r=sha(ds.r), sha_mu=sha(ds.mu), sha_D=sha(ds.D))
    np.savez_compressed(os.path.join(HERE, name + ".npz"), recipe=json.dumps(recipe),
                        hyper=json.dumps(hyper_recipe(hp)), fit_kw=json.dumps(kw),
                        init_K=hp.K0, init_Lam=hp.Lambda0, init_rho=1.0,
                        K=params.K, Lam=params.Lam, rho=params.rho, loglik=tr.loglik, tr_K=tr.K, tr_rho=tr.rho,
                        n_iter=len(tr), step_K=st.params.K, step_Lam=st.params.Lam, step_rho=st.params.rho,
                        idx=idx, step_Sigma=st.Sigma[idx], step_M=st.M[idx], step_S=st.S[idx])
    print(f"{name}: V={ds.V} iters={len(tr)} ll={tr.loglik[-1]!r}")


def main(which=None):
    cases = []
    # config 1: the reference's own test scale, CAVI to convergence
    cases.append(("fit_n2_v4000", lambda: (*regime(4000, 1, 2), model.default_hyperparams(2), {})))
    cases.append(("fit_n3_v4000_t1", lambda: (*regime(4000, 404, 3), model.default_hyperparams(3),
                                               {"max_iter": 3000})))
    cases.append(("fit_n3_v4000_cap300", lambda: (*regime(4000, 404, 3), model.default_hyperparams(3), {})))
    cases.append(("fit_n3_v120", lambda: (*regime(120, 21, 3), model.default_hyperparams(3), {"max_iter": 20})))
    # K=4 (d=3) and the K sweep shapes
    cases.append(("fit_n4_v20000", lambda: (*regime(20000, 2026, 4), model.default_hyperparams(4),
                                             {"max_iter": 60})))
    cases.append(("fit_n5_v3000", lambda: (*regime(3000, 5, 5), model.default_hyperparams(5), {"max_iter": 30})))
    cases.append(("fit_n8_v3000", lambda: (*regime(3000, 8, 8), model.default_hyperparams(8), {"max_iter": 20})))
    cases.append(("fit_n16_v3000", lambda: (*regime(3000, 16, 16), model.default_hyperparams(16),
                                             {"max_iter": 12})))
    # edge cases from the reference's own tests
    cases.append(("fit_flat_v80", lambda: (*fixed_profiles([[1, 1, 1]] * 80, 12, [0.1, 0.3], REF_LAM, 100.0),
                                            model.default_hyperparams(3), {"max_iter": 500, "rel_tol": 1e-12})))
    cases.append(("fit_v1_n2", lambda: (*fixed_profiles([[1, 0]], 10, [0.4], [[100.0]], 100.0),
                                         model.default_hyperparams(2), {"max_iter": 400})))
    cases.append(("fit_v5_proper", lambda: (*regime(5, 9, 3), model.HyperParams(
        a0=0.5, b0=0.5, q0=0.001, n0=3, K0=np.full(2, 1 / 3), Lambda0=REF_LAM), {"max_iter": 150})))
    cases.append(("fit_v1_n3", lambda: (*regime(1, 5, 3), model.default_hyperparams(3), {"max_iter": 1})))
    cases.append(("fit_paramtol_v60", lambda: (*regime(60, 13, 3), model.default_hyperparams(3),
                                                {"max_iter": 4000, "compute_elbo": False, "param_tol": 1e-11})))
    cases.append(("fit_v257_perm", lambda: (*regime(257, 6, 3), model.default_hyperparams(3), {"max_iter": 40})))
    # config 4: fibroblast-shaped (V=56, N=3, K=(0.65, 0.28), rho=5; test_acceptance.py:394-399)
    for s in range(8):
        cases.append((f"fit_fibro56_s{s}", (lambda s=s: (*regime(56, 560 + s, 3, K=[0.65, 0.28], rho=5.0),
                                                          model.default_hyperparams(3), {}))))
    # step-level goldens
    cases.append(("steps_n3_v30", lambda: (*regime(30, 4, 3), model.default_hyperparams(3))))
    cases.append(("steps_n4_v300", lambda: (*regime(300, 7, 4), model.default_hyperparams(4))))
    cases.append(("steps_n2_v50", lambda: (*regime(50, 3, 2), model.default_hyperparams(2))))

    # posterior draws (vb_posterior_sample): chunked (small nu*d) and one-draw-per-chunk regimes
    post = [("post_n3_v50", lambda: (*regime(50, 16, 3), model.default_hyperparams(3), {"max_iter": 40}, 91, 500)),
            ("post_n4_v200", lambda: (*regime(200, 15, 4), model.default_hyperparams(4), {"max_iter": 60}, 7, 300, 3, 11)),
            ("post_n2_v3000", lambda: (*regime(3000, 4, 2), model.default_hyperparams(2), {"max_iter": 30}, 5, 64)),
            ("post_n3_v700k", lambda: (*regime(700_000, 2, 3), model.default_hyperparams(3), {"max_iter": 3}, 12, 4))]
    for name, make in post:
        if which and name not in which:
            continue
        save_posterior(name, *make())

    ems = [("em_n3_v4000", lambda: (*regime(4000, 404, 3), model.default_hyperparams(3), {})),
           ("em_n4_v3000", lambda: (*regime(3000, 3, 4), model.default_hyperparams(4), {"max_iter": 300})),
           ("em_n3_v50", lambda: (*regime(50, 40, 3), model.default_hyperparams(3), {"max_iter": 150})),
           ("em_n2_v500", lambda: (*regime(500, 8, 2), model.default_hyperparams(2), {"max_iter": 500})),
           ("em_n8_v2000", lambda: (*regime(2000, 9, 8), model.default_hyperparams(8), {"max_iter": 40}))]
    for name, make in ems:
        if which and name not in which:
            continue
        save_em(name, *make())

    for name, make in cases:
        if which and name not in which:
            continue
        built = make()
        if name.startswith("steps_"):
            save_steps(name, *built)
        else:
            save_fit(name, *built)


if __name__ == "__main__":
    main(sys.argv[1:] or None)
