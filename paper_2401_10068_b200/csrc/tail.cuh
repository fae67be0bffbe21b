// tail.cuh -- the sweep tail of the streaming engine as ONE WARP over shared memory.
//
// Restates, from one pass's statistics [g | G upper | R | Q | Ld] (engine.cuh), the
// reference's (K, Lambda) block (vb.py:172-197) in centred form, the rho block of the next
// sweep (vb.py:141-144), the bound (vb.py:216-304), the fit loop's deltas and stop rule
// (vb.py:307-347) and vb_init's globals (vb.py:82-111) -- the same per-element formulas as the
// single-thread tail_t (engine.cuh), which the batched kernel keeps (a fit group's first lane).
//
// Why a warp and shared memory: the tail is on the critical path of every sweep (the next
// pass waits for it).  The single-thread version kept d x d blocks in registers / the stack
// (tail_kernel<6>: 409 LDL / 534 STL; <15>: 8.8k LDL) and ran every O(d^2) / O(d^3) loop
// serially.  Here:
//   phase 0  every global word the tail reads (statistics of all ranks, the pass's generator,
//            the previous state, the hyperparameters: ~110 words at d = 3, ~1.4k at d = 15) is
//            gathered by all 32 lanes in one burst of independent loads -> one L2 round trip;
//   phase 1  A^-1 G A^-1 and A^-1 g, element-parallel;
//   phase 2  the new Q(Lambda) rate, one element per lane; its inverse + log|det| with the
//            reference's semantics (adjugate + det guard for d <= 3, pivoted elimination above,
//            jitter-once retry, linalg.py:111-192, 279-298): lane 0 for d <= 3, the warp above;
//   phase 3  the bound's three d x d contractions as lane partials + butterflies, the scalar
//            assembly on lane 0; E[Lambda K] by rows; the deltas as warp max-reductions;
//   phase 4  every store lane-parallel (state, trace entry, the next pass's generator).
// No local memory at any d; every read of the control block precedes every write to it.
#pragma once

#include "engine.cuh"

namespace cavi {

template <int D>
struct TailSm {
  static constexpr int NS = n_stats(D);
  static constexpr int D2 = D * D;
  double tot[NS];
  double gc[D], gA[D2], gAi[D2], gsc[2];  // generator of the pass: c, A, A^-1, (lnA, e_rho)
  double k_old[D], l_old[D2], osc[4];     // previous state: k0k, lam0l_inv, (e_rho, a, b, ln|lam0l_inv|)
  double K0[D], L0[D2], L0i[D2];
  double hv[D], AG[D2], T[D2], k0c[D], dlt[D], k_new[D];
  double L[D2], C[D2], S[D2], M[2 * D2];
  double ld;
  int ok;
};

// Warp reductions.  Each starts with __syncwarp(): the lane-strided loops before them (an
// unrolled `if (e >= D2) break`) leave the warp diverged, and a shuffle in a diverged warp
// takes the emulated collective path (WARPSYNC.COLLECTIVE, ~10x the instructions).
// NaN-propagating max over the warp (rel_delta_t's `df > md || df != df`)
__device__ __forceinline__ double warp_max_nan(double v) {
  __syncwarp();
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double o = __shfl_xor_sync(0xffffffffu, v, off);
    v = (o > v || o != o) ? o : v;
  }
  return v;
}
__device__ __forceinline__ double warp_fmax(double v) {
  __syncwarp();
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
  __syncwarp();
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// N words global -> shared by the 32 lanes, split in two so that every load of phase 0 is
// issued before the first store that would wait on one (in-order issue: a store stalls the
// warp until its operand arrives, so load/store/load/store costs one round trip per copy)
template <int N>
struct WarpLoad {
  static constexpr int K = (N + 31) / 32;
  double v[K];
  __device__ __forceinline__ void load(const double* __restrict__ src, int lane) {
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (lane + 32 * k < N) v[k] = src[lane + 32 * k];
  }
  __device__ __forceinline__ void store(double* dst, int lane) const {
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (lane + 32 * k < N) dst[lane + 32 * k] = v[k];
  }
};

// Inverse + log|det| of the rate in sm.C -> sm.S, with the reference's semantics
// (ref_inv_once_t: adjugate + |det| guard for d <= 3, pivoted elimination above; jitter-once
// retry; no positive-definiteness test).  Lane 0 holds *ld; returns ok on every lane.  Up to
// kTailSerialD on lane 0 in registers (a d = 3 adjugate is a short dependent chain); beyond
// it, across the warp (ref_inv_logdet_warp).
constexpr int kTailSerialD = 3;
template <int D>
__device__ __forceinline__ bool tail_inverse(TailSm<D>& sm, double* ld, int lane) {
  if constexpr (D <= kTailSerialD) {
    int ok = 0;
    double l = 0.0;
    if (lane == 0) {
      double A[D * D], S[D * D];
#pragma unroll
      for (int e = 0; e < D * D; ++e) A[e] = sm.C[e];
      ok = spd_inv_logdet_t<D>(A, S, &l) ? 1 : 0;
#pragma unroll
      for (int e = 0; e < D * D; ++e) sm.S[e] = S[e];
    }
    __syncwarp();
    *ld = l;
    return __shfl_sync(0xffffffffu, ok, 0) != 0;
  } else {
    double l = 0.0;
    const bool ok = ref_inv_logdet_warp<D>(sm.C, sm.AG, sm.M, sm.S, &l, lane);
    *ld = l;
    return __shfl_sync(0xffffffffu, (int)(ok && isfinite(l)), 0) != 0;
  }
}

// EM (reference em.py:44-124) from the same statistics.  One pass with the generator
// theta_n = (K, Lambda, Lambda^-1, rho) yields both the marginal log-likelihood of theta_n
// (model.py:278-287: ll = -1/2 [V ln 2pi + sum ln den - V ln rho + sum rho (x - t)^2 / den] from
// Ld and Q) and the E-step sums of em.py:44-77 for theta_{n+1}; the joint M-step (em.py:80-94)
// in centred form: rho' = V / R, h = Lambda^-1 g, K' = K + h / V,
// Lambda'^-1 = Lambda^-1 + Lambda^-1 G Lambda^-1 / V - h h^T / V^2, Lambda' = inv(.).  Trace entry
// n-1 is ll(theta_n); stop when |ll_n - ll_{n-1}| < rel_tol |ll_n| or after max_iter M-steps.  sm.hv / sm.T hold
// A^-1 g and A^-1 G A^-1 of the generator theta_n (phase 1 of tail_warp).
template <int D>
__device__ __forceinline__ void em_tail_warp(Ctl* c, TailSm<D>& sm, int lane, double V, int n, int max_iter,
                                             int tr_cap, double prev_elbo, double rel_tol, double g_erho,
                                             double* tr_elbo, double* tr_drho, double* tr_k) {
  constexpr int D2 = D * D;
  cv_state& s = c->cur;
  int done = 0;
  double R = 0.0;
  if (lane == 0) {
    const double ll =
        -0.5 * (V * kLn2Pi + sm.tot[stat_Ld(D)] - V * log(g_erho) + sm.tot[stat_Q(D)]);
    if (n >= 1) {
      const int it = n - 1;
      if (it < tr_cap) {
        tr_elbo[it] = ll;
        tr_drho[it] = g_erho;
        for (int j = 0; j < D; ++j) tr_k[(size_t)it * D + j] = sm.gc[j];
      }
      if (fabs(ll - prev_elbo) < rel_tol * fabs(ll)) done = 1;
      if (n >= max_iter) done = 1;
    }
    c->prev_elbo = ll;
    s.d = D;
    s.n_iter = n;
    s.elbo = ll;
    s.e_rho = g_erho;
    c->iter = n + 1;
    R = sm.tot[stat_R(D)];
    if (!done && (!(R > 0.0) || !isfinite(R))) {  // "non-positive residual sum in M-step" (em.py:85-86)
      c->status = CV_ERR_NUMERIC;
      done = 1;
    }
    if (done) c->done = 1;
  }
  if (lane < D) s.k0k[lane] = sm.gc[lane];
  #pragma unroll
  for (int m_ = 0; m_ < (D2 + 31) / 32; ++m_) {
    const int e = lane + 32 * m_;
    if (e >= D2) break;
    s.lam0l_inv[e] = sm.gA[e];  // EM: the current precision Lambda
    s.e_lam[e] = sm.gAi[e];     //     and its inverse
  }
  __syncwarp();
  if (__shfl_sync(0xffffffffu, done, 0)) return;
  const double rV = 1.0 / V;
  #pragma unroll
  for (int m_ = 0; m_ < (D2 + 31) / 32; ++m_) {
    const int e = lane + 32 * m_;
    if (e >= D2) break;
    const int i = e / D, j = e % D;
    const int p = i < j ? i : j, q = i < j ? j : i;
    const double v = 0.5 * (sm.gAi[p * D + q] + sm.gAi[q * D + p]) + sm.T[p * D + q] * rV - sm.hv[p] * sm.hv[q] * rV * rV;
    sm.L[e] = v;
    sm.C[e] = v;
  }
  __syncwarp();
  double ldx = 0.0;
  if (!tail_inverse<D>(sm, &ldx, lane)) {  // "M-step precision" inversion failed
    if (lane == 0) {
      c->status = CV_ERR_NUMERIC;
      c->done = 1;
    }
    return;
  }
  if (lane < D) c->pass.c[lane] = sm.gc[lane] + sm.hv[lane] * rV;
  #pragma unroll
  for (int m_ = 0; m_ < (D2 + 31) / 32; ++m_) {
    const int e = lane + 32 * m_;
    if (e >= D2) break;
    const int i = e / D, j = e % D;
    c->pass.A[e] = 0.5 * (sm.S[i * D + j] + sm.S[j * D + i]);
    c->pass.Ainv[e] = sm.L[e];
  }
  if (lane == 0) {
    c->pass.lnA = -ldx;
    c->pass.e_rho = V / R;
  }
}

// The hyperparameter words the tail reads.  They are constant through a fit (set up before its
// first pass), so tail_kernel loads them BEFORE griddepcontrol.wait -- under programmatic
// dependent launch while the pass still streams -- and the post-wait burst is only the control
// block, the previous state and the pass's statistics.
template <int D>
struct TailHyp {
  WarpLoad<D> K0;
  WarpLoad<D * D> L0, L0i;
  double V, nu, qv, q0;
  double a0 = 0, b0 = 0, lnL0 = 0, a_fit = 0, ln_nu = 0, dg_afit = 0, lg_afit = 0, dg_a0 = 0, lg_a0 = 0, sum_dg_nu = 0,
         ln_q0 = 0, ln_qv = 0, ln_b0 = 0, zprior = 0, mgl_nu = 0;
  int n0 = 0, has_zprior = 0, proper_q = 1;
  __device__ __forceinline__ void load(const Hyp* __restrict__ hp, int lane) {
    K0.load(hp->K0, lane);
    L0.load(hp->L0, lane);
    L0i.load(hp->L0inv, lane);
    V = hp->V;
    nu = hp->nu;
    qv = hp->qv;
    q0 = hp->q0;
    if (lane == 0) {  // lane 0's scalars: every hyperparameter constant the bound uses
      a0 = hp->a0; b0 = hp->b0; lnL0 = hp->lnL0; a_fit = hp->a_fit; ln_nu = hp->ln_nu;
      dg_afit = hp->dg_afit; lg_afit = hp->lg_afit; dg_a0 = hp->dg_a0; lg_a0 = hp->lg_a0; sum_dg_nu = hp->sum_dg_nu;
      ln_q0 = hp->ln_q0; ln_qv = hp->ln_qv; ln_b0 = hp->ln_b0; zprior = hp->zprior; mgl_nu = hp->mgl_nu;
      n0 = hp->n0; has_zprior = hp->has_zprior; proper_q = hp->proper_q;
    }
  }
};

// The sweep tail (MODE_SWEEP, MODE_INIT, MODE_ELBO, MODE_EM) run by one warp.  `parts` holds
// the `world` rank partials to combine into sm.tot, unless the fused exchange already did
// (parts == nullptr).  Every global word the tail needs -- including the done flag, which is
// tested only afterwards -- is requested in ONE burst: the tail pays one L2 round trip for its
// inputs, not one per dependent step.
template <int D>
__device__ __forceinline__ void tail_warp(const TailHyp<D>& th, Ctl* c, const double* __restrict__ parts, int world,
                                       TailSm<D>& sm, int lane) {
  constexpr int NS = n_stats(D);
  constexpr int D2 = D * D;
  cv_state& s = c->cur;
  // ---- phase 0: one burst of loads (every load issued before the first dependent store)
  constexpr int K = (NS + 31) / 32;  // rank partials -> the fixed pairwise tree (as the fused exchange)
  double v[K][kOctants];
  if (parts) {
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int r = 0; r < kOctants; ++r)
        if (r < world && lane + 32 * k < NS) v[k][r] = __ldcg(parts + r * NS + lane + 32 * k);
  }
  WarpLoad<D> l_gc, l_ko;
  WarpLoad<D2> l_gA, l_gAi, l_lo;
  l_gc.load(c->pass.c, lane);
  l_gA.load(c->pass.A, lane);
  l_gAi.load(c->pass.Ainv, lane);
  l_ko.load(s.k0k, lane);
  l_lo.load(s.lam0l_inv, lane);
  const int done_in = *(volatile const int*)&c->done;
  const int mode = c->mode;
  const double V = th.V, nu = th.nu, qv = th.qv, q0 = th.q0;
  const double a0 = th.a0, b0 = th.b0, lnL0 = th.lnL0, a_fit = th.a_fit, ln_nu = th.ln_nu;
  const double dg_afit = th.dg_afit, lg_afit = th.lg_afit, dg_a0 = th.dg_a0, lg_a0 = th.lg_a0,
               sum_dg_nu = th.sum_dg_nu, ln_q0 = th.ln_q0, ln_qv = th.ln_qv, ln_b0 = th.ln_b0, zprior = th.zprior,
               mgl_nu = th.mgl_nu;
  const int n0 = th.n0, has_zprior = th.has_zprior, proper_q = th.proper_q;
  // lane 0's scalars: the control block, the trace pointers and the previous state
  double pend_a = 0, pend_b = 0, prev_elbo = 0, rel_tol = 0, param_tol = 0, g_lnA = 0, g_erho = 0, e_rho_old = 0,
         a_old = 0, b_old = 0, ld_old = 0;
  int compute_elbo = 0, have_prev = 0, iter = 0, max_iter = 0, tr_cap = 0, n_iter_old = 0;
  double *tr_elbo = nullptr, *tr_dk = nullptr, *tr_drho = nullptr, *tr_dlam = nullptr, *tr_k = nullptr;
  if (lane == 0) {
    pend_a = c->pend_a; pend_b = c->pend_b; prev_elbo = c->prev_elbo; rel_tol = c->rel_tol; param_tol = c->param_tol;
    compute_elbo = c->compute_elbo; have_prev = c->have_prev; iter = c->iter; max_iter = c->max_iter;
    tr_cap = c->tr_cap; n_iter_old = s.n_iter;
    tr_elbo = c->tr_elbo; tr_dk = c->tr_dk; tr_drho = c->tr_drho; tr_dlam = c->tr_dlam; tr_k = c->tr_k;
    g_lnA = c->pass.lnA; g_erho = c->pass.e_rho;
    e_rho_old = s.e_rho; a_old = s.a_rho; b_old = s.b_rho; ld_old = s.ln_det_lam0l_inv;
  }
  l_gc.store(sm.gc, lane);
  l_gA.store(sm.gA, lane);
  l_gAi.store(sm.gAi, lane);
  l_ko.store(sm.k_old, lane);
  l_lo.store(sm.l_old, lane);
  th.K0.store(sm.K0, lane);
  th.L0.store(sm.L0, lane);
  th.L0i.store(sm.L0i, lane);
  if (parts) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
      for (int w = 1; w < kOctants; w *= 2)
#pragma unroll
        for (int r = 0; r + w < kOctants; r += 2 * w)
          if (w < world && r + w < world) v[k][r] = v[k][r] + v[k][r + w];
      if (lane + 32 * k < NS) sm.tot[lane + 32 * k] = v[k][0];
    }
  }
  __syncwarp();
  if (done_in) return;  // the fit stopped: this sweep's pass exited at once
  TAIL_PROF(*c, 1);
  // ---- phase 1: T = A^-1 G A^-1 and hv = A^-1 g, element-parallel (d^2/32 dot products of
  // length d per lane, each in the serial code's k order)
  #pragma unroll
  for (int m_ = 0; m_ < (D2 + 31) / 32; ++m_) {
    const int e = lane + 32 * m_;
    if (e >= D2) break;  // G unpacked from the statistics' upper triangle
    const int i = e / D, j = e % D;
    const int lo = i < j ? i : j, hi = i < j ? j : i;
    sm.T[e] = sm.tot[D + lo * D - lo * (lo - 1) / 2 + (hi - lo)];
  }
  if (lane < D) {
    double t = 0.0;
    for (int j = 0; j < D; ++j) t += sm.gAi[lane * D + j] * sm.tot[j];
    sm.hv[lane] = t;
  }
  __syncwarp();
  {
    // this lane's KE elements, the KE dot products interleaved (independent FMA chains: one warp
    // has no other warps to hide a chain's latency behind)
    constexpr int KE = (D2 + 31) / 32;
    int ei[KE], ej[KE];
#pragma unroll
    for (int m = 0; m < KE; ++m) {
      const int e = lane + 32 * m < D2 ? lane + 32 * m : 0;
      ei[m] = e / D;
      ej[m] = e % D;
    }
    double u[KE];
#pragma unroll
    for (int m = 0; m < KE; ++m) u[m] = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k)
#pragma unroll
      for (int m = 0; m < KE; ++m) u[m] += sm.gAi[ei[m] * D + k] * sm.T[k * D + ej[m]];
    __syncwarp();
#pragma unroll
    for (int m = 0; m < KE; ++m)
      if (lane + 32 * m < D2) sm.AG[lane + 32 * m] = u[m];
    __syncwarp();
#pragma unroll
    for (int m = 0; m < KE; ++m) u[m] = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k)
#pragma unroll
      for (int m = 0; m < KE; ++m) u[m] += sm.AG[ei[m] * D + k] * sm.gAi[k * D + ej[m]];
#pragma unroll
    for (int m = 0; m < KE; ++m)
      if (lane + 32 * m < D2) sm.T[lane + 32 * m] = u[m];
  }
  __syncwarp();
  TAIL_PROF(*c, 6);

  if (mode == MODE_EM) {  // EM's trace entry and M-step (em.py:80-124)
    em_tail_warp<D>(c, sm, lane, V, iter, max_iter, tr_cap, prev_elbo, rel_tol, g_erho, tr_elbo, tr_drho, tr_k);
    return;
  }

  // ---- phase 2: the new globals
  bool finite = true;
  for (int i = lane; i < NS; i += 32) finite = finite && isfinite(sm.tot[i]);
  finite = __all_sync(0xffffffffu, finite);
  int status = CV_OK;
  double a = 0, b = 0, e_rho = 0;  // lane 0
  if (mode == MODE_ELBO) {  // vb_elbo of the current state from a pass with its own generator
#pragma unroll
    for (int m_ = 0; m_ < (D2 + 31) / 32; ++m_)
      if (lane + 32 * m_ < D2) sm.C[lane + 32 * m_] = sm.l_old[lane + 32 * m_];
    __syncwarp();
    double ldx = 0.0;
    const bool ok = tail_inverse<D>(sm, &ldx, lane);
    if (lane < D) sm.k_new[lane] = sm.k_old[lane];
    __syncwarp();
    a = a_old;
    b = b_old;
    if (lane == 0) sm.ld = ld_old;  // the bound uses the state's own ln|lam0l_inv| (tail_t)
    if (!ok) status = CV_ERR_NUMERIC;
  } else if (mode == MODE_INIT) {  // vb_init (vb.py:82-111): globals at the prior
    #pragma unroll
    for (int m_ = 0; m_ < (D2 + 31) / 32; ++m_) {
      const int e = lane + 32 * m_;
      if (e >= D2) break;
      sm.L[e] = sm.L0[e];
      sm.S[e] = sm.L0i[e];
    }
    if (lane < D) sm.k_new[lane] = sm.K0[lane];
    if (lane == 0) sm.ld = lnL0;
    a = a0;
    b = b0;
    e_rho = a0 / b0;
  } else {  // (K, Lambda) block, centred (vb.py:172-183)
    const double rqv = 1.0 / qv;
    if (lane < D) {
      const int i = lane;
      sm.k0c[i] = sm.K0[i] - sm.gc[i];
      sm.dlt[i] = (sm.hv[i] + q0 * sm.k0c[i]) * rqv;
      sm.k_new[i] = sm.gc[i] + sm.dlt[i];
    }
    __syncwarp();
    #pragma unroll
    for (int m_ = 0; m_ < (D2 + 31) / 32; ++m_) {
      const int e = lane + 32 * m_;
      if (e >= D2) break;  // the upper-triangle formula, mirrored (as tail_t)
      const int i = e / D, j = e % D;
      const int p = i < j ? i : j, q = i < j ? j : i;
      const double v = sm.L0i[p * D + q] + V * sm.gAi[p * D + q] + sm.T[p * D + q] + q0 * sm.k0c[p] * sm.k0c[q] -
                       qv * sm.dlt[p] * sm.dlt[q];
      sm.L[e] = v;
      sm.C[e] = v;  // the inverse works on a copy (the jitter retry modifies it)
    }
    __syncwarp();
    TAIL_PROF(*c, 7);
    double ldx = 0.0;
    const bool ok = tail_inverse<D>(sm, &ldx, lane);
    if (lane == 0) sm.ld = ldx;  // lane 0 holds the log-det
    if (!finite || !ok) status = CV_ERR_NUMERIC;
    a = pend_a;
    b = pend_b;
    e_rho = g_erho;
  }
  __syncwarp();
  TAIL_PROF(*c, 2);

  // ---- phase 3: the bound (vb.py:216-304 as elbo_t), E[Lambda K], deltas
  double elbo = qnan();
  int elbo_status = CV_OK;
  if (status == CV_OK && (compute_elbo || mode != MODE_SWEEP) && lane == 0 && !proper_q) elbo_status = CV_ERR_IMPROPER;
  __syncwarp();
  elbo_status = __shfl_sync(0xffffffffu, elbo_status, 0);
  const bool want_elbo = __shfl_sync(0xffffffffu, (int)(status == CV_OK && (compute_elbo || mode != MODE_SWEEP)), 0);
  if (want_elbo && elbo_status == CV_OK) {
    double tr1 = 0.0, quad = 0.0, tr0 = 0.0;
    // small d: lane 0 alone (d^2 <= 16 terms cost less than three butterflies); else lane-strided
    constexpr int ES = D <= kTailSerialD ? 1 : 32, KT = D <= kTailSerialD ? D2 : (D2 + 31) / 32;
    const int e0 = D <= kTailSerialD ? (lane == 0 ? 0 : D2) : lane;
#pragma unroll
    for (int m_ = 0; m_ < KT; ++m_) {
      const int e = e0 + ES * m_;
      if (e >= D2) break;
      const int i = e / D, j = e % D;
      const double di = sm.k_new[i] - sm.gc[i], dj = sm.k_new[j] - sm.gc[j];
      const double sc = V * sm.gAi[e] + sm.T[e] - di * sm.hv[j] - sm.hv[i] * dj + V * di * dj;
      const double sij = sm.S[e];
      tr1 += sij * sc;
      quad += (sm.k_new[i] - sm.K0[i]) * sij * (sm.k_new[j] - sm.K0[j]);
      tr0 += sm.L0i[j * D + i] * sij;
    }
    if constexpr (D > kTailSerialD) {
      tr1 = warp_sum(tr1);
      quad = warp_sum(quad);
      tr0 = warp_sum(tr0);
    }
    if (lane == 0) {
      const double R = sm.tot[stat_R(D)], Ld = sm.tot[stat_Ld(D)];
      const double ln_s = -sm.ld;
      const double dga = (a == a_fit) ? dg_afit : (a == a0 ? dg_a0 : digamma_pos(a));
      const double lga = (a == a_fit) ? lg_afit : (a == a0 ? lg_a0 : lgamma(a));
      const double er = a / b;
      const double lnb = log(b);
      const double e_lnrho = dga - lnb;
      const double e_lnlam = sum_dg_nu + D * kLn2 + ln_s;
      const double ldsig = -(V * g_lnA + Ld);
      const double t_lik = 0.5 * V * (e_lnrho - kLn2Pi) - 0.5 * er * R;
      const double t_beta = 0.5 * V * e_lnlam - 0.5 * V * D * kLn2Pi - 0.5 * (nu * tr1 + V * D / qv);
      const double t_k = 0.5 * D * ln_q0 - 0.5 * D * kLn2Pi + 0.5 * e_lnlam - 0.5 * q0 * (nu * quad + D / qv);
      double t_lam = 0.5 * (n0 - D - 1) * e_lnlam - 0.5 * nu * tr0;
      if (has_zprior) t_lam -= zprior;
      const double t_rho = a0 * ln_b0 - lg_a0 + (a0 - 1.0) * e_lnrho - b0 * er;
      const double h_beta = 0.5 * ldsig + 0.5 * V * D * (1.0 + kLn2Pi);
      const double h_rho = a - lnb + lga + (1.0 - a) * dga;
      const double e_lnq_k = 0.5 * D * ln_qv - 0.5 * D * kLn2Pi + 0.5 * e_lnlam - 0.5 * D;
      const double z_q = 0.5 * nu * D * kLn2 + 0.5 * nu * ln_s + mgl_nu;
      const double e_lnq_lam = 0.5 * (nu - D - 1) * e_lnlam - 0.5 * nu * D - z_q;
      elbo = t_lik + t_beta + t_k + t_lam + t_rho + h_beta + h_rho - e_lnq_k - e_lnq_lam;
    }
  }
  TAIL_PROF(*c, 3);
  if (mode == MODE_ELBO) {
    if (lane == 0) {
      s.elbo = status == CV_OK ? elbo : qnan();
      s.elbo_status = status == CV_OK ? elbo_status : status;
    }
    return;
  }
  // E[Lambda K] (vb.py:196-197) by rows; the deltas (vb.py:307-309) as warp reductions
  double elamk_i = 0.0;
  if (lane < D)
    for (int j = 0; j < D; ++j) elamk_i += nu * sm.S[lane * D + j] * sm.k_new[j];
  const bool sweep_ok = mode == MODE_SWEEP && status == CV_OK;
  double dk = 0.0, dl = 0.0;
  if (sweep_ok) {
    if constexpr (D <= kTailSerialD) {  // lane 0 alone: rel_delta_t over smem
      if (lane == 0) {
        double kn[D], ko[D], Ln[D * D], Lo[D * D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
          kn[i] = sm.k_new[i];
          ko[i] = sm.k_old[i];
        }
#pragma unroll
        for (int e = 0; e < D * D; ++e) {
          Ln[e] = sm.L[e];
          Lo[e] = sm.l_old[e];
        }
        dk = rel_delta_t<D>(kn, ko);
        dl = rel_delta_t<D * D>(Ln, Lo);
      }
    } else {
      double mo = 0.0, md = 0.0;
      if (lane < D) {
        mo = fabs(sm.k_old[lane]);
        md = fabs(sm.k_new[lane] - sm.k_old[lane]);
      }
      mo = warp_fmax(mo);
      md = warp_max_nan(md);
      dk = md / fmax(mo, 1e-300);
      mo = 0.0;
      md = 0.0;
      #pragma unroll
      for (int m_ = 0; m_ < (D2 + 31) / 32; ++m_) {
        const int e = lane + 32 * m_;
        if (e >= D2) break;
        mo = fmax(mo, fabs(sm.l_old[e]));
        const double df = fabs(sm.L[e] - sm.l_old[e]);
        md = (df > md || df != df) ? df : md;
      }
      mo = warp_fmax(mo);
      md = warp_max_nan(md);
      dl = md / fmax(mo, 1e-300);
    }
  }
  TAIL_PROF(*c, 4);

  // ---- phase 4: stores (every read of c / s happened above)
  #pragma unroll
  for (int m_ = 0; m_ < (D2 + 31) / 32; ++m_) {
    const int e = lane + 32 * m_;
    if (e >= D2) break;
    s.lam0l_inv[e] = sm.L[e];
    s.e_lam[e] = nu * sm.S[e];
    s.gen_A[e] = sm.gA[e];
    s.gen_Ainv[e] = sm.gAi[e];
  }
  if (lane < D) {
    s.k0k[lane] = sm.k_new[lane];
    s.e_lamk[lane] = elamk_i;
    s.gen_c[lane] = sm.gc[lane];
  }
  if (status == CV_OK) {  // generator of the next pass (vb.py:136-144)
    const double rnu = 1.0 / nu;
    if (lane < D) c->pass.c[lane] = sm.k_new[lane];
    #pragma unroll
    for (int m_ = 0; m_ < (D2 + 31) / 32; ++m_) {
      const int e = lane + 32 * m_;
      if (e >= D2) break;
      c->pass.A[e] = nu * sm.S[e];
      c->pass.Ainv[e] = sm.L[e] * rnu;
    }
  }
  if (lane == 0) {
    const double ld = sm.ld;
    const double R = sm.tot[stat_R(D)];
    int done = 0, c_status = CV_OK, new_iter = iter, new_have_prev = have_prev;
    double new_prev = prev_elbo, dr = 0.0;
    if (sweep_ok) {
      dr = rel_delta_t<1>(&e_rho, &e_rho_old);
      new_iter = iter + 1;
      if (compute_elbo) {
        if (elbo_status != CV_OK) {
          c_status = elbo_status;
          done = 1;
        } else {
          if (have_prev && fabs(elbo - prev_elbo) < rel_tol * fabs(elbo)) done = 1;
          new_prev = elbo;
          new_have_prev = 1;
        }
      } else if (fmax(dk, fmax(dr, dl)) < param_tol) {
        done = 1;
      }
      if (new_iter >= max_iter) done = 1;
    }
    if (status != CV_OK) {
      c_status = status;
      done = 1;
    }
    s.status = status;
    s.d = D;
    s.V = (int64_t)V;
    s.n_iter = mode == MODE_SWEEP ? n_iter_old + 1 : 0;
    s.a_rho = a;
    s.b_rho = b;
    s.e_rho = e_rho;
    s.ln_det_lam0l_inv = ld;
    s.resid = R;
    s.elbo = elbo;
    s.elbo_status = elbo_status;
    s.gen_lnA = g_lnA;
    s.gen_e_rho = g_erho;
    if (sweep_ok && iter < tr_cap) {
      tr_dk[iter] = dk;
      tr_drho[iter] = dr;
      tr_dlam[iter] = dl;
      tr_elbo[iter] = compute_elbo ? elbo : qnan();
    }
    c->iter = new_iter;
    c->have_prev = new_have_prev;
    c->prev_elbo = new_prev;
    if (c_status != CV_OK) c->status = c_status;
    if (done) c->done = 1;
    c->mode = MODE_SWEEP;
    if (status == CV_OK) {
      c->pass.lnA = D * ln_nu - ld;
      const double nb = b0 + 0.5 * R;
      c->pend_a = a_fit;
      c->pend_b = nb;
      c->pass.e_rho = a_fit / nb;
    }
  }
  TAIL_PROF(*c, 5);
}

// Test hook (cv_test_rate_inverse): the tail's rate inversion on one given matrix, exactly as a
// sweep runs it (tail_inverse: lane 0 for d <= kTailSerialD, the warp above).
template <int D>
__global__ void __launch_bounds__(32, 1) rate_inverse_test_kernel(const double* A, double* Ainv, double* ld, int* ok) {
  __shared__ TailSm<D> sm;
  for (int e = threadIdx.x; e < D * D; e += 32) sm.C[e] = A[e];
  __syncwarp();
  double l = 0.0;
  const bool good = tail_inverse<D>(sm, &l, threadIdx.x);
  for (int e = threadIdx.x; e < D * D; e += 32) Ainv[e] = sm.S[e];
  if (threadIdx.x == 0) {
    *ld = l;
    *ok = good ? 1 : 0;
  }
}

}  // namespace cavi
