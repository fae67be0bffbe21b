// engine.cuh -- device-side data structures, the O(d^3) "tail" of a CAVI sweep
// and the special functions it needs.  sm_100a, fp64.
//
// A sweep = one fused streaming pass over the measurements (pass.cuh) that
// yields the per-sweep statistic vector
//     [ g (d) | G upper triangle (d(d+1)/2) | R | Ld ]
// followed by this tail, run by the last CTA of the pass (single GPU) or by a
// one-CTA kernel after the NCCL exchange (multi-GPU).  The tail restates
// reference vb.py:136-197 (the rho and (K, Lambda) blocks) and vb.py:216-304
// (the bound) in the centred rank-1 form of SURVEY Appendix A, and the fit
// loop's bookkeeping and stop rule (vb.py:307-347).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/cavi.h"

namespace cavi {

constexpr int kMaxD = CV_MAX_DIM;
constexpr int kMaxD2 = CV_MAX_D2;
constexpr int kMaxStats = kMaxD + kMaxD * (kMaxD + 1) / 2 + 2;  // 137
constexpr int kChunk = 4096;         // genes per chunk (one CTA work unit)
constexpr int kGroupChunks = 64;     // chunks per group
constexpr int kOctants = 8;          // top of the reduction tree (GPU-count invariant)
constexpr int kThreads = 256;        // threads per CTA of the pass
constexpr int kWarps = kThreads / 32;

constexpr double kLn2 = 0.69314718055994530942;
constexpr double kLnPi = 1.14472988584940017414;
constexpr double kLn2Pi = 1.83787706640934548356;

__host__ __device__ constexpr int n_stats(int d) { return d + d * (d + 1) / 2 + 2; }

// Hyperparameters + sweep-invariant constants of the bound (reference model.py:126-151).
struct Hyp {
  int d, n0;
  double a0, b0, q0;
  double V, nu, qv;  // V = genes of the WHOLE dataset (all shards)
  double K0[kMaxD];
  double L0[kMaxD2];
  double L0inv[kMaxD2];
  double lnL0;
  int has_zprior;
  double zprior;     // Wishart prior log-normaliser (vb.py:201-207, 278-280)
  int proper_q;      // nu > d - 1 (vb.py:299-301)
  double a_fit;      // a0 + V/2 (vb.py:142)
  double dg_afit, lg_afit, dg_a0, lg_a0;
  double sum_dg_nu;  // sum_j digamma((nu + 1 - j)/2)   (vb.py:213)
  double mgl_nu;     // multigammaln(nu/2, d)
  int setup_status;
  double wL[kMaxD2], wJ[kMaxD2], wM[kMaxD2];  // setup workspace
};

// Expectations a pass streams against ("generator" of a state's per-gene moments).
struct Gen {
  double c[kMaxD];
  double A[kMaxD2];
  double Ainv[kMaxD2];
  double lnA;
  double e_rho;
};

enum { MODE_INIT = 0, MODE_SWEEP = 1, MODE_ELBO = 2 };

// Global-memory workspace of the (single-thread) tail: keeps the kernels' stack frames tiny.
struct Scratch {
  cv_state nw;
  double G[kMaxD2], AG[kMaxD2], S[kMaxD2], L[kMaxD2], J[kMaxD2], M[kMaxD2];
  double hv[kMaxD], dlt[kMaxD], k0c[kMaxD];
};

// Control block: current state, the generator of the next pass, fit loop control.
struct Ctl {
  Scratch scr;
  cv_state cur;
  Gen pass;
  double pend_a, pend_b;  // a_rho, b_rho of the state the next pass produces
  int mode;
  int done;
  int status;
  int iter, max_iter;
  int compute_elbo;
  int have_prev;
  double rel_tol, param_tol, prev_elbo;
  double* tr_elbo;
  double* tr_dk;
  double* tr_drho;
  double* tr_dlam;
  int tr_cap;
};

// ------------------------------------------------------------------ special functions
static __device__ inline double digamma_pos(double x) {
  // x > 0: recurrence up to x >= 10, then the asymptotic series (error < 1e-16).
  if (!(x > 0.0)) return __longlong_as_double(0x7ff8000000000000ULL);
  double acc = 0.0;
  while (x < 10.0) {
    acc -= 1.0 / x;
    x += 1.0;
  }
  const double f = 1.0 / (x * x);
  double t = -1.0 / 12.0 +
             f * (1.0 / 120.0 +
                  f * (-1.0 / 252.0 + f * (1.0 / 240.0 + f * (-1.0 / 132.0 + f * (691.0 / 32760.0 + f * (-1.0 / 12.0))))));
  return acc + log(x) - 0.5 / x + f * t;
}

static __device__ inline double multigammaln(double a, int d) {
  double s = 0.25 * d * (d - 1) * kLnPi;
  for (int j = 1; j <= d; ++j) s += lgamma(a + 0.5 * (1 - j));
  return s;
}

// ------------------------------------------------------------------ small dense SPD algebra
// Row-major d x d, d <= 15.  Cholesky with the reference's jitter-once policy
// (linalg.py:279-298): on failure add 1e-10 * trace/d to the diagonal and retry.
static __device__ __noinline__ bool chol(const double* A, double* L, int d) {
  for (int i = 0; i < d * d; ++i) L[i] = 0.0;
  for (int j = 0; j < d; ++j) {
    double s = A[j * d + j];
    for (int k = 0; k < j; ++k) s -= L[j * d + k] * L[j * d + k];
    if (!(s > 0.0)) return false;
    const double ljj = sqrt(s);
    L[j * d + j] = ljj;
    for (int i = j + 1; i < d; ++i) {
      double t = A[i * d + j];
      for (int k = 0; k < j; ++k) t -= L[i * d + k] * L[j * d + k];
      L[i * d + j] = t / ljj;
    }
  }
  return true;
}

// inverse + log-determinant of an SPD matrix; returns false if not PD after the retry.
// L, J, M: caller-provided d x d workspaces.
static __device__ __noinline__ bool spd_inv_logdet(const double* A, double* Ainv, double* logdet, int d, double* L,
                                            double* J, double* M) {
  if (!chol(A, L, d)) {
    double tr = 0.0;
    for (int j = 0; j < d; ++j) tr += A[j * d + j];
    const double jit = 1e-10 * tr / d;
    for (int i = 0; i < d * d; ++i) J[i] = A[i];
    for (int j = 0; j < d; ++j) J[j * d + j] += jit;
    if (!chol(J, L, d)) return false;
  }
  double ld = 0.0;
  for (int j = 0; j < d; ++j) ld += log(L[j * d + j]);
  *logdet = 2.0 * ld;
  // M = L^-1 (lower), then A^-1 = M^T M
  for (int i = 0; i < d * d; ++i) M[i] = 0.0;
  for (int j = 0; j < d; ++j) {
    M[j * d + j] = 1.0 / L[j * d + j];
    for (int i = j + 1; i < d; ++i) {
      double t = 0.0;
      for (int k = j; k < i; ++k) t -= L[i * d + k] * M[k * d + j];
      M[i * d + j] = t / L[i * d + i];
    }
  }
  for (int i = 0; i < d; ++i)
    for (int j = i; j < d; ++j) {
      double t = 0.0;
      for (int k = j; k < d; ++k) t += M[k * d + i] * M[k * d + j];
      Ainv[i * d + j] = t;
      Ainv[j * d + i] = t;
    }
  return true;
}

static __device__ inline double rel_delta(const double* nw, const double* old, int n) {
  // reference vb.py:307-309
  double mo = 0.0, md = 0.0;
  for (int i = 0; i < n; ++i) {
    mo = fmax(mo, fabs(old[i]));
    const double df = fabs(nw[i] - old[i]);
    md = (df > md || df != df) ? df : md;
  }
  return md / fmax(mo, 1e-300);
}

// ------------------------------------------------------------------ setup of the constants
static __device__ __noinline__ void hyp_setup(Hyp& h) {
  const int d = h.d;
  h.setup_status = CV_OK;
  if (!spd_inv_logdet(h.L0, h.L0inv, &h.lnL0, d, h.wL, h.wJ, h.wM)) {
    h.setup_status = CV_ERR_NUMERIC;
    return;
  }
  h.nu = h.n0 + h.V;
  h.qv = h.q0 + h.V;
  h.a_fit = h.a0 + 0.5 * h.V;
  h.dg_afit = digamma_pos(h.a_fit);
  h.lg_afit = lgamma(h.a_fit);
  h.dg_a0 = digamma_pos(h.a0);
  h.lg_a0 = lgamma(h.a0);
  h.proper_q = h.nu > d - 1;
  h.sum_dg_nu = 0.0;
  h.mgl_nu = 0.0;
  if (h.proper_q) {
    for (int j = 1; j <= d; ++j) h.sum_dg_nu += digamma_pos(0.5 * (h.nu + 1 - j));
    h.mgl_nu = multigammaln(0.5 * h.nu, d);
  }
  h.has_zprior = h.n0 > d - 1;
  h.zprior = 0.0;
  if (h.has_zprior) h.zprior = 0.5 * h.n0 * d * kLn2 + 0.5 * h.n0 * h.lnL0 + multigammaln(0.5 * h.n0, d);
}

// ------------------------------------------------------------------ the bound
// vb_elbo (reference vb.py:216-304) of state `st`, whose per-gene moments come
// from generator `gen`, from the pass statistics of that generator.
static __device__ __noinline__ double elbo_of(const Hyp& h, const cv_state& st, const Gen& gen, const double* stats,
                                       int* status, Scratch& w) {
  const int d = h.d;
  if (!h.proper_q) {
    *status = CV_ERR_IMPROPER;
    return __longlong_as_double(0x7ff8000000000000ULL);
  }
  const double V = h.V, nu = h.nu, qv = h.qv;
  const double* g = stats;
  const double R = stats[n_stats(d) - 2];
  const double Ld = stats[n_stats(d) - 1];
  double* G = w.G;
  {
    int p = d;
    for (int j = 0; j < d; ++j)
      for (int k = j; k < d; ++k) {
        G[j * d + k] = stats[p];
        G[k * d + j] = stats[p];
        ++p;
      }
  }
  double* S = w.S;
  double lnL;
  if (!spd_inv_logdet(st.lam0l_inv, S, &lnL, d, w.L, w.J, w.M)) {
    *status = CV_ERR_NUMERIC;
    return __longlong_as_double(0x7ff8000000000000ULL);
  }
  const double ln_s = -st.ln_det_lam0l_inv;
  const double a = st.a_rho, b = st.b_rho;
  const double dga = (a == h.a_fit) ? h.dg_afit : (a == h.a0 ? h.dg_a0 : digamma_pos(a));
  const double lga = (a == h.a_fit) ? h.lg_afit : (a == h.a0 ? h.lg_a0 : lgamma(a));
  const double e_rho = a / b;
  const double lnb = log(b);
  const double e_lnrho = dga - lnb;
  const double e_lnlam = h.sum_dg_nu + d * kLn2 + ln_s;
  // h_ = Ainv g, dlt = k0k - c
  double* hv = w.hv;
  double* dlt = w.dlt;
  for (int i = 0; i < d; ++i) {
    double t = 0.0;
    for (int j = 0; j < d; ++j) t += gen.Ainv[i * d + j] * g[j];
    hv[i] = t;
    dlt[i] = st.k0k[i] - gen.c[i];
  }
  // T = Ainv G Ainv ; scatter = V Ainv + T - dlt h^T - h dlt^T + V dlt dlt^T ; tr(S scatter)
  double* AG = w.AG;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      double t = 0.0;
      for (int k = 0; k < d; ++k) t += gen.Ainv[i * d + k] * G[k * d + j];
      AG[i * d + j] = t;
    }
  double tr1 = 0.0;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      double T = 0.0;
      for (int k = 0; k < d; ++k) T += AG[i * d + k] * gen.Ainv[k * d + j];
      const double sc = V * gen.Ainv[i * d + j] + T - dlt[i] * hv[j] - hv[i] * dlt[j] + V * dlt[i] * dlt[j];
      tr1 += S[i * d + j] * sc;
    }
  double quad = 0.0, tr0 = 0.0;
  for (int i = 0; i < d; ++i) {
    const double dki = st.k0k[i] - h.K0[i];
    for (int j = 0; j < d; ++j) {
      quad += dki * S[i * d + j] * (st.k0k[j] - h.K0[j]);
      tr0 += h.L0inv[i * d + j] * S[j * d + i];
    }
  }
  const double ldsig = -(V * gen.lnA + Ld);
  const double t_lik = 0.5 * V * (e_lnrho - kLn2Pi) - 0.5 * e_rho * R;
  const double t_beta = 0.5 * V * e_lnlam - 0.5 * V * d * kLn2Pi - 0.5 * (nu * tr1 + V * d / qv);
  const double t_k = 0.5 * d * log(h.q0) - 0.5 * d * kLn2Pi + 0.5 * e_lnlam - 0.5 * h.q0 * (nu * quad + d / qv);
  double t_lam = 0.5 * (h.n0 - d - 1) * e_lnlam - 0.5 * nu * tr0;
  if (h.has_zprior) t_lam -= h.zprior;
  const double t_rho = h.a0 * log(h.b0) - h.lg_a0 + (h.a0 - 1.0) * e_lnrho - h.b0 * e_rho;
  const double h_beta = 0.5 * ldsig + 0.5 * V * d * (1.0 + kLn2Pi);
  const double h_rho = a - lnb + lga + (1.0 - a) * dga;
  const double e_lnq_k = 0.5 * d * log(qv) - 0.5 * d * kLn2Pi + 0.5 * e_lnlam - 0.5 * d;
  const double z_q = 0.5 * nu * d * kLn2 + 0.5 * nu * ln_s + h.mgl_nu;
  const double e_lnq_lam = 0.5 * (nu - d - 1) * e_lnlam - 0.5 * nu * d - z_q;
  *status = CV_OK;
  return t_lik + t_beta + t_k + t_lam + t_rho + h_beta + h_rho - e_lnq_k - e_lnq_lam;
}

// generator of the next pass from the current state (vb.py:136-144)
static __device__ inline void derive_pass(const Hyp& h, Ctl& c) {
  const int d = h.d;
  const cv_state& s = c.cur;
  for (int i = 0; i < d; ++i) c.pass.c[i] = s.k0k[i];
  for (int i = 0; i < d * d; ++i) {
    c.pass.A[i] = s.e_lam[i];
    c.pass.Ainv[i] = s.lam0l_inv[i] / h.nu;
  }
  c.pass.lnA = d * log(h.nu) - s.ln_det_lam0l_inv;
  c.pend_a = h.a_fit;
  c.pend_b = h.b0 + 0.5 * s.resid;
  c.pass.e_rho = c.pend_a / c.pend_b;
}

static __device__ inline void copy_gen_to_state(const Gen& g, cv_state& s, int d) {
  for (int i = 0; i < d; ++i) s.gen_c[i] = g.c[i];
  for (int i = 0; i < d * d; ++i) {
    s.gen_A[i] = g.A[i];
    s.gen_Ainv[i] = g.Ainv[i];
  }
  s.gen_lnA = g.lnA;
  s.gen_e_rho = g.e_rho;
}

// The tail: new state from the pass statistics; trace, stop rule, next generator.
static __device__ __noinline__ void tail(const Hyp& h, Ctl& c, const double* stats) {
  const int d = h.d;
  const int ns = n_stats(d);
  if (c.mode == MODE_ELBO) {  // vb_elbo of the current state from a pass with its own generator
    int es;
    c.cur.elbo = elbo_of(h, c.cur, c.pass, stats, &es, c.scr);
    c.cur.elbo_status = es;
    return;
  }
  bool finite = true;
  for (int i = 0; i < ns; ++i) finite = finite && isfinite(stats[i]);
  cv_state& nw = c.scr.nw;
  nw = c.cur;
  const Gen& gen = c.pass;
  nw.status = CV_OK;
  nw.d = d;
  nw.V = (int64_t)h.V;
  if (c.mode == MODE_INIT) {
    // vb_init (vb.py:82-111): globals at the prior; this pass measured the init moments.
    nw.n_iter = 0;
    nw.a_rho = h.a0;
    nw.b_rho = h.b0;
    nw.e_rho = h.a0 / h.b0;
    for (int i = 0; i < d; ++i) nw.k0k[i] = h.K0[i];
    for (int i = 0; i < d * d; ++i) {
      nw.lam0l_inv[i] = h.L0[i];
      nw.e_lam[i] = h.nu * h.L0inv[i];
    }
    nw.ln_det_lam0l_inv = h.lnL0;
  } else {
    // (K, Lambda) block, centred (vb.py:172-183):
    //   dlt = (Ainv g + q0 (K0 - c)) / qv ; k0k = c + dlt
    //   lam0l_inv = L0inv + V Ainv + Ainv G Ainv + q0 (K0-c)(K0-c)^T - qv dlt dlt^T
    const double* g = stats;
    double* G = c.scr.G;
    int p = d;
    for (int j = 0; j < d; ++j)
      for (int k = j; k < d; ++k) {
        G[j * d + k] = stats[p];
        G[k * d + j] = stats[p];
        ++p;
      }
    double* k0c = c.scr.k0c;
    double* dlt = c.scr.dlt;
    for (int i = 0; i < d; ++i) {
      double t = 0.0;
      for (int j = 0; j < d; ++j) t += gen.Ainv[i * d + j] * g[j];
      k0c[i] = h.K0[i] - gen.c[i];
      dlt[i] = (t + h.q0 * k0c[i]) / h.qv;
      nw.k0k[i] = gen.c[i] + dlt[i];
    }
    double* AG = c.scr.AG;
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) {
        double t = 0.0;
        for (int k = 0; k < d; ++k) t += gen.Ainv[i * d + k] * G[k * d + j];
        AG[i * d + j] = t;
      }
    for (int i = 0; i < d; ++i)
      for (int j = i; j < d; ++j) {
        double T = 0.0;
        for (int k = 0; k < d; ++k) T += AG[i * d + k] * gen.Ainv[k * d + j];
        const double v = h.L0inv[i * d + j] + h.V * gen.Ainv[i * d + j] + T + h.q0 * k0c[i] * k0c[j] -
                         h.qv * dlt[i] * dlt[j];
        nw.lam0l_inv[i * d + j] = v;
        nw.lam0l_inv[j * d + i] = v;
      }
    double* S = c.scr.S;
    double ld;
    if (!finite) {
      nw.status = CV_ERR_NUMERIC;
    } else if (!spd_inv_logdet(nw.lam0l_inv, S, &ld, d, c.scr.L, c.scr.J, c.scr.M)) {
      nw.status = CV_ERR_NUMERIC;  // "Q(Lambda) rate inversion failed after jitter retry"
    } else {
      nw.ln_det_lam0l_inv = ld;
      for (int i = 0; i < d * d; ++i) nw.e_lam[i] = h.nu * S[i];
    }
    nw.a_rho = c.pend_a;
    nw.b_rho = c.pend_b;
    nw.e_rho = gen.e_rho;
    nw.n_iter = c.cur.n_iter + 1;
  }
  for (int i = 0; i < d; ++i) {
    double t = 0.0;
    for (int j = 0; j < d; ++j) t += nw.e_lam[i * d + j] * nw.k0k[j];
    nw.e_lamk[i] = t;
  }
  copy_gen_to_state(gen, nw, d);
  nw.resid = stats[ns - 2];
  nw.elbo = __longlong_as_double(0x7ff8000000000000ULL);
  nw.elbo_status = CV_OK;
  if (nw.status == CV_OK && (c.compute_elbo || c.mode == MODE_INIT)) {
    int es;
    nw.elbo = elbo_of(h, nw, gen, stats, &es, c.scr);
    nw.elbo_status = es;
  }
  if (c.mode == MODE_SWEEP && nw.status == CV_OK) {
    // fit bookkeeping (vb.py:332-347)
    const double dk = rel_delta(nw.k0k, c.cur.k0k, d);
    const double dr = rel_delta(&nw.e_rho, &c.cur.e_rho, 1);
    const double dl = rel_delta(nw.lam0l_inv, c.cur.lam0l_inv, d * d);
    const int it = c.iter;
    if (it < c.tr_cap) {
      c.tr_dk[it] = dk;
      c.tr_drho[it] = dr;
      c.tr_dlam[it] = dl;
      c.tr_elbo[it] = c.compute_elbo ? nw.elbo : __longlong_as_double(0x7ff8000000000000ULL);
    }
    c.iter = it + 1;
    if (c.compute_elbo) {
      if (nw.elbo_status != CV_OK) {
        c.status = nw.elbo_status;
        c.done = 1;
      } else {
        if (c.have_prev && fabs(nw.elbo - c.prev_elbo) < c.rel_tol * fabs(nw.elbo)) c.done = 1;
        c.prev_elbo = nw.elbo;
        c.have_prev = 1;
      }
    } else if (fmax(dk, fmax(dr, dl)) < c.param_tol) {
      c.done = 1;
    }
    if (c.iter >= c.max_iter) c.done = 1;
  }
  if (nw.status != CV_OK) {
    c.status = nw.status;
    c.done = 1;
  }
  c.cur = nw;
  c.mode = MODE_SWEEP;
  if (nw.status == CV_OK) derive_pass(h, c);
}

}  // namespace cavi
