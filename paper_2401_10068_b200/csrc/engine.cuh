// engine.cuh -- device-side data structures, the O(d^3) "tail" of a CAVI sweep
// and the special functions it needs.  sm_100a, fp64.
//
// A sweep = one fused streaming pass over the measurements (pass.cuh) that
// yields the per-sweep statistic vector
//     [ g (d) | G upper triangle (d(d+1)/2) | R | Ld ]
// followed by this tail, run by a separate one-warp kernel (pass.cuh tail_kernel) after
// the pass (and, on several GPUs, after the exchange).  The tail restates
// reference vb.py:136-197 (the rho and (K, Lambda) blocks) and vb.py:216-304
// (the bound) in the centred rank-1 form of SURVEY Appendix A, and the fit
// loop's bookkeeping and stop rule (vb.py:307-347).
//
// The tail is templated on d and works in registers and in place on the control
// block: it sits on the critical path of every sweep, so it must cost
// microseconds, not a walk through global-memory scratch.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/cavi.h"

namespace cavi {

constexpr int kMaxD = CV_MAX_DIM;
constexpr int kMaxD2 = CV_MAX_D2;
constexpr int kMaxStats = kMaxD + kMaxD * (kMaxD + 1) / 2 + 3;  // 138
// Reduction plan: chunk (one partial row) -> group (kGroupGenes genes) -> octant -> total.
// The chunk size is per dataset (plan_chunk_genes): 8192 genes halves the per-chunk finish
// work, which pays wherever there are enough chunks to balance (V >= 2^23) and the sweep is
// not purely bandwidth-trivial per gene (d >= 3): same-box A/B, V=1e8 (profiles/r02_c8k_ab.log):
// N=8 822 -> 890 sweeps/s, N=13 375 -> 388, N=4 sustained 448 -> 443 us; N=2, 3 lose ~1.5% and
// V <= 1e6 loses 15% (fewer chunks than CTAs), so those keep 4096.  Groups stay kGroupGenes
// genes either way: shard and octant boundaries do not depend on the chunk size.
constexpr int kChunk = 4096;                              // smallest chunk (genes)
constexpr int64_t kGroupGenes = 262144;                   // genes per group (64 x 4096 = 32 x 8192)
#ifndef CAVI_CHUNK_LARGE
#define CAVI_CHUNK_LARGE 8192
#endif
#ifndef CAVI_CHUNK_LARGE_MIN_V
#define CAVI_CHUNK_LARGE_MIN_V (1ll << 23)
#endif
#ifndef CAVI_CHUNK_LARGE_MIN_D
#define CAVI_CHUNK_LARGE_MIN_D 3
#endif
inline int plan_chunk_genes(int64_t V_total, int d) {
  return (d >= CAVI_CHUNK_LARGE_MIN_D && V_total >= CAVI_CHUNK_LARGE_MIN_V) ? CAVI_CHUNK_LARGE : kChunk;
}
constexpr int kOctants = 8;          // top of the reduction tree (GPU-count invariant)

constexpr double kLn2 = 0.69314718055994530942;
constexpr double kLnPi = 1.14472988584940017414;
constexpr double kLn2Pi = 1.83787706640934548356;

// statistic vector: [ g (d) | G upper (d(d+1)/2) | R | Q | Ld ]
//   R  = sum (x - t - s w)^2 + s/den   (residual moment sum, vb.py:114-126)
//   Q  = sum w (x - t) = sum e_rho (x - t)^2 / den   (marginal log-likelihood term, model.py:278-287)
//   Ld = sum ln den
__host__ __device__ constexpr int n_stats(int d) { return d + d * (d + 1) / 2 + 3; }
__host__ __device__ constexpr int stat_R(int d) { return n_stats(d) - 3; }
__host__ __device__ constexpr int stat_Q(int d) { return n_stats(d) - 2; }
__host__ __device__ constexpr int stat_Ld(int d) { return n_stats(d) - 1; }

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000ULL); }

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
  double ln_nu, ln_q0, ln_qv, ln_b0;
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

enum { MODE_INIT = 0, MODE_SWEEP = 1, MODE_ELBO = 2, MODE_EM = 3 };

// Control block: current state, the generator of the next pass, fit loop control.
struct Ctl {
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
  double* tr_k;  // EM: K per iteration [tr_cap][d]
  int tr_cap;
  unsigned long long prof[8];  // CAVI_TAIL_PROF builds: clock64 stamps of the last tail
  unsigned long long* tl_trace;  // diagnostics (CAVI_TRACE_CTA): globaltimer at tail entry / exit, per sweep
  int tl_n;
};

#ifdef CAVI_TAIL_PROF
#define TAIL_PROF(c, i) ((c).prof[i] = clock64())
#else
#define TAIL_PROF(c, i) ((void)0)
#endif

// ------------------------------------------------------------------ special functions
static __device__ inline double digamma_pos(double x) {
  // x > 0: recurrence up to x >= 10, then the asymptotic series (error < 1e-16).
  if (!(x > 0.0)) return qnan();
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
// Row-major D x D.  Cholesky with the reference's jitter-once policy
// (linalg.py:279-298): on failure add 1e-10 * trace/d to the diagonal and retry.
template <int D>
__device__ __forceinline__ bool chol_t(const double* A, double* L) {
#pragma unroll
  for (int i = 0; i < D * D; ++i) L[i] = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    double s = A[j * D + j];
#pragma unroll
    for (int k = 0; k < j; ++k) s -= L[j * D + k] * L[j * D + k];
    if (!(s > 0.0)) return false;
    const double ljj = sqrt(s);
    const double rl = 1.0 / ljj;
    L[j * D + j] = ljj;
#pragma unroll
    for (int i = j + 1; i < D; ++i) {
      double t = A[i * D + j];
#pragma unroll
      for (int k = 0; k < j; ++k) t -= L[i * D + k] * L[j * D + k];
      L[i * D + j] = t * rl;
    }
  }
  return true;
}

// inverse + log-determinant of an SPD matrix by Cholesky; false if not PD after the retry
// (the posterior sampler's covariance, where a factor is needed anyway)
template <int D>
__device__ __forceinline__ bool spd_inv_logdet_chol_t(const double* A, double* Ainv, double* logdet) {
  double L[D * D];
  if (!chol_t<D>(A, L)) {
    double tr = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) tr += A[j * D + j];
    const double jit = 1e-10 * tr / D;
    double J[D * D];
#pragma unroll
    for (int i = 0; i < D * D; ++i) J[i] = A[i];
#pragma unroll
    for (int j = 0; j < D; ++j) J[j * D + j] += jit;
    if (!chol_t<D>(J, L)) return false;
  }
  double prod = 1.0;
  double M[D * D];  // L^-1, lower
#pragma unroll
  for (int i = 0; i < D * D; ++i) M[i] = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    prod *= L[j * D + j];
    M[j * D + j] = 1.0 / L[j * D + j];
#pragma unroll
    for (int i = j + 1; i < D; ++i) {
      double t = 0.0;
#pragma unroll
      for (int k = j; k < i; ++k) t -= L[i * D + k] * M[k * D + j];
      M[i * D + j] = t / L[i * D + i];
    }
  }
  *logdet = 2.0 * log(prod);
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = i; j < D; ++j) {
      double t = 0.0;
#pragma unroll
      for (int k = j; k < D; ++k) t += M[k * D + i] * M[k * D + j];
      Ainv[i * D + j] = t;
      Ainv[j * D + i] = t;
    }
  return isfinite(*logdet);
}

// The reference's batched inverse (linalg.py:111-192) on one matrix, for the rate / precision
// inversions the sweep and the bound perform (vb.py:137, 183, 216-304; em.py:84-93):
//   d <= 3  closed-form adjugate times 1/det, cofactor by cofactor as _inv2 / _inv3, "singular"
//           when |det| < 1e-300 (DET_GUARD);
//   d >= 4  elimination with partial pivoting (LAPACK getrf/getri's algorithm class), "singular"
//           only on an exactly zero pivot (LinAlgError).
// No positive-definiteness test: like the reference, an indefinite but non-singular matrix is
// inverted.  *logdet = ln|det| (the reference's slogdet, sign dropped).
template <int D>
__device__ __forceinline__ bool ref_inv_once_t(const double* A, double* Ainv, double* logabs) {
  if constexpr (D == 1) {
    if (!(fabs(A[0]) >= 1e-300)) return false;
    Ainv[0] = 1.0 / A[0];
    *logabs = log(fabs(A[0]));
    return true;
  } else if constexpr (D == 2) {
    const double a = A[0], b = A[1], c = A[2], d = A[3];
    const double det = a * d - b * c;
    if (!(fabs(det) >= 1e-300)) return false;
    const double r = 1.0 / det;
    Ainv[0] = d * r;
    Ainv[1] = -b * r;
    Ainv[2] = -c * r;
    Ainv[3] = a * r;
    *logabs = log(fabs(det));
    return true;
  } else if constexpr (D == 3) {
    auto m = [&](int i, int j) { return A[i * 3 + j]; };
    const double c00 = m(1, 1) * m(2, 2) - m(1, 2) * m(2, 1);
    const double c01 = m(1, 2) * m(2, 0) - m(1, 0) * m(2, 2);
    const double c02 = m(1, 0) * m(2, 1) - m(1, 1) * m(2, 0);
    const double det = m(0, 0) * c00 + m(0, 1) * c01 + m(0, 2) * c02;
    if (!(fabs(det) >= 1e-300)) return false;
    const double c10 = m(0, 2) * m(2, 1) - m(0, 1) * m(2, 2);
    const double c11 = m(0, 0) * m(2, 2) - m(0, 2) * m(2, 0);
    const double c12 = m(0, 1) * m(2, 0) - m(0, 0) * m(2, 1);
    const double c20 = m(0, 1) * m(1, 2) - m(0, 2) * m(1, 1);
    const double c21 = m(0, 2) * m(1, 0) - m(0, 0) * m(1, 2);
    const double c22 = m(0, 0) * m(1, 1) - m(0, 1) * m(1, 0);
    const double r = 1.0 / det;
    Ainv[0] = c00 * r;
    Ainv[1] = c10 * r;
    Ainv[2] = c20 * r;
    Ainv[3] = c01 * r;
    Ainv[4] = c11 * r;
    Ainv[5] = c21 * r;
    Ainv[6] = c02 * r;
    Ainv[7] = c12 * r;
    Ainv[8] = c22 * r;
    *logabs = log(fabs(det));
    return true;
  } else {
    // Gauss-Jordan with partial pivoting on [A | I] (one thread; the batched kernel's d >= 4)
    double M[D * 2 * D];
    for (int i = 0; i < D; ++i)
      for (int j = 0; j < 2 * D; ++j) M[i * 2 * D + j] = j < D ? A[i * D + j] : (j - D == i ? 1.0 : 0.0);
    double prod = 1.0;
    int ex = 0;
    for (int k = 0; k < D; ++k) {
      int p = k;
      for (int i = k + 1; i < D; ++i)
        if (fabs(M[i * 2 * D + k]) > fabs(M[p * 2 * D + k])) p = i;
      const double piv = M[p * 2 * D + k];
      if (piv == 0.0) return false;
      if (p != k)
        for (int j = 0; j < 2 * D; ++j) {
          const double t = M[k * 2 * D + j];
          M[k * 2 * D + j] = M[p * 2 * D + j];
          M[p * 2 * D + j] = t;
        }
      const double rp = 1.0 / piv;
      for (int j = 0; j < 2 * D; ++j) M[k * 2 * D + j] *= rp;
      for (int i = 0; i < D; ++i) {
        if (i == k) continue;
        const double f = M[i * 2 * D + k];
        for (int j = 0; j < 2 * D; ++j) M[i * 2 * D + j] = fma(-f, M[k * 2 * D + j], M[i * 2 * D + j]);
      }
      prod *= fabs(piv);
      const int hi = __double2hiint(prod);
      ex += ((hi >> 20) & 0x7ff) - 1023;
      prod = __hiloint2double((hi & 0x800fffff) | 0x3ff00000, __double2loint(prod));
    }
    for (int i = 0; i < D; ++i)
      for (int j = 0; j < D; ++j) Ainv[i * D + j] = M[i * 2 * D + D + j];
    *logabs = log(prod) + (double)ex * kLn2;
    return true;
  }
}

// ref_inv_once_t with the jitter-once retry (linalg.py:279-298); *logdet = ln|det| of the
// matrix actually inverted.  False: singular after the retry (NumericError).
template <int D>
__device__ __forceinline__ bool spd_inv_logdet_t(const double* A, double* Ainv, double* logdet) {
  double ld = 0.0;
  if (!ref_inv_once_t<D>(A, Ainv, &ld)) {
    double tr = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) tr += A[j * D + j];
    const double jit = 1e-10 * tr / D;
    double J[D * D];
#pragma unroll
    for (int i = 0; i < D * D; ++i) J[i] = A[i];
#pragma unroll
    for (int j = 0; j < D; ++j) J[j * D + j] += jit;
    if (!ref_inv_once_t<D>(J, Ainv, &ld)) return false;
  }
  *logdet = ld;
  return isfinite(ld);
}

// runtime-d variant, used once per call by the setup kernel (workspaces in Hyp)
static __device__ __noinline__ bool spd_inv_logdet_rt(const double* A, double* Ainv, double* logdet, int d,
                                                      double* L, double* J, double* M) {
  auto chol = [&](const double* X) {
    for (int i = 0; i < d * d; ++i) L[i] = 0.0;
    for (int j = 0; j < d; ++j) {
      double s = X[j * d + j];
      for (int k = 0; k < j; ++k) s -= L[j * d + k] * L[j * d + k];
      if (!(s > 0.0)) return false;
      L[j * d + j] = sqrt(s);
      for (int i = j + 1; i < d; ++i) {
        double t = X[i * d + j];
        for (int k = 0; k < j; ++k) t -= L[i * d + k] * L[j * d + k];
        L[i * d + j] = t / L[j * d + j];
      }
    }
    return true;
  };
  if (!chol(A)) {
    double tr = 0.0;
    for (int j = 0; j < d; ++j) tr += A[j * d + j];
    for (int i = 0; i < d * d; ++i) J[i] = A[i];
    for (int j = 0; j < d; ++j) J[j * d + j] += 1e-10 * tr / d;
    if (!chol(J)) return false;
  }
  double ld = 0.0;
  for (int j = 0; j < d; ++j) ld += log(L[j * d + j]);
  *logdet = 2.0 * ld;
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

template <int N>
__device__ __forceinline__ double rel_delta_t(const double* nw, const double* old) {
  // reference vb.py:307-309
  double mo = 0.0, md = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    mo = fmax(mo, fabs(old[i]));
    const double df = fabs(nw[i] - old[i]);
    md = (df > md || df != df) ? df : md;
  }
  return md / fmax(mo, 1e-300);
}

// ref_inv_once_t's d >= 4 branch across one warp: Gauss-Jordan with partial pivoting on
// [A | I] (2 d^2 / 32 elements per lane per pivot; the pivot search a warp argmax with the lowest
// row on ties, as idamax).  "Singular" only on an exactly zero pivot, like LAPACK's getrf.
template <int D>
__device__ bool ref_inv_once_warp(const double* A, double* M, double* Ainv, double* logabs, int lane) {
  constexpr int W = 2 * D, N = D * W, K = (N + 31) / 32;
  for (int e = lane; e < N; e += 32) {
    const int i = e / W, j = e % W;
    M[e] = j < D ? A[i * D + j] : (j - D == i ? 1.0 : 0.0);
  }
  __syncwarp();
  int ei[K], ej[K];
#pragma unroll
  for (int m = 0; m < K; ++m) {
    const int e = lane + 32 * m < N ? lane + 32 * m : 0;
    ei[m] = e / W;
    ej[m] = e % W;
  }
  double prod = 1.0;  // lane 0: product of |pivots|, exponent renormalised
  int ex = 0;
#pragma unroll 1
  for (int k = 0; k < D; ++k) {
    double v = (lane >= k && lane < D) ? fabs(M[lane * W + k]) : -1.0;
    int p = lane;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, off);
      const int op = __shfl_xor_sync(0xffffffffu, p, off);
      if (ov > v || (ov == v && op < p)) {
        v = ov;
        p = op;
      }
    }
    const double piv = M[p * W + k];
    if (piv == 0.0) return false;  // every lane has the same p
    if (p != k) {
      for (int j = lane; j < W; j += 32) {
        const double t = M[k * W + j];
        M[k * W + j] = M[p * W + j];
        M[p * W + j] = t;
      }
      __syncwarp();
    }
    const double rp = 1.0 / piv;
    double nv[K];
#pragma unroll
    for (int m = 0; m < K; ++m) {
      const int i = ei[m], j = ej[m];
      const double mkj = M[k * W + j] * rp;
      nv[m] = i == k ? mkj : fma(-M[i * W + k], mkj, M[i * W + j]);
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < K; ++m)
      if (lane + 32 * m < N) M[lane + 32 * m] = nv[m];
    __syncwarp();
    if (lane == 0) {
      prod *= fabs(piv);
      const int hi = __double2hiint(prod);
      ex += ((hi >> 20) & 0x7ff) - 1023;
      prod = __hiloint2double((hi & 0x800fffff) | 0x3ff00000, __double2loint(prod));
    }
  }
  for (int e = lane; e < D * D; e += 32) Ainv[e] = M[(e / D) * W + D + e % D];
  if (lane == 0) *logabs = log(prod) + (double)ex * kLn2;
  __syncwarp();
  return true;
}

// Symmetric sweep (Gauss-Jordan without pivoting: after sweeping every pivot k, W = -A^-1) --
// the fast path for the positive-definite rates every real sweep produces.  W lives in
// registers: lane r + 16 h holds row r's column half h (H = ceil(d / 2) columns), so a pivot is
// 2 + H shuffles (pivot, column k, row k) and H branch-free updates per lane, with no shared-memory
// round trip or warp barrier between pivots (one warp alone runs the tail: every pivot is pure
// latency).  Returns false on a non-positive pivot (indefinite or singular), where the pivoted
// elimination decides as the reference would.
template <int D>
__device__ bool spd_sweep_warp(const double* A, double* /*W*/, double* Ainv, double* logabs, int lane) {
  static_assert(D <= 16, "two column halves of at most 16 rows");
  constexpr int H = (D + 1) / 2;
  const int r = lane & 15, h = lane >> 4;
  double w[H];
#pragma unroll
  for (int t = 0; t < H; ++t) {
    const int j = h * H + t;
    w[t] = (r < D && j < D) ? A[r * D + j] : 0.0;
  }
  double prod = 1.0;
  int ex = 0;
  // Rolled over the column half of the pivot, unrolled within it (the register index of the
  // pivot's column must be static: a dynamic index goes to local memory).  The tail runs once
  // per sweep with its code fetched cold; the half-rolled form measured fastest in the tail at
  // d = 15 (tools/tail_cycles.sh: unrolled 9.3k, half-rolled 7.7k, fully rolled with selects 8.4k cycles).
#pragma unroll 1
  for (int hk = 0; hk < 2; ++hk)
#pragma unroll
  for (int tk = 0; tk < H; ++tk) {
    const int k = hk * H + tk;
    if (k >= D) break;
    const double p = __shfl_sync(0xffffffffu, w[tk], k + 16 * hk);
    const double wik = __shfl_sync(0xffffffffu, w[tk], r + 16 * hk);
    double wkj[H];
#pragma unroll
    for (int t = 0; t < H; ++t) wkj[t] = __shfl_sync(0xffffffffu, w[t], k + 16 * h);
    if (!(p > 0.0)) return false;  // every lane has the same pivot
    const double rp = 1.0 / p;
#pragma unroll
    for (int t = 0; t < H; ++t) {
      const int j = h * H + t;
      const double gen = fma(-wik * rp, wkj[t], w[t]);
      const double rowcol = (r == k ? wkj[t] : wik) * rp;
      w[t] = (r == k && j == k) ? -rp : ((r == k || j == k) ? rowcol : gen);
    }
    if (lane == 0) {
      prod *= p;
      const int hi = __double2hiint(prod);
      ex += ((hi >> 20) & 0x7ff) - 1023;
      prod = __hiloint2double((hi & 0x800fffff) | 0x3ff00000, __double2loint(prod));
    }
  }
#pragma unroll
  for (int t = 0; t < H; ++t) {
    const int j = h * H + t;
    if (r < D && j < D) Ainv[r * D + j] = -w[t];
  }
  if (lane == 0) *logabs = log(prod) + (double)ex * kLn2;
  __syncwarp();
  return true;
}

// The reference's inverse across the warp: the sweep when every pivot is positive, else the
// pivoted elimination, with the jitter-once retry (linalg.py:279-298) on a jittered copy of A
template <int D>
__device__ bool ref_inv_logdet_warp(const double* A, double* J, double* M, double* Ainv, double* logdet, int lane) {
  if (spd_sweep_warp<D>(A, M, Ainv, logdet, lane)) return true;
  if (ref_inv_once_warp<D>(A, M, Ainv, logdet, lane)) return true;
  double tr = 0.0;
  for (int j = 0; j < D; ++j) tr += A[j * D + j];  // every lane: the same sum
  for (int e = lane; e < D * D; e += 32) J[e] = A[e] + ((e / D == e % D) ? 1e-10 * tr / D : 0.0);
  __syncwarp();
  return ref_inv_once_warp<D>(J, M, Ainv, logdet, lane);
}

// ------------------------------------------------------------------ setup of the constants
static __device__ __noinline__ void hyp_setup(Hyp& h) {
  const int d = h.d;
  h.setup_status = CV_OK;
  if (d <= 3) {  // vb_init inverts Lambda0 per gene by the adjugate (vb.py:94-97, linalg.py:111-153): its guard
    const double* A = h.L0;
    const double det = d == 1 ? A[0]
                       : d == 2 ? A[0] * A[3] - A[1] * A[2]
                                : A[0] * (A[4] * A[8] - A[5] * A[7]) + A[1] * (A[5] * A[6] - A[3] * A[8]) +
                                      A[2] * (A[3] * A[7] - A[4] * A[6]);
    if (!(fabs(det) >= 1e-300)) {
      h.setup_status = CV_ERR_SINGULAR;
      return;
    }
  }
  if (!spd_inv_logdet_rt(h.L0, h.L0inv, &h.lnL0, d, h.wL, h.wJ, h.wM)) {
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
  h.ln_nu = log(h.nu);
  h.ln_q0 = log(h.q0);
  h.ln_qv = log(h.qv);
  h.ln_b0 = log(h.b0);
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

// Register/stack copy of the hyperparameters a d-specialised tail needs, loaded in
// one burst of independent loads (the tail is latency-bound: one thread, end of sweep).
// A fixed-size read-only block: a register copy, or a pointer to the global original.
template <int N, bool Reg>
struct Mat {
  double v[N];
  __device__ __forceinline__ void load(const double* __restrict__ p) {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = p[i];
  }
  __device__ __forceinline__ double operator[](int i) const { return v[i]; }
  __device__ __forceinline__ operator const double*() const { return v; }
};
template <int N>
struct Mat<N, false> {
  const double* v;
  __device__ __forceinline__ void load(const double* p) { v = p; }
  __device__ __forceinline__ double operator[](int i) const { return v[i]; }
  __device__ __forceinline__ operator const double*() const { return v; }
};

template <int D>
struct HypT {
  // d x d blocks: registers for small d; for d > 8 (4 x 225 doubles would spill the whole
  // tail to local memory) they stay in the L1-cached global structs and are read in place
  static constexpr bool kReg = D <= 8;
  int n0, has_zprior, proper_q;
  double a0, b0, q0, V, nu, qv, lnL0, zprior, a_fit, dg_afit, lg_afit, dg_a0, lg_a0, sum_dg_nu, mgl_nu;
  double ln_nu, ln_q0, ln_qv, ln_b0;
  double K0[D];
  Mat<D * D, kReg> L0, L0inv;
  __device__ __forceinline__ void load(const Hyp& __restrict__ h) {
    n0 = h.n0;
    has_zprior = h.has_zprior;
    proper_q = h.proper_q;
    a0 = h.a0; b0 = h.b0; q0 = h.q0; V = h.V; nu = h.nu; qv = h.qv; lnL0 = h.lnL0; zprior = h.zprior;
    a_fit = h.a_fit; dg_afit = h.dg_afit; lg_afit = h.lg_afit; dg_a0 = h.dg_a0; lg_a0 = h.lg_a0;
    sum_dg_nu = h.sum_dg_nu; mgl_nu = h.mgl_nu; ln_nu = h.ln_nu; ln_q0 = h.ln_q0; ln_qv = h.ln_qv; ln_b0 = h.ln_b0;
#pragma unroll
    for (int i = 0; i < D; ++i) K0[i] = h.K0[i];
    L0.load(h.L0);
    L0inv.load(h.L0inv);
  }
};

// the generator a pass streamed against, in registers (d x d blocks in place for d > 8)
template <int D>
struct GenT {
  static constexpr bool kReg = D <= 8;
  double c[D];
  Mat<D * D, kReg> A, Ainv;
  double lnA, e_rho;
  __device__ __forceinline__ void load(const Gen& __restrict__ g) {
#pragma unroll
    for (int i = 0; i < D; ++i) c[i] = g.c[i];
    A.load(g.A);
    Ainv.load(g.Ainv);
    lnA = g.lnA;
    e_rho = g.e_rho;
  }
};

// ------------------------------------------------------------------ the bound
// vb_elbo (reference vb.py:216-304) of the state (a, b, k0k, S = lam0l_inv^-1,
// ln|lam0l_inv|), whose per-gene moments come from generator `gen`, from the
// pass statistics of that generator.
// Tm = Ainv G Ainv (full), hv = Ainv g from a pass's statistics [g | G upper | ...]
template <int D>
__device__ __forceinline__ void pass_products_t(const double* Ai, const double* stats, double* Tm, double* hv) {
  double G[D * D], AG[D * D];
  {
    int p = D;
#pragma unroll
    for (int j = 0; j < D; ++j)
#pragma unroll
      for (int k = j; k < D; ++k) {
        G[j * D + k] = stats[p];
        G[k * D + j] = stats[p];
        ++p;
      }
  }
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) t += Ai[i * D + j] * stats[j];
    hv[i] = t;
  }
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) t += Ai[i * D + k] * G[k * D + j];
      AG[i * D + j] = t;
    }
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) t += AG[i * D + k] * Ai[k * D + j];
      Tm[i * D + j] = t;
    }
}

template <int D>
__device__ __forceinline__ double elbo_t(const HypT<D>& h, double a, double b, const double* k0k, const double* S,
                                         double ln_det_l, const GenT<D>& gen, const double* stats, const double* Tm,
                                         const double* hv, int* status) {
  // Tm = Ainv G Ainv and hv = Ainv g of this pass (shared with the (K, Lambda) update)
  if (!h.proper_q) {
    *status = CV_ERR_IMPROPER;
    return qnan();
  }
  const double V = h.V, nu = h.nu, qv = h.qv;
  const double R = stats[stat_R(D)];
  const double Ld = stats[stat_Ld(D)];
  const double* Ai = gen.Ainv;
  const double ln_s = -ln_det_l;
  const double dga = (a == h.a_fit) ? h.dg_afit : (a == h.a0 ? h.dg_a0 : digamma_pos(a));
  const double lga = (a == h.a_fit) ? h.lg_afit : (a == h.a0 ? h.lg_a0 : lgamma(a));
  const double e_rho = a / b;
  const double lnb = log(b);
  const double e_lnrho = dga - lnb;
  const double e_lnlam = h.sum_dg_nu + D * kLn2 + ln_s;
  double dlt[D];  // k0k - c
#pragma unroll
  for (int i = 0; i < D; ++i) dlt[i] = k0k[i] - gen.c[i];
  // scatter = V Ainv + Ainv G Ainv - dlt h^T - h dlt^T + V dlt dlt^T ; tr(S scatter)
  double tr1 = 0.0, quad = 0.0, tr0 = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double sc = V * Ai[i * D + j] + ((const volatile double*)Tm)[i * D + j] - dlt[i] * hv[j] - hv[i] * dlt[j] +
                        V * dlt[i] * dlt[j];
      const double sij = S[i * D + j];
      tr1 += sij * sc;
      quad += (k0k[i] - h.K0[i]) * sij * (k0k[j] - h.K0[j]);
      tr0 += h.L0inv[j * D + i] * sij;
    }
  const double ldsig = -(V * gen.lnA + Ld);
  const double t_lik = 0.5 * V * (e_lnrho - kLn2Pi) - 0.5 * e_rho * R;
  const double t_beta = 0.5 * V * e_lnlam - 0.5 * V * D * kLn2Pi - 0.5 * (nu * tr1 + V * D / qv);
  const double t_k = 0.5 * D * h.ln_q0 - 0.5 * D * kLn2Pi + 0.5 * e_lnlam - 0.5 * h.q0 * (nu * quad + D / qv);
  double t_lam = 0.5 * (h.n0 - D - 1) * e_lnlam - 0.5 * nu * tr0;
  if (h.has_zprior) t_lam -= h.zprior;
  const double t_rho = h.a0 * h.ln_b0 - h.lg_a0 + (h.a0 - 1.0) * e_lnrho - h.b0 * e_rho;
  const double h_beta = 0.5 * ldsig + 0.5 * V * D * (1.0 + kLn2Pi);
  const double h_rho = a - lnb + lga + (1.0 - a) * dga;
  const double e_lnq_k = 0.5 * D * h.ln_qv - 0.5 * D * kLn2Pi + 0.5 * e_lnlam - 0.5 * D;
  const double z_q = 0.5 * nu * D * kLn2 + 0.5 * nu * ln_s + h.mgl_nu;
  const double e_lnq_lam = 0.5 * (nu - D - 1) * e_lnlam - 0.5 * nu * D - z_q;
  *status = CV_OK;
  return t_lik + t_beta + t_k + t_lam + t_rho + h_beta + h_rho - e_lnq_k - e_lnq_lam;
}

// runtime-d generator derivation (after a host-provided state)
static __device__ __noinline__ void derive_pass_rt(const Hyp& h, Ctl& c) {
  const int d = h.d;
  cv_state& s = c.cur;
  const double rnu = 1.0 / h.nu;  // same arithmetic as tail_t's hand-over
  for (int i = 0; i < d; ++i) c.pass.c[i] = s.k0k[i];
  for (int i = 0; i < d * d; ++i) {
    c.pass.A[i] = s.e_lam[i];
    c.pass.Ainv[i] = s.lam0l_inv[i] * rnu;
  }
  c.pass.lnA = d * h.ln_nu - s.ln_det_lam0l_inv;
  c.pend_a = h.a_fit;
  c.pend_b = h.b0 + 0.5 * s.resid;
  c.pass.e_rho = h.a_fit / c.pend_b;
}

// The tail: new state (in place in c.cur) from the pass statistics; trace, stop rule,
// next generator.  Structured as load-everything / compute in registers / store-everything:
// a single thread runs it at the end of every sweep, so its dependent global round trips
// (not its flops) are what the sweep pays for.
template <int D>
__device__ __forceinline__ void tail_t(const Hyp& hyp, Ctl& c, const double* stats, const double* Tm,
                                       const double* hv, const double* preL = nullptr, const double* preS = nullptr,
                                       double preld = 0.0, int pre_ok = 1) {
  // preL / preS / preld: the new lam0l_inv, its inverse and log-det from the warp (tail_kernel,
  // d > 8, sweep mode); otherwise computed here
  // Tm / hv: Ainv G Ainv and Ainv g of this pass (pass_products_t; the warp computes them in
  // tail_kernel, a batched thread for itself)
  constexpr int NS = n_stats(D);
  // ---- loads (independent, issued back to back)
  HypT<D> h;
  h.load(hyp);
  GenT<D> gen;
  gen.load(c.pass);
  cv_state& s = c.cur;
  const int mode = c.mode, compute_elbo = c.compute_elbo, have_prev = c.have_prev, iter = c.iter;
  const int max_iter = c.max_iter, tr_cap = c.tr_cap, n_iter_old = s.n_iter;
  const double prev_elbo = c.prev_elbo, rel_tol = c.rel_tol, param_tol = c.param_tol;
  const double pend_a = c.pend_a, pend_b = c.pend_b;
  double* tr_elbo = c.tr_elbo;
  double* tr_dk = c.tr_dk;
  double* tr_drho = c.tr_drho;
  double* tr_dlam = c.tr_dlam;
  double st[NS];
#pragma unroll
  for (int i = 0; i < NS; ++i) st[i] = stats[i];
  double k_old[D];
  Mat<D * D, (D <= 8)> l_old;  // read in place for d > 8 (the stores below come after its last use)
  const double e_rho_old = s.e_rho, a_old = s.a_rho, b_old = s.b_rho, ld_old = s.ln_det_lam0l_inv;
#pragma unroll
  for (int i = 0; i < D; ++i) k_old[i] = s.k0k[i];
  l_old.load(s.lam0l_inv);

  TAIL_PROF(c, 1);
  if (mode == MODE_ELBO) {  // vb_elbo of the current state from a pass with its own generator
    double S[D * D], ld;
    int es = CV_ERR_NUMERIC;
    double e = qnan();
    if (spd_inv_logdet_t<D>(l_old, S, &ld)) e = elbo_t<D>(h, a_old, b_old, k_old, S, ld_old, gen, st, Tm, hv, &es);
    s.elbo = e;
    s.elbo_status = es;
    return;
  }
  bool finite = true;
#pragma unroll
  for (int i = 0; i < NS; ++i) finite = finite && isfinite(st[i]);

  // ---- compute
  double k_new[D], L[D * D], S[D * D], ld = 0.0;
  int status = CV_OK;
  double a, b, e_rho;
  if (mode == MODE_INIT) {
    // vb_init (vb.py:82-111): globals at the prior; this pass measured the init moments.
    a = h.a0;
    b = h.b0;
    e_rho = h.a0 / h.b0;
#pragma unroll
    for (int i = 0; i < D; ++i) k_new[i] = h.K0[i];
#pragma unroll
    for (int i = 0; i < D * D; ++i) {
      L[i] = h.L0[i];
      S[i] = h.L0inv[i];
    }
    ld = h.lnL0;
  } else {
    // (K, Lambda) block, centred (vb.py:172-183):
    //   dlt = (Ainv g + q0 (K0 - c)) / qv ; k0k = c + dlt
    //   lam0l_inv = L0inv + V Ainv + Ainv G Ainv + q0 (K0-c)(K0-c)^T - qv dlt dlt^T
    const double* Ai = gen.Ainv;
    double k0c[D], dlt[D];
    const double rqv = 1.0 / h.qv;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      k0c[i] = h.K0[i] - gen.c[i];
      dlt[i] = (hv[i] + h.q0 * k0c[i]) * rqv;
      k_new[i] = gen.c[i] + dlt[i];
    }
    if (preL) {
#pragma unroll
      for (int i = 0; i < D * D; ++i) {
        L[i] = preL[i];
        S[i] = preS[i];
      }
      ld = preld;
      if (!finite || !pre_ok) status = CV_ERR_NUMERIC;  // rate inversion failed
    } else {
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = i; j < D; ++j) {
          const double v = h.L0inv[i * D + j] + h.V * Ai[i * D + j] + ((const volatile double*)Tm)[i * D + j] +
                           h.q0 * k0c[i] * k0c[j] - h.qv * dlt[i] * dlt[j];
          L[i * D + j] = v;
          L[j * D + i] = v;
        }
      if (!finite || !spd_inv_logdet_t<D>(L, S, &ld)) status = CV_ERR_NUMERIC;  // rate inversion failed
    }
    a = pend_a;
    b = pend_b;
    e_rho = gen.e_rho;
  }
  TAIL_PROF(c, 2);
  double elbo = qnan();
  int elbo_status = CV_OK;
  if (status == CV_OK && (compute_elbo || mode == MODE_INIT))
    elbo = elbo_t<D>(h, a, b, k_new, S, ld, gen, st, Tm, hv, &elbo_status);
  TAIL_PROF(c, 3);
  double elamk[D];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) t += h.nu * S[i * D + j] * k_new[j];
    elamk[i] = t;
  }
  // fit bookkeeping (vb.py:332-347)
  int done = 0, c_status = CV_OK, new_iter = iter, new_have_prev = have_prev;
  double new_prev = prev_elbo, dk = 0.0, dr = 0.0, dl = 0.0;
  const bool sweep_ok = mode == MODE_SWEEP && status == CV_OK;
  if (sweep_ok) {
    dk = rel_delta_t<D>(k_new, k_old);
    dr = rel_delta_t<1>(&e_rho, &e_rho_old);
    dl = rel_delta_t<D * D>(L, l_old);
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

  TAIL_PROF(c, 4);
  // ---- stores
  s.status = status;
  s.d = D;
  s.V = (int64_t)h.V;
  s.n_iter = mode == MODE_SWEEP ? n_iter_old + 1 : 0;
  s.a_rho = a;
  s.b_rho = b;
  s.e_rho = e_rho;
  s.ln_det_lam0l_inv = ld;
  s.resid = st[stat_R(D)];
  s.elbo = elbo;
  s.elbo_status = elbo_status;
  s.gen_lnA = gen.lnA;
  s.gen_e_rho = gen.e_rho;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    s.k0k[i] = k_new[i];
    s.e_lamk[i] = elamk[i];
    s.gen_c[i] = gen.c[i];
  }
#pragma unroll
  for (int i = 0; i < D * D; ++i) {
    s.lam0l_inv[i] = L[i];
    s.e_lam[i] = h.nu * S[i];
    s.gen_A[i] = gen.A[i];
    s.gen_Ainv[i] = gen.Ainv[i];
  }
  if (sweep_ok && iter < tr_cap) {
    tr_dk[iter] = dk;
    tr_drho[iter] = dr;
    tr_dlam[iter] = dl;
    tr_elbo[iter] = compute_elbo ? elbo : qnan();
  }
  c.iter = new_iter;
  c.have_prev = new_have_prev;
  c.prev_elbo = new_prev;
  if (c_status != CV_OK) c.status = c_status;
  if (done) c.done = 1;
  c.mode = MODE_SWEEP;
  if (status == CV_OK) {
    // generator of the next pass (vb.py:136-144)
    const double rnu = 1.0 / h.nu;
#pragma unroll
    for (int i = 0; i < D; ++i) c.pass.c[i] = k_new[i];
#pragma unroll
    for (int i = 0; i < D * D; ++i) {
      c.pass.A[i] = h.nu * S[i];
      c.pass.Ainv[i] = L[i] * rnu;
    }
    c.pass.lnA = D * h.ln_nu - ld;
    const double nb = h.b0 + 0.5 * st[stat_R(D)];
    c.pend_a = h.a_fit;
    c.pend_b = nb;
    c.pass.e_rho = h.a_fit / nb;
  }
  TAIL_PROF(c, 5);
}

}  // namespace cavi
