// batched.cuh -- many independent small CAVI fits in one launch (BASELINE config 4:
// 1e4 fibroblast-shaped tissue samples, V=56, N=3).  One THREAD owns one fit and runs its
// whole vb_fit loop (reference vb.py:312-354) in-kernel: per sweep a serial pass over the
// fit's genes (the same per-gene algebra as the streaming kernel, gene<D>()) and the same
// tail_t<D> as the single-fit engine on the fit's own control block.  All 32 lanes of a
// warp run 32 fits' tails side by side (a warp-per-fit layout ran the serial tail on one
// lane: 1/32 of the FP64 issue).  Fits are independent: no inter-thread communication;
// multi-GPU partitions the fits (no collective).
#pragma once

#include "pass.cuh"

namespace cavi {

struct BatchArgs {
  const double* r;            // concatenated readings of all fits
  const double* mu;
  const double* D;            // row-major (genes, d)
  const int64_t* offsets;     // [n_fits + 1] gene ranges
  int64_t n_fits;
  Hyp* hyps;                  // [n_fits] (V differs per fit)
  Ctl* ctls;                  // [n_fits]
};

constexpr int kBatchThreads = 32;  // fits per CTA: spreads 1e4 fits over every SM

template <int D>
__global__ void __launch_bounds__(kBatchThreads) batched_fit_kernel(BatchArgs a) {
  constexpr int NS = n_stats(D);
  const int64_t fit = (int64_t)blockIdx.x * kBatchThreads + threadIdx.x;
  if (fit >= a.n_fits) return;
  Hyp& h = a.hyps[fit];
  Ctl& c = a.ctls[fit];
  const int64_t g0 = a.offsets[fit], g1 = a.offsets[fit + 1];
  // vb_init's generator (K0, Lambda0, e_rho = 0): the init pass measures resid_0 and the bound
  for (int i = 0; i < D; ++i) c.pass.c[i] = h.K0[i];
  for (int i = 0; i < D * D; ++i) {
    c.pass.A[i] = h.L0[i];
    c.pass.Ainv[i] = h.L0inv[i];
  }
  c.pass.lnA = h.lnL0;
  c.pass.e_rho = 0.0;
  c.mode = MODE_INIT;
  for (;;) {
    GeneCoef<D> k;
    load_coef<D>(k, c.pass);
    double acc[NS];
#pragma unroll
    for (int i = 0; i < NS; ++i) acc[i] = 0.0;
    LogAcc lg;
    lg.init();
    for (int64_t gi = g0; gi < g1; ++gi) {
      double Dv[D];
#pragma unroll
      for (int j = 0; j < D; ++j) Dv[j] = __ldg(a.D + gi * D + j);
      const double x = __dsub_rn(__ldg(a.r + gi), __ldg(a.mu + gi));  // rm = r - mu (vb.py:149)
      lg.mul(gene<D>(k, x, Dv, acc));
    }
    acc[stat_Ld(D)] = lg.log_value();
    double Tm[D * D], hv[D];
    pass_products_t<D>(c.pass.Ainv, acc, Tm, hv);
    tail_t<D>(h, c, acc, Tm, hv);
    if (c.done) break;
  }
}

}  // namespace cavi
