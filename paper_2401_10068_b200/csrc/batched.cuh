// batched.cuh -- many independent small CAVI fits in one launch (BASELINE config 4:
// 1e4 fibroblast-shaped tissue samples, V=56, N=3).  One warp owns one fit and runs
// its whole vb_fit loop (reference vb.py:312-354) in-kernel: per sweep a warp-wide
// pass over the fit's genes (the same per-gene algebra as the streaming kernel,
// gene<D>()), a fixed warp-butterfly reduction, and lane 0 runs the same tail_t<D>
// as the single-fit engine on the fit's own control block.  Fits are independent:
// no inter-warp communication at all; multi-GPU partitions the fits (no collective).
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

constexpr int kBatchWarps = 4;  // fits per CTA

template <int D>
__global__ void __launch_bounds__(kBatchWarps * 32) batched_fit_kernel(BatchArgs a) {
  constexpr int NS = n_stats(D);
  __shared__ double s_stats[kBatchWarps][NS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t fit = (int64_t)blockIdx.x * kBatchWarps + warp;
  if (fit >= a.n_fits) return;
  Hyp& h = a.hyps[fit];
  Ctl& c = a.ctls[fit];
  const int64_t g0 = a.offsets[fit], g1 = a.offsets[fit + 1];
  if (lane == 0) {
    // vb_init's generator (K0, Lambda0, e_rho = 0): the init pass measures resid_0 and the bound
    for (int i = 0; i < D; ++i) c.pass.c[i] = h.K0[i];
    for (int i = 0; i < D * D; ++i) {
      c.pass.A[i] = h.L0[i];
      c.pass.Ainv[i] = h.L0inv[i];
    }
    c.pass.lnA = h.lnL0;
    c.pass.e_rho = 0.0;
    c.mode = MODE_INIT;
  }
  __syncwarp();
  for (;;) {
    GeneCoef<D> k;
    load_coef<D>(k, c.pass);
    double acc[NS];
#pragma unroll
    for (int i = 0; i < NS; ++i) acc[i] = 0.0;
    LogAcc lg;
    lg.init();
    for (int64_t gi = g0 + lane; gi < g1; gi += 32) {
      double Dv[D];
#pragma unroll
      for (int j = 0; j < D; ++j) Dv[j] = __ldg(a.D + gi * D + j);
      const double x = __dsub_rn(__ldg(a.r + gi), __ldg(a.mu + gi));  // rm = r - mu (vb.py:149)
      lg.mul(gene<D>(k, x, Dv, acc));
    }
    acc[stat_Ld(D)] = lg.log_value();
#pragma unroll
    for (int i = 0; i < NS; ++i) {
      double v = acc[i];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == (i & 31)) s_stats[warp][i] = v;
    }
    __syncwarp();
    int done = 0;
    if (lane == 0) {
      tail_t<D>(h, c, s_stats[warp]);
      done = c.done;
    }
    done = __shfl_sync(0xffffffffu, done, 0);
    __syncwarp();
    if (done) break;
  }
}

}  // namespace cavi
