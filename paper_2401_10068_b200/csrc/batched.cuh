// batched.cuh -- many independent small CAVI fits in one launch (BASELINE config 4:
// 1e4 fibroblast-shaped tissue samples, V=56, N=3).  Each fit runs its whole vb_fit loop
// (reference vb.py:312-354) in-kernel on a GROUP of kBatchLanes lanes:
//   per sweep  the group's lanes split the fit's genes (lane j: genes j, j + L, ...), each
//              accumulating the per-gene algebra of the streaming kernel (gene<D>()) into
//              registers; an xor butterfly inside the group (log2 L steps) gives every lane
//              the fit's statistic vector;
//   tail       the group's first lane runs the single-fit engine's tail (tail_t<D>) on the
//              fit's own control block; the other lanes wait at the group's next shuffle.
// With L = 8, 1e4 fits are 8e4 threads (17 warps per SM) where one thread per fit left ~2
// warps per SM to hide every load and FP64 latency (round 1: 18 ms of kernel for 1e4 fits).
// The 32 / L groups of a warp are independent fits (different V, different iteration counts):
// every shuffle is masked to the group.  Fits are independent: multi-GPU partitions them.
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

#ifndef CAVI_BATCH_LANES
#define CAVI_BATCH_LANES 8
#endif
constexpr int kBatchLanes = CAVI_BATCH_LANES;        // lanes per fit
constexpr int kBatchThreads = 128;                    // 16 fits per CTA
constexpr int kBatchFitsPerCta = kBatchThreads / kBatchLanes;

template <int D>
__global__ void __launch_bounds__(kBatchThreads) batched_fit_kernel(BatchArgs a) {
  constexpr int NS = n_stats(D);
  constexpr int L = kBatchLanes;
  const int lane = threadIdx.x & 31;
  const int sub = lane % L;                                   // lane within the fit's group
  const unsigned gmask = (L == 32 ? 0xffffffffu : ((1u << L) - 1u)) << (lane - sub);
  const int64_t fit = (int64_t)blockIdx.x * kBatchFitsPerCta + threadIdx.x / L;
  if (fit >= a.n_fits) return;  // whole groups leave together
  Hyp& h = a.hyps[fit];
  Ctl& c = a.ctls[fit];
  const int64_t g0 = a.offsets[fit], g1 = a.offsets[fit + 1];
  if (sub == 0) {  // vb_init's generator (K0, Lambda0, e_rho = 0): the init pass measures resid_0 and the bound
    for (int i = 0; i < D; ++i) c.pass.c[i] = h.K0[i];
    for (int i = 0; i < D * D; ++i) {
      c.pass.A[i] = h.L0[i];
      c.pass.Ainv[i] = h.L0inv[i];
    }
    c.pass.lnA = h.lnL0;
    c.pass.e_rho = 0.0;
    c.mode = MODE_INIT;
  }
  __syncwarp(gmask);
  for (;;) {
    GeneCoef<D> k;
    load_coef<D>(k, c.pass);
    double acc[NS];
#pragma unroll
    for (int i = 0; i < NS; ++i) acc[i] = 0.0;
    LogAcc lg;
    lg.init();
    for (int64_t gi = g0 + sub; gi < g1; gi += L) {
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
      for (int off = L / 2; off > 0; off >>= 1) v += __shfl_xor_sync(gmask, v, off);
      acc[i] = v;
    }
    int done = 0;
    if (sub == 0) {
      double Tm[D * D], hv[D];
      pass_products_t<D>(c.pass.Ainv, acc, Tm, hv);
      tail_t<D>(h, c, acc, Tm, hv);
      done = c.done;
    }
    __syncwarp(gmask);  // the tail's stores (next generator) before the group's next loads
    if (__shfl_sync(gmask, done, lane - sub)) break;
  }
}

}  // namespace cavi
