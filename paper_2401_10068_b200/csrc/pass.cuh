// pass.cuh -- the fused CAVI E-pass: one streaming read of the measurement
// stream per sweep, per-gene rank-1 beta block in registers, deterministic
// hierarchical reduction, and the sweep tail in the last CTA.
//
// Restates, per gene i (reference vb.py:146-170 + vb.py:114-126 + vb.py:233-258):
//   Lambda_beta_i = A + e_rho D_i D_i^T, mu_beta_i = Lambda_beta_i^-1 (A c + e_rho x_i D_i)
// via Sherman-Morrison:  s = D^T A^-1 D, t = D^T c, den = 1 + e_rho s,
//   w = e_rho (x - t)/den,  gamma = w^2 - e_rho/den,  resid = (x - t - s w)^2 + s/den
// accumulating  g += w D,  G += gamma D D^T,  R += resid,  Ld += ln den.
//
// HBM layout (SoA, padded to whole chunks with zero genes, which contribute
// exactly 0 to every statistic):  x[Vp] then D column j at D + j*Vp.
// Work decomposition: persistent CTAs stride over 4096-gene chunks; the
// thread->gene map inside a chunk is fixed, so each chunk's partial is
// bit-reproducible whatever CTA computes it.  Chunk partials -> group (64
// chunks, index order, by the CTA that completes the group) -> octants (index
// order) -> pairwise tree over the octants, by the CTA that completes the last
// group, which then runs the tail (engine.cuh) or, on a multi-GPU shard,
// publishes its octant subtree for the exchange.
#pragma once

#include "engine.cuh"

namespace cavi {

struct PassArgs {
  const void* x;
  const void* D;
  int64_t Vp;
  int64_t n_chunks;        // local chunks
  int64_t n_groups;        // local groups
  int64_t group_lo;        // global index of local group 0
  int64_t n_groups_total;  // groups of the whole dataset
  int64_t groups_per_octant;
  int oct_lo, oct_hi;      // octants this shard owns
  double* partials;        // [n_chunks][ns]
  double* gpartials;       // [n_groups][ns]
  unsigned int* gcount;    // [n_groups]
  unsigned int* gdone;     // [1]
  Ctl* ctl;
  const Hyp* hyp;
  double* rank_out;        // multi-GPU: [ns] subtree partial of this shard; null -> run the tail
};

__device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t lmax(int64_t a, int64_t b) { return a > b ? a : b; }

template <typename T>
struct Vec2;
template <>
struct Vec2<double> {
  using type = double2;
};
template <>
struct Vec2<float> {
  using type = float2;
};

__device__ __forceinline__ double2 ld2(const double* p, int64_t i) {
  return __ldg(reinterpret_cast<const double2*>(p) + i);
}
__device__ __forceinline__ double2 ld2(const float* p, int64_t i) {
  const float2 v = __ldg(reinterpret_cast<const float2*>(p) + i);
  return make_double2((double)v.x, (double)v.y);
}

// Running product of den with exponent renormalisation: one log per thread-chunk.
struct LogAcc {
  double m;
  int e;
  __device__ __forceinline__ void init() {
    m = 1.0;
    e = 0;
  }
  __device__ __forceinline__ void mul(double a, double b) {
    m *= a * b;
    const int hi = __double2hiint(m);
    const int lo = __double2loint(m);
    e += ((hi >> 20) & 0x7ff) - 1023;
    m = __hiloint2double((hi & 0x800fffff) | 0x3ff00000, lo);
  }
  __device__ __forceinline__ double log_value() const { return log(m) + (double)e * kLn2; }
};

template <int D>
struct GeneCoef {
  double c[D];
  double A2[D * (D + 1) / 2];  // upper triangle of A^-1, off-diagonals doubled
  double erho;
};

template <int D>
__device__ __forceinline__ double gene(const GeneCoef<D>& k, double x, const double (&Dv)[D],
                                       double (&acc)[n_stats(D)]) {
  double P[D * (D + 1) / 2];
  double t = 0.0, s = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) t = fma(k.c[j], Dv[j], t);
  {
    int p = 0;
#pragma unroll
    for (int j = 0; j < D; ++j)
#pragma unroll
      for (int q = j; q < D; ++q) {
        P[p] = Dv[j] * Dv[q];
        s = fma(k.A2[p], P[p], s);
        ++p;
      }
  }
  const double den = fma(k.erho, s, 1.0);
  const double inv = __drcp_rn(den);
  const double xt = x - t;
  const double ei = k.erho * inv;
  const double w = ei * xt;
  const double gam = fma(w, w, -ei);
  const double e = fma(-s, w, xt);
  acc[n_stats(D) - 2] += fma(e, e, s * inv);
#pragma unroll
  for (int j = 0; j < D; ++j) acc[j] = fma(w, Dv[j], acc[j]);
#pragma unroll
  for (int p = 0; p < D * (D + 1) / 2; ++p) acc[D + p] = fma(gam, P[p], acc[D + p]);
  return den;
}

// Sum of the group's chunk partials (index order) / octants (index order) / pairwise tree.
template <int NS>
__device__ void finish_group_and_maybe_tail(const PassArgs& a, int64_t grp, double* s_tot, int* s_flag) {
  const int tid = threadIdx.x;
  const int64_t c0 = grp * kGroupChunks;
  const int64_t c1 = lmin(c0 + kGroupChunks, a.n_chunks);
  if (tid < NS) {
    double s = 0.0;
    for (int64_t c = c0; c < c1; ++c) s += __ldcg(a.partials + c * NS + tid);
    a.gpartials[grp * NS + tid] = s;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    a.gcount[grp] = 0u;  // ready for the next sweep
    const unsigned int prev = atomicAdd(a.gdone, 1u);
    *s_flag = (prev == (unsigned int)(a.n_groups - 1));
  }
  __syncthreads();
  if (!*s_flag) return;
  __threadfence();
  if (tid < NS) {
    double oct[kOctants];
#pragma unroll
    for (int o = 0; o < kOctants; ++o) oct[o] = 0.0;
    for (int o = a.oct_lo; o < a.oct_hi; ++o) {
      const int64_t g0 = lmax((int64_t)o * a.groups_per_octant, a.group_lo);
      const int64_t g1 = lmin(lmin((int64_t)(o + 1) * a.groups_per_octant, a.n_groups_total),
                                      a.group_lo + a.n_groups);
      double s = 0.0;
      for (int64_t gg = g0; gg < g1; ++gg) s += __ldcg(a.gpartials + (gg - a.group_lo) * NS + tid);
      oct[o] = s;
    }
    // pairwise tree over the owned octants (a power-of-two aligned span)
    for (int w = 1; w < a.oct_hi - a.oct_lo; w *= 2)
      for (int o = a.oct_lo; o + w < a.oct_hi; o += 2 * w) oct[o] = oct[o] + oct[o + w];
    s_tot[tid] = oct[a.oct_lo];
  }
  if (tid == 0) *a.gdone = 0u;
  __syncthreads();
  if (a.rank_out) {
    if (tid < NS) a.rank_out[tid] = s_tot[tid];
  } else if (tid == 0) {
    tail(*a.hyp, *a.ctl, s_tot);
  }
}

template <int D, typename T>
__global__ void __launch_bounds__(kThreads, 2) pass_kernel(PassArgs a) {
  constexpr int NS = n_stats(D);
  constexpr int PAIRS = kChunk / 2 / kThreads;  // 8 double-pairs per thread per chunk
  constexpr int BATCH = (D <= 2) ? 4 : (D <= 4 ? 2 : 1);
  __shared__ double s_warp[kWarps][NS];
  __shared__ double s_tot[NS];
  __shared__ int s_flag;
  const Ctl* ctl = a.ctl;
  if (*(volatile const int*)&ctl->done) return;

  GeneCoef<D> k;
  {
    const Gen& g = ctl->pass;
#pragma unroll
    for (int j = 0; j < D; ++j) k.c[j] = g.c[j];
    int p = 0;
#pragma unroll
    for (int j = 0; j < D; ++j)
#pragma unroll
      for (int q = j; q < D; ++q) k.A2[p++] = (q == j ? 1.0 : 2.0) * g.Ainv[j * D + q];
    k.erho = g.e_rho;
  }
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const T* __restrict__ xs = static_cast<const T*>(a.x);
  const T* __restrict__ Ds = static_cast<const T*>(a.D);

  for (int64_t chunk = blockIdx.x; chunk < a.n_chunks; chunk += gridDim.x) {
    double acc[NS];
#pragma unroll
    for (int i = 0; i < NS; ++i) acc[i] = 0.0;
    LogAcc lg;
    lg.init();
    const int64_t pair0 = chunk * (kChunk / 2) + tid;
#pragma unroll 1
    for (int b = 0; b < PAIRS; b += BATCH) {
      double2 xv[BATCH];
      double2 dv[BATCH][D];
#pragma unroll
      for (int u = 0; u < BATCH; ++u) {
        const int64_t pi = pair0 + (int64_t)(b + u) * kThreads;
        xv[u] = ld2(xs, pi);
#pragma unroll
        for (int j = 0; j < D; ++j) dv[u][j] = ld2(Ds + (int64_t)j * a.Vp, pi);
      }
#pragma unroll
      for (int u = 0; u < BATCH; ++u) {
        double d0[D], d1[D];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          d0[j] = dv[u][j].x;
          d1[j] = dv[u][j].y;
        }
        const double den0 = gene<D>(k, xv[u].x, d0, acc);
        const double den1 = gene<D>(k, xv[u].y, d1, acc);
        lg.mul(den0, den1);
      }
    }
    acc[NS - 1] = lg.log_value();
    // block reduction, fixed order: warp butterfly, then warps in index order
#pragma unroll
    for (int i = 0; i < NS; ++i) {
      double v = acc[i];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) s_warp[warp][i] = v;
    }
    __syncthreads();
    if (tid < NS) {
      double s = s_warp[0][tid];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) s += s_warp[w][tid];
      a.partials[chunk * NS + tid] = s;
    }
    __threadfence();
    __syncthreads();
    const int64_t grp = chunk / kGroupChunks;
    if (tid == 0) {
      const unsigned int need = (unsigned int)(lmin((grp + 1) * kGroupChunks, a.n_chunks) - grp * kGroupChunks);
      const unsigned int prev = atomicAdd(a.gcount + grp, 1u);
      s_flag = (prev == need - 1);
    }
    __syncthreads();
    if (s_flag) {
      __threadfence();
      finish_group_and_maybe_tail<NS>(a, grp, s_tot, &s_flag);
    }
    __syncthreads();
  }
}

typedef void (*PassFn)(PassArgs);

}  // namespace cavi
