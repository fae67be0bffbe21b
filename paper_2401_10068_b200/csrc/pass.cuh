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
//
// Kernel (sm_100a, persistent, one CTA per SM): a producer warp streams the
// CTA's chunks tile by tile into a ring of shared-memory stages with TMA bulk
// copies (cp.async.bulk + mbarrier complete_tx, L2 evict-first for streams
// larger than L2); 8 consumer warps compute out of shared memory and release
// stages through "empty" mbarriers.  The thread->gene map inside a chunk is
// fixed, so each chunk partial is bit-reproducible whatever CTA computes it.
// Chunk partials -> group (64 chunks, index order, by the CTA that completes
// the group) -> octants (index order) -> pairwise tree over the octants, by
// the CTA that completes the last group, which then runs the tail
// (engine.cuh) or, on a multi-GPU shard, publishes its octant subtree.
#pragma once

#include "engine.cuh"
#include "ptx.cuh"

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
  int l2_keep;             // stream fits in L2: keep it resident across sweeps
  double* partials;        // [n_chunks][ns]
  double* gpartials;       // [n_groups][ns]
  unsigned int* gcount;    // [n_groups]
  unsigned int* gdone;     // [1]
  Ctl* ctl;
  const Hyp* hyp;
  double* rank_out;        // multi-GPU: [ns] subtree partial of this shard; null -> run the tail
};

typedef void (*PassFn)(PassArgs);

struct PassKernel {
  PassFn fn;
  int threads;
  int smem;  // dynamic shared memory bytes
};

__device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t lmax(int64_t a, int64_t b) { return a > b ? a : b; }

// Running product of den with exponent renormalisation: one log per thread-chunk.
struct LogAcc {
  double m;
  int e;
  __device__ __forceinline__ void init() {
    m = 1.0;
    e = 0;
  }
  __device__ __forceinline__ void mul(double p) {
    m *= p;
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
__device__ __forceinline__ void load_coef(GeneCoef<D>& k, const Gen& g) {
#pragma unroll
  for (int j = 0; j < D; ++j) k.c[j] = g.c[j];
  int p = 0;
#pragma unroll
  for (int j = 0; j < D; ++j)
#pragma unroll
    for (int q = j; q < D; ++q) k.A2[p++] = (q == j ? 1.0 : 2.0) * g.Ainv[j * D + q];
  k.erho = g.e_rho;
}

// one gene: accumulate its statistics, return den
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
  const double inv = ptx::rcp_nr(den);
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
// Executed by the `nthr` consumer threads (tid in [0, nthr)), synchronised on named barrier 1.
template <int D>
__device__ void finish_group_and_maybe_tail(const PassArgs& a, int64_t grp, double* s_tot, int* s_flag, int tid,
                                            int nthr) {
  constexpr int NS = n_stats(D);
  const int64_t c0 = grp * kGroupChunks;
  const int64_t c1 = lmin(c0 + kGroupChunks, a.n_chunks);
  if (tid < NS) {
    double s = 0.0;
    const int n = (int)(c1 - c0);
#pragma unroll 8
    for (int i = 0; i < kGroupChunks; ++i)
      if (i < n) s += __ldcg(a.partials + (c0 + i) * NS + tid);
    a.gpartials[grp * NS + tid] = s;
  }
  __threadfence();
  ptx::bar_sync(1, nthr);
  if (tid == 0) {
    a.gcount[grp] = 0u;  // ready for the next sweep
    const unsigned int prev = atomicAdd(a.gdone, 1u);
    *s_flag = (prev == (unsigned int)(a.n_groups - 1));
  }
  ptx::bar_sync(1, nthr);
  if (!*s_flag) return;
  __threadfence();
  if (tid < NS) {
    double oct[kOctants];
#pragma unroll
    for (int o = 0; o < kOctants; ++o) oct[o] = 0.0;
    for (int o = a.oct_lo; o < a.oct_hi; ++o) {
      const int64_t g0 = lmax((int64_t)o * a.groups_per_octant, a.group_lo);
      const int64_t g1 = lmin(lmin((int64_t)(o + 1) * a.groups_per_octant, a.n_groups_total), a.group_lo + a.n_groups);
      double s = 0.0;
#pragma unroll 8
      for (int64_t gg = g0; gg < g1; ++gg) s += __ldcg(a.gpartials + (gg - a.group_lo) * NS + tid);
      oct[o] = s;
    }
    // pairwise tree over the owned octants (a power-of-two aligned span)
    for (int w = 1; w < a.oct_hi - a.oct_lo; w *= 2)
      for (int o = a.oct_lo; o + w < a.oct_hi; o += 2 * w) oct[o] = oct[o] + oct[o + w];
    s_tot[tid] = oct[a.oct_lo];
  }
  if (tid == 0) *a.gdone = 0u;
  ptx::bar_sync(1, nthr);
  if (a.rank_out) {
    if (tid < NS) a.rank_out[tid] = s_tot[tid];
  } else if (tid == 0) {
    tail_t<D>(*a.hyp, *a.ctl, s_tot);
  }
}

// chunk partial (fixed-order block reduction) -> partials[chunk]; group / final bookkeeping
template <int D, int NWARPS, int NS = n_stats(D)>
__device__ __forceinline__ void publish_chunk(const PassArgs& a, int64_t chunk, double (&acc)[NS],
                                              double (*s_warp)[NS], double* s_tot, int* s_flag, int tid) {
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int NTHR = NWARPS * 32;
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    double v = acc[i];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) s_warp[warp][i] = v;
  }
  ptx::bar_sync(1, NTHR);
  if (tid < NS) {
    double s = s_warp[0][tid];
#pragma unroll
    for (int w = 1; w < NWARPS; ++w) s += s_warp[w][tid];
    a.partials[chunk * NS + tid] = s;
  }
  __threadfence();
  ptx::bar_sync(1, NTHR);
  const int64_t grp = chunk / kGroupChunks;
  if (tid == 0) {
    const unsigned int need = (unsigned int)(lmin((grp + 1) * kGroupChunks, a.n_chunks) - grp * kGroupChunks);
    const unsigned int prev = atomicAdd(a.gcount + grp, 1u);
    *s_flag = (prev == need - 1);
  }
  ptx::bar_sync(1, NTHR);
  if (*s_flag) {
    __threadfence();
    finish_group_and_maybe_tail<D>(a, grp, s_tot, s_flag, tid, NTHR);
  }
  ptx::bar_sync(1, NTHR);
}

// ---------------------------------------------------------------- pipeline geometry
template <int D, typename T>
struct Geometry {
  static constexpr int kTile = D <= 3 ? 1024 : (D <= 7 ? 512 : 256);  // genes per stage
  static constexpr int kTilesPerChunk = kChunk / kTile;
  static constexpr int kGenesPerThread = kTile / kThreads;  // consumer genes per stage
  static constexpr uint32_t kColBytes = kTile * sizeof(T);
  static constexpr uint32_t kStageBytes = kColBytes * (1 + D);
  static constexpr int kStages = (196608 / kStageBytes) > 8 ? 8 : (196608 / kStageBytes);
  static constexpr int kSmem = kStages * kStageBytes + 2 * kStages * 8;
  static_assert(kStages >= 2, "stage too large");
  static_assert(kTile % kThreads == 0, "tile must split evenly across consumers");
};

constexpr int kProducerWarp = kWarps;       // warp index of the TMA producer
constexpr int kCtaThreads = kThreads + 32;  // 8 consumer warps + 1 producer warp

template <int D, typename T>
__global__ void __launch_bounds__(kCtaThreads, 1) pass_kernel(PassArgs a) {
  using G = Geometry<D, T>;
  constexpr int NS = n_stats(D);
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double s_warp[kWarps][NS];
  __shared__ double s_tot[NS];
  __shared__ int s_flag;
  T* stage_base = reinterpret_cast<T*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G::kStages * G::kStageBytes);
  uint64_t* empty = full + G::kStages;

  const Ctl* ctl = a.ctl;
  if (*(volatile const int*)&ctl->done) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < G::kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], kWarps);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();

  if (warp == kProducerWarp) {
    // ---------------- TMA producer: one elected lane streams every tile of this CTA's chunks
    if (lane == 0) {
      const T* xs = static_cast<const T*>(a.x);
      const T* Ds = static_cast<const T*>(a.D);
      const uint64_t pol = a.l2_keep ? ptx::policy_evict_last() : ptx::policy_evict_first();
      int stage = 0;
      uint32_t parity = 1;  // fresh "empty" barriers count as released
      for (int64_t chunk = blockIdx.x; chunk < a.n_chunks; chunk += gridDim.x) {
        for (int t = 0; t < G::kTilesPerChunk; ++t) {
          ptx::mbar_wait(&empty[stage], parity);
          ptx::mbar_arrive_expect_tx(&full[stage], G::kStageBytes);
          const int64_t g0 = chunk * kChunk + (int64_t)t * G::kTile;
          T* dst = stage_base + (size_t)stage * (G::kStageBytes / sizeof(T));
          ptx::bulk_g2s(dst, xs + g0, G::kColBytes, &full[stage], pol);
#pragma unroll
          for (int j = 0; j < D; ++j)
            ptx::bulk_g2s(dst + (size_t)(j + 1) * G::kTile, Ds + (int64_t)j * a.Vp + g0, G::kColBytes, &full[stage],
                          pol);
          if (++stage == G::kStages) {
            stage = 0;
            parity ^= 1u;
          }
        }
      }
    }
    return;  // consumers synchronise on named barrier 1 only
  }

  // ---------------- consumers
  GeneCoef<D> k;
  load_coef<D>(k, ctl->pass);
  const int tid = threadIdx.x;  // 0 .. kThreads-1
  int stage = 0;
  uint32_t parity = 0;
  for (int64_t chunk = blockIdx.x; chunk < a.n_chunks; chunk += gridDim.x) {
    double acc[NS];
#pragma unroll
    for (int i = 0; i < NS; ++i) acc[i] = 0.0;
    LogAcc lg;
    lg.init();
#pragma unroll 1
    for (int t = 0; t < G::kTilesPerChunk; ++t) {
      ptx::mbar_wait(&full[stage], parity);
      const T* tile = stage_base + (size_t)stage * (G::kStageBytes / sizeof(T));
      double prod = 1.0;
#pragma unroll
      for (int u = 0; u < G::kGenesPerThread; ++u) {
        const int gi = u * kThreads + tid;
        double Dv[D];
#pragma unroll
        for (int j = 0; j < D; ++j) Dv[j] = (double)tile[(j + 1) * G::kTile + gi];
        prod *= gene<D>(k, (double)tile[gi], Dv, acc);
      }
      lg.mul(prod);
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&empty[stage]);
      if (++stage == G::kStages) {
        stage = 0;
        parity ^= 1u;
      }
    }
    acc[NS - 1] = lg.log_value();
    publish_chunk<D, kWarps>(a, chunk, acc, s_warp, s_tot, &s_flag, tid);
  }
}

}  // namespace cavi
