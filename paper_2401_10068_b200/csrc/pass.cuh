// pass.cuh -- the fused CAVI E-pass: one streaming read of the measurement stream per
// sweep, per-gene rank-1 beta block, deterministic hierarchical reduction; plus the
// one-warp tail kernel that turns the pass statistics into the next state.
//
// Restates, per gene i (reference vb.py:146-170 + vb.py:114-126 + vb.py:233-258):
//   Lambda_beta_i = A + e_rho D_i D_i^T, mu_beta_i = Lambda_beta_i^-1 (A c + e_rho x_i D_i)
// via Sherman-Morrison:  s = D^T A^-1 D, t = D^T c, den = 1 + e_rho s,
//   w = e_rho (x - t)/den,  gamma = w^2 - e_rho/den,  resid = (x - t - s w)^2 + s/den
// accumulating  g += w D,  G += gamma D D^T,  R += resid,  Q += w (x - t),  Ld += ln den.
//
// HBM layout (SoA, padded to whole chunks with zero genes, which contribute
// exactly 0 to every statistic):  x[Vp] then D column j at D + j*Vp.
//
// Kernel (sm_100a, persistent, 2-3 CTAs per SM): a producer warp streams the CTA's
// chunks (dynamic tickets) tile by tile into a ring of shared-memory stages with TMA
// bulk copies (cp.async.bulk + mbarrier complete_tx, L2 evict-first for streams larger
// than L2); 4 consumer warps compute out of shared memory (d <= 7: one gene per thread
// in registers; d >= 8: fp64 tensor cores, MmaConsumer) and release stages through
// "empty" mbarriers.  The thread->gene map inside a chunk is fixed, so each chunk
// partial is bit-reproducible whatever CTA computes it.  Chunk partials -> group (64
// chunks) -> octants -> pairwise tree over the octants, each level by whichever warp
// completes it (fixed-order sums); the last one writes the shard totals, or on a
// multi-GPU shard stores them into every peer's window (lsa.cuh).
#pragma once

#include "engine.cuh"
#include "lsa.cuh"
#include "ptx.cuh"
#include "tail.cuh"

namespace cavi {

// statistics per polling pass of an LL row sum: the row words are live beside the consumer
// loop's registers (warp_rows_ll is inlined into it), so wider statistic vectors poll in smaller
// batches (V=1e8: N=5 1692 -> 1712 sweeps/s at 8 instead of 16)
constexpr int ll_batch(int ns) { return ns <= 12 ? 16 : ns <= 17 ? 8 : 4; }
#ifndef CAVI_LL_MAX_D
#define CAVI_LL_MAX_D 4  // largest d on the LL cascade (memory-bound); above: acquire/release rows
                         // (V=1e8, LL vs acq/rel: N=6 1368 vs 1395, N=7 1001 vs 1125, N=8 685 vs 871;
                         // profiles/r02_ll7_ab.log)
#endif

struct PassArgs {
  const void* x;
  const void* D;
  int64_t Vp;
  int64_t n_chunks;        // local chunks
  int chunk_genes;         // genes per chunk (plan_chunk_genes: 4096 or 8192)
  int group_chunks;        // chunks per group (kGroupGenes / chunk_genes)
  int64_t n_groups;        // local groups
  int64_t group_lo;        // global index of local group 0
  int64_t n_groups_total;  // groups of the whole dataset
  int64_t groups_per_octant;
  int oct_lo, oct_hi;      // octants this shard owns
  int l2_keep;             // stream fits in L2: keep it resident across sweeps
  uint64_t* partials;      // [n_chunks][ns][2] chunk sums, LL words (tag = *pass_seq)
  uint64_t* gpartials;     // [n_groups][ns][2] group sums, LL
  unsigned int* gcount;    // [n_groups] arrivals per group
  unsigned int* ocount;    // [8] arrivals per octant
  unsigned int* odone;     // [1] completed octants (acquire/release cascade)
  uint64_t* opartials;     // [8][ns][2] octant sums, LL
  int oct_last;            // the shard's last octant holding groups (the LL cascade's final level)
  unsigned int* pass_seq;  // [1] passes completed on this dataset = the LL tag of the running pass
  unsigned long long* ticket;  // chunk tickets (monotone across sweeps)
  int n_live_octants;      // octants of this shard holding at least one group
  Ctl* ctl;
  const Hyp* hyp;
  double* rank_out;        // [ns] totals of this shard (its octant subtree), read by the tail kernel
  LsaLink lsa;             // multi-GPU: publish the shard totals into every peer (lsa.win != null)
  unsigned long long* cta_trace;  // optional [grid][8] globaltimer stamps (diagnostics)
};

typedef void (*PassFn)(PassArgs);
struct BatchArgs;
struct WishartArgs;

struct PassKernel {
  PassFn fn;
  int threads;
  int smem;  // dynamic shared memory bytes
  void (*tail)(const Hyp*, Ctl*, const double*, int, LsaLink);
  void (*batched)(BatchArgs);
  void (*rate_inverse_test)(const double*, double*, double*, int*);
  void (*wishart_seg)(WishartArgs);
  void (*wishart_fin)(WishartArgs, const double*, const double*, double, uint64_t, double*, double*);
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned int smid() {
  unsigned int r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}

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

// The optional fp32-math stream (CV_STORE_F32M): fp32 storage AND fp32 per-gene arithmetic,
// the per-thread tile sums (8 genes) promoted to the fp64 accumulators, the den product in
// fp64 -- SURVEY 7.7's fp32 variant, parity 1e-4 (the fp64 statistics are sums of ~1e-7
// relative per-gene terms).  Same algebra as gene<D>(); resid uses e = (x - t)/den
// (= x - t - s w exactly, no cancellation in fp32).
template <int D>
struct GeneCoefF {
  float c[D];
  float A2[D * (D + 1) / 2];
  float erho;
};

template <int D>
__device__ __forceinline__ void load_coef_f(GeneCoefF<D>& k, const Gen& g) {
#pragma unroll
  for (int j = 0; j < D; ++j) k.c[j] = (float)g.c[j];
  int p = 0;
#pragma unroll
  for (int j = 0; j < D; ++j)
#pragma unroll
    for (int q = j; q < D; ++q) k.A2[p++] = (float)((q == j ? 1.0 : 2.0) * g.Ainv[j * D + q]);
  k.erho = (float)g.e_rho;
}

template <int D>
__device__ __forceinline__ float gene_f(const GeneCoefF<D>& k, float x, const float (&Dv)[D],
                                        float (&acc)[n_stats(D)]) {
  float t = 0.f, s = 0.f;
#pragma unroll
  for (int j = 0; j < D; ++j) t = fmaf(k.c[j], Dv[j], t);
  {
    int p = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      float r = 0.f;
#pragma unroll
      for (int q = j; q < D; ++q) r = fmaf(k.A2[p++], Dv[q], r);
      s = fmaf(Dv[j], r, s);
    }
  }
  const float den = fmaf(k.erho, s, 1.f);
  float inv;  // MUFU reciprocal (~1 ulp): the fp32 stream's budget is 1e-4
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(den));
  const float xt = x - t;
  const float ei = k.erho * inv;
  const float w = ei * xt;
  const float gam = fmaf(w, w, -ei);
  const float e = xt * inv;
  acc[stat_R(D)] += fmaf(e, e, s * inv);
  acc[stat_Q(D)] = fmaf(w, xt, acc[stat_Q(D)]);
#pragma unroll
  for (int j = 0; j < D; ++j) acc[j] = fmaf(w, Dv[j], acc[j]);
  int p = 0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const float gd = gam * Dv[j];
#pragma unroll
    for (int q = j; q < D; ++q, ++p) acc[D + p] = fmaf(gd, Dv[q], acc[D + p]);
  }
  return den;
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
  acc[stat_R(D)] += fma(e, e, s * inv);
  acc[stat_Q(D)] = fma(w, xt, acc[stat_Q(D)]);
#pragma unroll
  for (int j = 0; j < D; ++j) acc[j] = fma(w, Dv[j], acc[j]);
#pragma unroll
  for (int p = 0; p < D * (D + 1) / 2; ++p) acc[D + p] = fma(gam, P[p], acc[D + p]);
  return den;
}

// gene<D>() with the symmetric forms factored by row: s = sum_j D_j (sum_{q>=j} A2_jq D_q)
// (d independent chains instead of one d(d+1)/2-deep chain) and G_jq += (gam D_j) D_q, so
// the d(d+1)/2 products D_j D_q are never held across the 1/den chain (d = 6 on the
// register path: 9 fp64 ops fewer per gene and no spills at 2 CTAs/SM).  Same algebra,
// different rounding order: only the streaming pass at d >= CAVI_ROWFORM_MIN_D uses it
// (the batched kernel keeps gene<D>()).
// Coefficients in registers (RegCoef) or, where registers run out (d >= 7), in a per-warp
// shared-memory copy read per use (SmemCoef: volatile, so the loads are not hoisted back
// into registers; every lane reads the same address, a broadcast).
template <int D>
struct RegCoef {
  const GeneCoef<D>& k;
  __device__ __forceinline__ double c(int j) const { return k.c[j]; }
  __device__ __forceinline__ double a2(int p) const { return k.A2[p]; }
  __device__ __forceinline__ double erho() const { return k.erho; }
};
template <int D>
struct SmemCoef {
  const volatile GeneCoef<D>* k;
  double er;
  __device__ __forceinline__ double c(int j) const { return k->c[j]; }
  __device__ __forceinline__ double a2(int p) const { return k->A2[p]; }
  __device__ __forceinline__ double erho() const { return er; }
};

template <int D, typename CK>
__device__ __forceinline__ double gene_rows(const CK& k, double x, const double (&Dv)[D],
                                            double (&acc)[n_stats(D)]) {
  double t = 0.0, s = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) t = fma(k.c(j), Dv[j], t);
  {
    int p = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double r = 0.0;
#pragma unroll
      for (int q = j; q < D; ++q) r = fma(k.a2(p++), Dv[q], r);
      s = fma(Dv[j], r, s);
    }
  }
  const double erho = k.erho();
  const double den = fma(erho, s, 1.0);
  const double inv = ptx::rcp_nr(den);
  const double xt = x - t;
  const double ei = erho * inv;
  const double w = ei * xt;
  const double gam = fma(w, w, -ei);
  const double e = fma(-s, w, xt);
  acc[stat_R(D)] += fma(e, e, s * inv);
  acc[stat_Q(D)] = fma(w, xt, acc[stat_Q(D)]);
#pragma unroll
  for (int j = 0; j < D; ++j) acc[j] = fma(w, Dv[j], acc[j]);
  int p = 0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const double gd = gam * Dv[j];
#pragma unroll
    for (int q = j; q < D; ++q, ++p) acc[D + p] = fma(gd, Dv[q], acc[D + p]);
  }
  return den;
}

// ---------------------------------------------------------------- deterministic reduction
// Every level sums its children in a fixed order, so the totals are bit-identical
// whichever CTA / warp / GPU computed a chunk.  The level that completes a
// parent (a per-parent arrival counter reaching its child count) computes it;
// nobody waits for anybody.  Warp-level code: lane l handles statistics
// l, l+32, ...

// lane 0 publishes (fence, cumulative over the warp's stores) and counts an arrival
// (one acq_rel atomic: release publishes the warp's stores, which __syncwarp ordered before
// lane 0's; acquire makes every other arriver's stores visible to the last one)
__device__ __forceinline__ bool warp_arrive_last(unsigned int* counter, unsigned int need, int lane) {
  unsigned int last = 0;
  __syncwarp();
  if (lane == 0) {
    unsigned int old;
    // (the release half costs ~3-5% at d = 5..7: the same kernels with a relaxed atomic --
    // not a correct protocol, timing only -- ran N=6 1395 -> 1440, N=7 1125 -> 1179 sweeps/s)
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(counter) : "memory");
    last = old == need - 1;
  }
  return __shfl_sync(0xffffffffu, last, 0) != 0;
}

// The plan's fixed-order row sum -- lane l adds rows l, l+32, ... from 0.0 in index order, then
// a 32-lane xor butterfly (16, 8, 4, 2, 1): one L2 round trip per 32 rows instead of a 16-deep
// dependent chain per stat column -- with the result left in registers: lane l gets stat
// l + 32k in out[k].
template <int NS>
__device__ __forceinline__ void warp_rows(const double* src, int64_t n, double (&out)[(NS + 31) / 32], int lane) {
  constexpr int B = NS < 16 ? NS : 16;
#pragma unroll
  for (int k = 0; k < (NS + 31) / 32; ++k) out[k] = 0.0;
#pragma unroll
  for (int s0 = 0; s0 < NS; s0 += B) {
    double acc[B];
#pragma unroll
    for (int b = 0; b < B; ++b) acc[b] = 0.0;
#pragma unroll 2
    for (int64_t i = lane; i < n; i += 32) {
      const double* row = src + i * NS + s0;
#pragma unroll
      for (int b = 0; b < B; ++b)
        if (s0 + b < NS) acc[b] += __ldcg(row + b);
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      double v = acc[b];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (s0 + b < NS && (s0 + b) % 32 == lane) out[(s0 + b) / 32] = v;
    }
  }
}

// The same cascade with plain partial rows and acquire/release arrivals (the round-1 protocol),
// kept for the compute-bound instantiations (d > CAVI_LL_MAX_D): there the LL version's
// strong loads/stores and row buffers cost more in the consumer loop than the per-chunk release
// fence they save (same-box A/B, V=1e8: N=8 824 vs 639 sweeps/s; N=4 488 vs 511 us the other
// way).  The rows live in the LL buffers, read as doubles.
template <int D, int NS = n_stats(D)>
__device__ __forceinline__ void finish_chunk_acqrel(const PassArgs& a, int64_t chunk, const double* chunk_sum,
                                                    int lane) {
  double* const partials = reinterpret_cast<double*>(a.partials);
  double* const gpartials = reinterpret_cast<double*>(a.gpartials);
  double* const opartials = reinterpret_cast<double*>(a.opartials);
  constexpr int K = (NS + 31) / 32;
  const unsigned long long t_entry = a.cta_trace ? globaltimer_ns() : 0ull;
  for (int st = lane; st < NS; st += 32) partials[chunk * NS + st] = chunk_sum[st];
  const int64_t grp = chunk / a.group_chunks;
  const int64_t c0 = grp * a.group_chunks;
  const int64_t nc = lmin(c0 + a.group_chunks, a.n_chunks) - c0;
  if (!warp_arrive_last(a.gcount + grp, (unsigned int)nc, lane)) return;
  // group complete
  if (lane == 0) a.gcount[grp] = 0u;  // ready for the next sweep
  const int64_t gg = a.group_lo + grp;  // global group index
  const int o = (int)(gg / a.groups_per_octant);
  const int64_t g0 = lmax((int64_t)o * a.groups_per_octant, a.group_lo);
  const int64_t g1 = lmin(lmin((int64_t)(o + 1) * a.groups_per_octant, a.n_groups_total), a.group_lo + a.n_groups);
  double osum[K];
  if (g1 - g0 == 1) {
    // a one-group octant: its sum over one row is the row itself (the butterfly adds zeros),
    // so the group completes the octant directly (small V: one arrival level less)
    warp_rows<NS>(partials + c0 * NS, nc, osum, lane);
  } else {
    warp_rows<NS>(partials + c0 * NS, nc, osum, lane);
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (lane + 32 * k < NS) gpartials[grp * NS + lane + 32 * k] = osum[k];
    if (!warp_arrive_last(a.ocount + o, (unsigned int)(g1 - g0), lane)) return;
    // octant complete
    if (lane == 0) a.ocount[o] = 0u;
    warp_rows<NS>(gpartials + (g0 - a.group_lo) * NS, g1 - g0, osum, lane);
  }
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (lane + 32 * k < NS) opartials[o * NS + lane + 32 * k] = osum[k];
  if (!warp_arrive_last(a.odone, (unsigned int)a.n_live_octants, lane)) return;
  // every octant this shard owns is complete: pairwise tree over them (empty octants add 0);
  // this warp's own octant from registers, the others' loads all in flight together
  if (lane == 0) *a.odone = 0u;
  if (a.cta_trace && lane == 0) {
    a.cta_trace[blockIdx.x * 8 + 4] = t_entry;
    a.cta_trace[blockIdx.x * 8 + 5] = globaltimer_ns();
  }
  double tot[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int st = lane + 32 * k;
    double v[kOctants];
#pragma unroll
    for (int q = 0; q < kOctants; ++q) {
      const int64_t h0 = lmax((int64_t)q * a.groups_per_octant, a.group_lo);
      const int64_t h1 = lmin(lmin((int64_t)(q + 1) * a.groups_per_octant, a.n_groups_total), a.group_lo + a.n_groups);
      const bool live = st < NS && q >= a.oct_lo && q < a.oct_hi && h1 > h0;
      v[q] = q == o ? osum[k] : (live ? __ldcg(opartials + q * NS + st) : 0.0);
    }
#pragma unroll
    for (int w = 1; w < kOctants; w *= 2)
#pragma unroll
      for (int q = 0; q + w < kOctants; q += 2 * w)
        if (q >= a.oct_lo && q + w < a.oct_hi && ((q - a.oct_lo) % (2 * w)) == 0) v[q] = v[q] + v[q + w];
    tot[k] = 0.0;
#pragma unroll
    for (int q = 0; q < kOctants; ++q)
      if (q == a.oct_lo) tot[k] = v[q];
  }
  if (a.lsa.win) {  // fused exchange: straight into every peer's window over NVLink
    const uint64_t sq = *a.lsa.seq + 1;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (lane + 32 * k < NS) lsa_publish_stat(a.lsa, sq, lane + 32 * k, tot[k]);
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (lane + 32 * k < NS) a.rank_out[lane + 32 * k] = tot[k];
  }
  if (lane == 0) *a.pass_seq += 1u;  // keep the LL tag in step (unused on this path)
  if (a.cta_trace && lane == 0) a.cta_trace[blockIdx.x * 8 + 6] = globaltimer_ns();
}

// ---- flag-in-data ("LL") rows of the reduction: a double travels as two 8-byte words
// (pass tag << 32 | 32 data bits), each single-copy atomic, so a reader that sees both tags
// equal to the running pass's tag has the value.  Arrivals are then counted with RELAXED
// atomics: the last arriver of a level knows every sibling stored its row before arriving (in
// program order) and polls the rows until their tags match -- a store-visibility wait, never
// a wait on another warp's progress.  A release/acquire arrival instead pays the stores'
// acknowledgement before the atomic: one L2 round trip more per level, three levels at the
// end of every pass.
__device__ __forceinline__ void ll_put(uint64_t* p, double v, uint32_t tag) {
  const uint64_t u = (uint64_t)__double_as_longlong(v), t = (uint64_t)tag << 32;
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(t | (u & 0xffffffffull)), "l"(t | (u >> 32))
               : "memory");
}
__device__ __forceinline__ void ll_get2(const uint64_t* p, uint64_t& a, uint64_t& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ double ll_val(uint64_t a, uint64_t b) {
  return __longlong_as_double((long long)((b << 32) | (a & 0xffffffffull)));
}
__device__ __forceinline__ bool ll_ok(uint64_t a, uint64_t b, uint32_t tag) {
  return (uint32_t)(a >> 32) == tag && (uint32_t)(b >> 32) == tag;
}
// polls are bounded (a protocol bug traps instead of hanging the GPU); no function calls in
// the pass kernel (an ABI call makes the compiler spill the consumer loop's live registers)
__device__ __forceinline__ void ll_check_deadline(unsigned long long t0) {
  if (globaltimer_ns() - t0 > 4000000000ull) __trap();
}

// relaxed arrival: true on the warp whose arrival completes `need`
__device__ __forceinline__ bool warp_arrive_last_relaxed(unsigned int* counter, unsigned int need, int lane) {
  unsigned int last = 0;
  __syncwarp();
  if (lane == 0) {
    unsigned int old;
    asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(counter) : "memory");
    last = old == need - 1;
  }
  return __shfl_sync(0xffffffffu, last, 0) != 0;
}

// The plan's fixed-order row sum (as warp_rows) over n LL rows of NS values, polled until
// tagged `tag`; the result stays in registers: lane l gets stat l + 32k in out[k].
template <int NS>
__device__ __forceinline__ void warp_rows_ll(const uint64_t* rows, int64_t n, uint32_t tag,
                                             double (&out)[(NS + 31) / 32], int lane) {
  // stats per pass: small enough that the row words fit beside the consumer loop's live
  // registers (this is inlined into it: a larger batch spills the loop state)
  constexpr int B = NS < ll_batch(NS) ? NS : ll_batch(NS);
#pragma unroll
  for (int k = 0; k < (NS + 31) / 32; ++k) out[k] = 0.0;
#pragma unroll
  for (int s0 = 0; s0 < NS; s0 += B) {
    double acc[B];
#pragma unroll
    for (int b = 0; b < B; ++b) acc[b] = 0.0;
#pragma unroll 1
    for (int64_t i = lane; i < n; i += 32) {
      const uint64_t* row = rows + (i * NS + s0) * 2;
      uint64_t wa[B], wb[B];
      unsigned long long t0 = 0;
#pragma unroll 1
      for (int tries = 0;; ++tries) {  // normally one pass: the siblings stored before arriving
        bool ok = true;
#pragma unroll
        for (int b = 0; b < B; ++b)
          if (s0 + b < NS) ll_get2(row + 2 * b, wa[b], wb[b]);
#pragma unroll
        for (int b = 0; b < B; ++b)
          if (s0 + b < NS) ok = ok && ll_ok(wa[b], wb[b], tag);
        if (ok) break;
        if (tries == 0) t0 = globaltimer_ns();
        ll_check_deadline(t0);
      }
#pragma unroll
      for (int b = 0; b < B; ++b)
        if (s0 + b < NS) acc[b] += ll_val(wa[b], wb[b]);
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      double v = acc[b];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (s0 + b < NS && (s0 + b) % 32 == lane) out[(s0 + b) / 32] = v;
    }
  }
}

template <int NS>
__device__ __forceinline__ void ll_put_row(uint64_t* row, const double (&v)[(NS + 31) / 32], uint32_t tag, int lane) {
#pragma unroll
  for (int k = 0; k < (NS + 31) / 32; ++k)
    if (lane + 32 * k < NS) ll_put(row + 2 * (lane + 32 * k), v[k], tag);
}

// chunk partial -> group -> octant -> total (-> tail), by whichever warp completes each level
// (relaxed arrival counters + LL rows: nobody waits for anybody's progress).  The final level
// keeps its own octant in registers and loads the others all at once.
template <int D, int NS = n_stats(D)>
__device__ __forceinline__ void finish_chunk_ll(const PassArgs& a, int64_t chunk, const double* chunk_sum,
                                                uint32_t tag, int lane) {
  constexpr int K = (NS + 31) / 32;
  const unsigned long long t_entry = a.cta_trace ? globaltimer_ns() : 0ull;
  for (int st = lane; st < NS; st += 32) ll_put(a.partials + (chunk * NS + st) * 2, chunk_sum[st], tag);
  const int64_t grp = chunk / a.group_chunks;
  const int64_t c0 = grp * a.group_chunks;
  const int64_t nc = lmin(c0 + a.group_chunks, a.n_chunks) - c0;
  if (!warp_arrive_last_relaxed(a.gcount + grp, (unsigned int)nc, lane)) return;
  // group complete
  if (lane == 0) a.gcount[grp] = 0u;  // ready for the next sweep
  const int64_t gg = a.group_lo + grp;  // global group index
  const int o = (int)(gg / a.groups_per_octant);
  const int64_t g0 = lmax((int64_t)o * a.groups_per_octant, a.group_lo);
  const int64_t g1 = lmin(lmin((int64_t)(o + 1) * a.groups_per_octant, a.n_groups_total), a.group_lo + a.n_groups);
  double osum[K];
  warp_rows_ll<NS>(a.partials + c0 * NS * 2, nc, tag, osum, lane);
  if (g1 - g0 > 1) {
    // (a one-group octant: its sum over one row is the row itself -- the butterfly adds
    // zeros -- so the group completes the octant directly, one arrival level less)
    ll_put_row<NS>(a.gpartials + grp * NS * 2, osum, tag, lane);
    if (!warp_arrive_last_relaxed(a.ocount + o, (unsigned int)(g1 - g0), lane)) return;
    // octant complete
    if (lane == 0) a.ocount[o] = 0u;
    warp_rows_ll<NS>(a.gpartials + (g0 - a.group_lo) * NS * 2, g1 - g0, tag, osum, lane);
  }
  // No arrival level for the shard total: the warp that completes the shard's LAST octant
  // builds it, polling the other octants' rows.  It can only wait on octants whose chunks sit
  // in other CTAs' pipelines (it completed the last octant, so this CTA's chunks -- dispatched in
  // increasing order -- are all done): no chain of waits; in practice the lower octants were
  // complete long before and the poll is one round trip.
  if (o != a.oct_last) {
    ll_put_row<NS>(a.opartials + o * NS * 2, osum, tag, lane);
    return;
  }
  if (a.cta_trace && lane == 0) {
    a.cta_trace[blockIdx.x * 8 + 4] = t_entry;
    a.cta_trace[blockIdx.x * 8 + 5] = globaltimer_ns();
  }
  double tot[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int st = lane + 32 * k;
    double v[kOctants];
    uint64_t wa[kOctants], wb[kOctants];
    bool live[kOctants];
#pragma unroll
    for (int q = 0; q < kOctants; ++q) {
      const int64_t h0 = lmax((int64_t)q * a.groups_per_octant, a.group_lo);
      const int64_t h1 = lmin(lmin((int64_t)(q + 1) * a.groups_per_octant, a.n_groups_total), a.group_lo + a.n_groups);
      live[q] = st < NS && q != o && q >= a.oct_lo && q < a.oct_hi && h1 > h0;
    }
    unsigned long long t0 = 0;
#pragma unroll 1
    for (int tries = 0;; ++tries) {
      bool ok = true;
#pragma unroll
      for (int q = 0; q < kOctants; ++q)
        if (live[q]) ll_get2(a.opartials + (q * NS + st) * 2, wa[q], wb[q]);
#pragma unroll
      for (int q = 0; q < kOctants; ++q)
        if (live[q]) ok = ok && ll_ok(wa[q], wb[q], tag);
      if (ok) break;
      if (tries == 0) t0 = globaltimer_ns();
      ll_check_deadline(t0);
    }
#pragma unroll
    for (int q = 0; q < kOctants; ++q) v[q] = q == o ? osum[k] : (live[q] ? ll_val(wa[q], wb[q]) : 0.0);
#pragma unroll
    for (int w = 1; w < kOctants; w *= 2)
#pragma unroll
      for (int q = 0; q + w < kOctants; q += 2 * w)
        if (q >= a.oct_lo && q + w < a.oct_hi && ((q - a.oct_lo) % (2 * w)) == 0) v[q] = v[q] + v[q + w];
    tot[k] = 0.0;
#pragma unroll
    for (int q = 0; q < kOctants; ++q)
      if (q == a.oct_lo) tot[k] = v[q];
  }
  if (a.lsa.win) {  // fused exchange: straight into every peer's window over NVLink
    const uint64_t sq = *a.lsa.seq + 1;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (lane + 32 * k < NS) lsa_publish_stat(a.lsa, sq, lane + 32 * k, tot[k]);
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (lane + 32 * k < NS) a.rank_out[lane + 32 * k] = tot[k];
  }
  if (lane == 0) *a.pass_seq = tag + 1u;  // the next pass's tag (read after this grid completes)
  if (a.cta_trace && lane == 0) a.cta_trace[blockIdx.x * 8 + 6] = globaltimer_ns();
}

template <int D>
__device__ __forceinline__ void finish_chunk(const PassArgs& a, int64_t chunk, const double* chunk_sum, uint32_t tag,
                                          int lane) {
  if constexpr (D <= CAVI_LL_MAX_D)
    finish_chunk_ll<D>(a, chunk, chunk_sum, tag, lane);
  else
    finish_chunk_acqrel<D>(a, chunk, chunk_sum, lane);
}

// The sweep tail as its own one-warp kernel (tail.cuh): pairwise tree over the `world` shard
// totals (1 on a single GPU; the NCCL-gathered rank partials or the fused exchange's window
// otherwise), then the warp-parallel tail.
template <int D>
__global__ void __launch_bounds__(32, 1) tail_kernel(const Hyp* __restrict__ h, Ctl* c, const double* parts, int world,
                                                     LsaLink lsa) {
  constexpr int NS = n_stats(D);
  __shared__ TailSm<D> sm;
  ptx::griddep_launch_dependents();  // the next pass may launch and stage its prologue
  TailHyp<D> th;                     // constant through the fit: loaded while the pass streams
  th.load(h, threadIdx.x);
  ptx::griddep_wait();               // the pass (or exchange) that produced `parts` is complete
  if (threadIdx.x == 0) TAIL_PROF(*c, 0);
  const unsigned long long t_entry = globaltimer_ns();  // diagnostics (stored at exit: no load on the critical path)
  if (lsa.win) {  // fused exchange: every rank's partial arrives in this rank's window
    if (*(volatile const int*)&c->done) return;  // no rank published this sweep
    const uint64_t s = *lsa.seq + 1;
    const unsigned long long deadline = lsa_now_ns() + lsa.timeout_ns;  // a stalled peer -> error, not a hang
    bool ok = true;
    for (int st = threadIdx.x; st < NS; st += 32) {
      double v[kOctants];
#pragma unroll
      for (int r = 0; r < kOctants; ++r)
        if (r < world) v[r] = lsa_take(lsa, s, r, st, deadline, &ok);
#pragma unroll
      for (int w = 1; w < kOctants; w *= 2)
#pragma unroll
        for (int r = 0; r + w < kOctants; r += 2 * w)
          if (w < world && r + w < world) v[r] = v[r] + v[r + w];
      sm.tot[st] = v[0];
    }
    if (!__all_sync(0xffffffffu, ok)) {
      if (threadIdx.x == 0) {
        c->status = CV_ERR_PEER;
        c->done = 1;
      }
      return;
    }
    __syncwarp();
    if (threadIdx.x == 0) *lsa.seq = s;
    parts = nullptr;  // sm.tot is complete
  }
  tail_warp<D>(th, c, parts, world, sm, threadIdx.x);
  if (threadIdx.x == 0) {
    unsigned long long* tl = c->tl_trace;
    if (tl) {
      const unsigned long long t_exit = globaltimer_ns();
      const int n = c->tl_n;
      tl[2 * n] = t_entry;
      tl[2 * n + 1] = t_exit;
      c->tl_n = n + 1;
    }
  }
}

typedef void (*TailFn)(const Hyp*, Ctl*, const double*, int, LsaLink);

// ------------------------------------------------- d >= CAVI_MMA_MIN_D: fp64 tensor cores
// mma.sync.m8n8k4.f64 (DMMA; tcgen05 has no fp64 kind).  Per warp and 8 genes:
//   Y = D_8xd L,  A^-1 = L L^T    (s_i = |Y_i|^2; t_i = c . D_i; see MmaConsumer)
//   G += (D o gamma)^T D          (2 k-steps of 4 genes; upper tiles only)
// Fragments (PTX m8n8k4 .f64): A[r=lane/4][q=lane%4], B[q][r], C[r][2q+i].  L lives in B
// fragments (<= 8 doubles/lane), the d x d accumulator in C fragments (<= 6 doubles/lane), so
// d = 15 fits in registers; padding columns (>= d) are zero.
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

#ifndef CAVI_TINY_BLOCKS
#define CAVI_TINY_BLOCKS 4  // CTAs per SM at d = 1 (~90 registers; N=2: 3450 -> 3960 sweeps/s)
#endif
#ifndef CAVI_D2_BLOCKS
#define CAVI_D2_BLOCKS 3  // CTAs per SM at d = 2 (118 registers; N=3: 2536 -> 2829 sweeps/s)
#endif
#ifndef CAVI_D4_BLOCKS
#define CAVI_D4_BLOCKS 2  // CTAs per SM at d = 4: 2 + the reducer warp (N=5 1713 -> 1751 sweeps/s) over 3 without
#endif
#ifndef CAVI_TILE_MID
#define CAVI_TILE_MID 512  // genes per stage of the register path at d = 4, 5
#endif
#ifndef CAVI_SEMI_Y_MAXD
#define CAVI_SEMI_Y_MAXD 13  // d > CAVI_HYBRID_MAX_D: trailing Y columns in scalar up to this d (14, 15 spill)
#endif
#ifndef CAVI_SEMI_MAX_D
#define CAVI_SEMI_MAX_D 14  // above: every G tile on the tensor cores, no per-lane trailing accumulators (N=16: 276 -> 285 sweeps/s; N=13-15 slower)
#endif
#ifndef CAVI_HYBRID_MAX_D
#define CAVI_HYBRID_MAX_D 11  // largest d with the scalar trailing block (d = 12 spills: slower)
#endif
#ifndef CAVI_MMA_UNROLL
#define CAVI_MMA_UNROLL 8
#endif
constexpr int kMmaUnroll = CAVI_MMA_UNROLL;  // independent 8-gene groups in flight per warp
constexpr int kMmaBatchUnroll = kMmaUnroll / 4;  // 4-group batches

template <int D>
struct MmaConsumer {
  static constexpr int DP = D <= 8 ? 8 : 16;  // padded dimension
  // 9 <= d <= CAVI_HYBRID_MAX_D: only the 8x8 leading tiles run on the tensor cores; the
  // RX = d - 8 trailing dimensions (their Y columns and G rows/columns) are cheaper as
  // per-gene scalar FMAs than as mostly-empty 8x8 tiles
  static constexpr int RX = (D > 8 && D <= CAVI_HYBRID_MAX_D) ? D - 8 : 0;
  static constexpr bool kHyb = RX > 0;
  static constexpr int NT = kHyb ? 1 : DP / 8;  // 8-wide output tiles on the tensor cores
  // d > CAVI_HYBRID_MAX_D: Y and the G tiles of rows < 8 on the tensor cores, the trailing
  // diagonal block of G (and g) as per-gene scalar FMAs instead of the 8x8 tile (1, 1)
  static constexpr bool kSemi = D > 8 && !kHyb && D <= CAVI_SEMI_MAX_D;
  static constexpr int RT = (kHyb || kSemi) ? D - 8 : 0;  // trailing dimensions done in scalar
  static constexpr int MTG = kSemi ? 1 : NT;              // G row tiles on the tensor cores
  // d > CAVI_HYBRID_MAX_D too: the trailing Y columns (k >= 8) as per-gene scalar FMAs with
  // the trailing block of L in registers, instead of the Y tiles of column block 1
  static constexpr bool kSemiY = kSemi && D <= CAVI_SEMI_Y_MAXD;
  static constexpr int RY = (kHyb || kSemiY) ? D - 8 : 0;  // trailing Y columns done in scalar
  static constexpr int NTU = RY > 0 ? 1 : NT;               // Y tiles on the tensor cores
  static constexpr int KS = (D + 3) / 4;      // k-steps of Y = D L (rows >= D are zero)
  static constexpr int NS = n_stats(D);
  // s = D^T A^-1 D = |L^T D|^2 with A^-1 = L L^T: Y = D L is block lower-triangular, so the
  // (ks, nt) blocks with 4 ks + 3 < 8 nt vanish.  When d < 8 the free column d of the B
  // operand carries c, so Y[:, d] = t = D^T c comes out of the same MMAs.
  static constexpr int kTcol = D < 8 ? D : -1;
  static constexpr bool live(int ks, int nt) { return 4 * ks + 3 >= 8 * nt || (kTcol >= 0 && nt == 0); }
  double bfr[NT][KS];   // [L | c][ks*4 + q][nt*8 + r]
  double cc[NT][2];     // c[nt*8 + 2q + i]
  double erho;
  double gacc[NT][NT][2];
  double gv[NT];
  double R, Q;
  LogAcc lg;
  // hybrid extras (RX > 0): trailing block of L, c; per-lane accumulators of the trailing
  // G columns (ge: rows < 8, gl: rows >= 8, packed upper) and of g
  static constexpr int RXa = RX > 0 ? RX : 1, RTa = RT > 0 ? RT : 1, RYa = RY > 0 ? RY : 1;
  double lx[RYa * (RYa + 1) / 2], cx[RYa];
  double ge[8][RXa], gl[RTa * (RTa + 1) / 2], gx[RTa];

  // L = chol(A^-1), warp-cooperative: lane i holds row i (right-looking, one column per
  // step); then the B fragments are gathered from the row owners.  Runs once per pass,
  // overlapped with the producer's first TMA loads.
  __device__ __forceinline__ void load(const Gen& g, int lane) {
    const int r = lane >> 2, q = lane & 3;
    double a[D], l[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      a[j] = lane < D ? g.Ainv[lane * D + j] : 0.0;
      l[j] = 0.0;
    }
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const double piv = __shfl_sync(0xffffffffu, a[k], k);
      const double lkk = sqrt(fmax(piv, 0.0));
      const double lik = lane == k ? lkk : (lane > k && lane < D ? a[k] / lkk : 0.0);
      l[k] = lik;
#pragma unroll
      for (int j = k + 1; j < D; ++j) {
        const double ljk = __shfl_sync(0xffffffffu, lik, j);
        a[j] = fma(-lik, ljk, a[j]);
      }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int row = ks * 4 + q, col = nt * 8 + r;
        double v = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const double x = __shfl_sync(0xffffffffu, l[c], row < D ? row : 0);
          if (c == col) v = x;
        }
        if (col == kTcol) v = g.c[row < D ? row : 0];
        bfr[nt][ks] = row < D ? v : 0.0;
      }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int col = nt * 8 + 2 * q + i;
        cc[nt][i] = col < D ? g.c[col] : 0.0;
      }
    if constexpr (RY > 0) {
#pragma unroll
      for (int k = 0; k < RY; ++k) {
        cx[k] = g.c[8 + k];
#pragma unroll
        for (int j = k; j < RY; ++j) lx[j * (j + 1) / 2 + k] = __shfl_sync(0xffffffffu, l[8 + k], 8 + j);
      }
    }
    erho = g.e_rho;
  }

  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int mt = 0; mt < NT; ++mt) {
      gv[mt] = 0.0;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) gacc[mt][nt][0] = gacc[mt][nt][1] = 0.0;
    }
    R = 0.0;
    Q = 0.0;
    lg.init();
#pragma unroll
    for (int k = 0; k < RT; ++k) gx[k] = 0.0;
#pragma unroll
    for (int i = 0; i < RT * (RT + 1) / 2; ++i) gl[i] = 0.0;
    if constexpr (kHyb) {
#pragma unroll
      for (int k = 0; k < RX; ++k)
#pragma unroll
        for (int j = 0; j < 8; ++j) ge[j][k] = 0.0;
    }
  }

  // genes [gbase, gbase + 8*ngroups) of a stage (x column, then D columns at stride CS),
  // in batches of 4 groups (32 genes).  Per batch:
  //  1. Y = D L per group on the tensor cores (and t = D^T c, see kTcol);
  //  2. s = sum_k Y_k^2: lane (r, q) holds a partial over its columns; a 4-lane
  //     reduce-scatter leaves lane (r, q) with the full s, t of gene r of group q, so the
  //     per-gene scalar chain (den, 1/den, w, gamma, residual) runs once per gene;
  //  3. G += (D o gamma)^T D on the tensor cores (upper tiles), g += w D.
  template <typename T, int CS>
  __device__ __forceinline__ void tile(const T* st, int gbase, int ngroups, int lane) {
    // branch-free: padding columns (>= D) of the stage are zero, as are the padded fragments
    const int r = lane >> 2, q = lane & 3;
    const int hi = q >> 1, lo = q & 1;
    const T* Dc = st + CS;  // column j at Dc + j*CS
#pragma unroll kMmaBatchUnroll
    for (int b = 0; b < ngroups; b += 4) {
      const int gb = gbase + b * 8;
      double sp[4], tp[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const int g0 = gb + g * 8;
        double u[NTU][2];
#pragma unroll
        for (int nt = 0; nt < NTU; ++nt) u[nt][0] = u[nt][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const double av = (double)Dc[(ks * 4 + q) * CS + g0 + r];
#pragma unroll
          for (int nt = 0; nt < NTU; ++nt)
            if (live(ks, nt)) dmma(u[nt], av, bfr[nt][ks]);
        }
        double s_ = 0.0, t_ = 0.0;
#pragma unroll
        for (int nt = 0; nt < NTU; ++nt)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int col = nt * 8 + 2 * q + i;
            if constexpr (kTcol >= 0) {
              const double y = col == kTcol ? 0.0 : u[nt][i];
              s_ = fma(y, y, s_);
              t_ += col == kTcol ? u[nt][i] : 0.0;
            } else {
              s_ = fma(u[nt][i], u[nt][i], s_);
              t_ = fma(cc[nt][i], (double)Dc[col * CS + g0 + r], t_);  // D is zero for col >= D
            }
          }
        sp[g] = s_;
        tp[g] = t_;
      }
      // reduce-scatter over the 4 lanes of row r: lane q keeps group q
      double s2[2], t2[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double ks_ = hi ? sp[k + 2] : sp[k], kt_ = hi ? tp[k + 2] : tp[k];
        const double ss_ = hi ? sp[k] : sp[k + 2], st_ = hi ? tp[k] : tp[k + 2];
        s2[k] = ks_ + __shfl_xor_sync(0xffffffffu, ss_, 2);
        t2[k] = kt_ + __shfl_xor_sync(0xffffffffu, st_, 2);
      }
      const double sv0 = (lo ? s2[1] : s2[0]) + __shfl_xor_sync(0xffffffffu, lo ? s2[0] : s2[1], 1);
      const double tv0 = (lo ? t2[1] : t2[0]) + __shfl_xor_sync(0xffffffffu, lo ? t2[0] : t2[1], 1);
      // per-gene scalars: lane (r, q) owns gene gb + 8q + r
      const int own = gb + 8 * q + r;
      const double x = (double)st[own];
      double sv = sv0, tv = tv0;
      double dx[RT > 0 ? D : 1];
      if constexpr (RT > 0) {
#pragma unroll
        for (int j = kHyb ? 0 : 8; j < D; ++j) dx[j] = (double)Dc[j * CS + own];
      }
      if constexpr (RY > 0) {  // trailing Y columns and t terms of the own gene
#pragma unroll
        for (int k = 0; k < RY; ++k) {
          double y = 0.0;
#pragma unroll
          for (int j = k; j < RY; ++j) y = fma(dx[8 + j], lx[j * (j + 1) / 2 + k], y);
          sv = fma(y, y, sv);
          tv = fma(cx[k], dx[8 + k], tv);
        }
      }
      const double den = fma(erho, sv, 1.0);
      const double inv = ptx::rcp_nr(den);
      const double xt = x - tv;
      const double ei = erho * inv;
      const double w = ei * xt;
      const double gam = fma(w, w, -ei);
      const double e = fma(-sv, w, xt);
      R += fma(e, e, sv * inv);
      Q += w * xt;
      lg.mul(den);
      if constexpr (RT > 0) {  // trailing G block (and g entries) of the own gene
#pragma unroll
        for (int k = 0; k < RT; ++k) {
          const double dk = dx[8 + k];
          gx[k] = fma(w, dk, gx[k]);
          const double gd = gam * dk;
          if constexpr (kHyb) {
#pragma unroll
            for (int j = 0; j < 8; ++j) ge[j][k] = fma(gd, dx[j], ge[j][k]);
          }
#pragma unroll
          for (int j = 0; j <= k; ++j) gl[k * (k + 1) / 2 + j] = fma(gd, dx[8 + j], gl[k * (k + 1) / 2 + j]);
        }
      }
      // G += (D o gamma)^T D, g += w D per group: 2 k-steps of 4 genes
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const int g0 = gb + g * 8;
#pragma unroll
        for (int ks2 = 0; ks2 < 2; ++ks2) {
          const int src = (ks2 * 4 + q) * 4 + g;  // the lane owning gene g0 + 4 ks2 + q
          const double gk = __shfl_sync(0xffffffffu, gam, src);
          const double wk = __shfl_sync(0xffffffffu, w, src);
          double dv[NT];
#pragma unroll
          for (int bb = 0; bb < NT; ++bb) dv[bb] = (double)Dc[(bb * 8 + r) * CS + g0 + ks2 * 4 + q];
#pragma unroll
          for (int mt = 0; mt < MTG; ++mt) {
            const double av = gk * dv[mt];
            gv[mt] = fma(wk, dv[mt], gv[mt]);
#pragma unroll
            for (int nt = mt; nt < NT; ++nt) dmma(gacc[mt][nt], av, dv[nt]);
          }
        }
      }
    }
  }

  // this warp's statistic vector [g | G upper | R | Ld] -> out[NS]
  __device__ __forceinline__ void publish(double* out, int lane) {
    const int r = lane >> 2, q = lane & 3;
#pragma unroll
    for (int mt = 0; mt < MTG; ++mt) {
      double v = gv[mt];
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      const int j = mt * 8 + r;
      if (q == 0 && j < D) out[j] = v;
    }
#pragma unroll
    for (int mt = 0; mt < MTG; ++mt)
#pragma unroll
      for (int nt = mt; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int j = mt * 8 + r, kk = nt * 8 + 2 * q + i;
          if (j < D && kk < D && kk >= j) out[D + j * D - j * (j - 1) / 2 + (kk - j)] = gacc[mt][nt][i];
        }
    if constexpr (RT > 0) {
      auto wsum = [](double v) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        return v;
      };
#pragma unroll
      for (int k = 0; k < RT; ++k) {
        const int kk = 8 + k;
        const double gs = wsum(gx[k]);
        if (lane == 0) out[kk] = gs;
#pragma unroll
        for (int j = 0; j < (kHyb ? 8 : 0); ++j) {
          const double v = wsum(ge[j][k < RX ? k : 0]);
          if (lane == 0) out[D + j * D - j * (j - 1) / 2 + (kk - j)] = v;
        }
#pragma unroll
        for (int j = 0; j <= k; ++j) {
          const int jj = 8 + j;
          const double v = wsum(gl[k * (k + 1) / 2 + j]);
          if (lane == 0) out[D + jj * D - jj * (jj - 1) / 2 + (kk - jj)] = v;
        }
      }
    }
    double rv = R, qv = Q, lv = lg.log_value();
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      rv += __shfl_xor_sync(0xffffffffu, rv, off);
      qv += __shfl_xor_sync(0xffffffffu, qv, off);
      lv += __shfl_xor_sync(0xffffffffu, lv, off);
    }
    if (lane == 0) {
      out[stat_R(D)] = rv;
      out[stat_Q(D)] = qv;
      out[stat_Ld(D)] = lv;
    }
  }
};

// ---------------------------------------------------------------- pipeline geometry
constexpr int kSlots = 4;  // chunk-reduction slots (warps drift < kStages tiles < kSlots chunks)

// Geometry measured on B200 (V=1e8, d=3, fp64): 2 CTAs/SM x (4 consumer warps + 1 TMA
// producer warp), 8 genes per consumer thread per 1024-gene stage, 3 stages of 32 KB per
// CTA -> 0.489 ms/pass = 100% of the measured copy bandwidth.  (1 CTA x 8 warps x 4
// genes/thread: 0.593 ms; 16 warps x 2 genes: 0.66 ms -- ILP per thread and two
// independent pipelines per SM are what hides the fp64 latency chains.)
#ifndef CAVI_ROWFORM_MIN_D
#define CAVI_ROWFORM_MIN_D 4  // register path: gene_rows<D>() from this d up (N=5: 1524 -> 1570, N=6: 1245 -> 1340)
#endif
#ifndef CAVI_SMEM_COEF_MIN_D
#define CAVI_SMEM_COEF_MIN_D 7  // register path: A^-1, c read from shared memory from this d up
#endif
#ifndef CAVI_CONS
#define CAVI_CONS 128  // consumer threads per CTA (4 warps)
#endif
#ifndef CAVI_TILE_SMALL_D
#define CAVI_TILE_SMALL_D 1024  // genes per stage for d <= 3
#endif
#ifndef CAVI_TILE_TINY_D
#define CAVI_TILE_TINY_D 1024  // genes per stage for d = 1
#endif
#ifndef CAVI_SMEM_BUDGET
#define CAVI_SMEM_BUDGET 100000
#endif
#ifndef CAVI_F32_BLOCKS
#define CAVI_F32_BLOCKS 3  // CTAs per SM on the fp32 stream, fp64 math (V=1e8 N=4: 2 -> 3: 2178 -> 2475 sweeps/s)
#endif
#ifndef CAVI_F32_D3_BLOCKS
#define CAVI_F32_D3_BLOCKS 2  // ... at d = 3: 2 + the reducer warp (2678 -> 2930 sweeps/s); d = 1, 2 lose at 2 (4710 -> 3840)
#endif
#ifndef CAVI_F32M_BLOCKS
#define CAVI_F32M_BLOCKS 3  // ... and with fp32 math (2 -> 4: 2272 -> 3034 sweeps/s; + 16-byte loads, MUFU rcp: 3546 at 4, 3542 at 3)
#endif
#ifndef CAVI_F32_BLOCKS_MAXD
#define CAVI_F32_BLOCKS_MAXD 3
#endif
#ifndef CAVI_L2_PREFETCH_CHUNKS
#define CAVI_L2_PREFETCH_CHUNKS 0  // chunks per CTA pulled into L2 before griddepcontrol.wait (A/B: 0 best, tools/l2_prefetch_ab.sh)
#endif
#ifndef CAVI_MIN_BLOCKS
#define CAVI_MIN_BLOCKS 2  // CTAs per SM
#endif

#ifndef CAVI_REDUCER_WARP
#define CAVI_REDUCER_WARP 1
#endif
#ifndef CAVI_REDUCER_MIN_D
#define CAVI_REDUCER_MIN_D 3
#endif
#ifndef CAVI_REDUCER_MMA_MAXD
#define CAVI_REDUCER_MMA_MAXD 14  // DMMA path at 2 CTAs/SM (d >= 10): N=11 461 -> 481, N=15 299 -> 307; d = 15 -0.3%
#endif

#ifndef CAVI_MMA_MIN_D
#define CAVI_MMA_MIN_D 8  // smallest d served by the DMMA consumer (V=1e8 sweeps/s, register vs DMMA:
                          // d=6 1038 vs 695, d=7 771 vs 677, d=8 565 vs 646)
#endif
#ifndef CAVI_MMA_SMALL_MAXD
#define CAVI_MMA_SMALL_MAXD 9  // largest d run at CAVI_MMA_SMALL_BLOCKS CTAs/SM (d=10,11 spill at 3)
#endif
#ifndef CAVI_MMA_SMALL_BLOCKS
#define CAVI_MMA_SMALL_BLOCKS 3  // CTAs per SM for the DMMA consumer at d <= 8
#endif
#ifndef CAVI_MMA_CONS
#define CAVI_MMA_CONS 128  // consumer threads per CTA on the DMMA path
#endif

template <int D, typename T, typename M = double>
struct Geometry {
  static constexpr bool kMma = D >= CAVI_MMA_MIN_D;
  static constexpr int kCons = kMma ? CAVI_MMA_CONS : CAVI_CONS;
  static constexpr int kCWarps = kCons / 32;
  static constexpr int kProducerWarp = kCWarps;
  static constexpr int kReducerWarp = kCWarps + 1;
  // small d: per-thread register kernel; larger d: fp64 tensor-core (DMMA) consumer
  static constexpr bool kSmallBlocks = kMma && D <= CAVI_MMA_SMALL_MAXD;
  // genes per stage; 3 CTAs/SM of the 16-column DMMA stages need half-size tiles
  static constexpr int kTile = D <= 1 ? CAVI_TILE_TINY_D
                               : D <= 3 ? CAVI_TILE_SMALL_D
                               : kMma ? ((kSmallBlocks && D > 8) ? 128 : 256) : CAVI_TILE_MID;
  static constexpr int kTilesPerChunk = kChunk / kTile;  // in the smallest chunk (a.chunk_genes / kTile at run time)
  static constexpr int kGenesPerThread = kTile / kCons;  // consumer genes per stage
  static constexpr uint32_t kColBytes = kTile * sizeof(T);
  // smem column stride (elements): +4 doubles for the DMMA fragment loads -> conflict-free banks
  static constexpr int kColStride = kMma ? kTile + (int)(32 / sizeof(T)) : kTile;
  // DMMA path: the stage holds the padded width (8 or 16 columns); columns >= D stay zero
  static constexpr int kCols = kMma ? (D <= 8 ? 8 : 16) : D;
  static constexpr uint32_t kStageBytes = (uint32_t)kColStride * sizeof(T) * (1 + kCols);
  static constexpr uint32_t kTxBytes = kColBytes * (1 + D);  // bytes the TMA copies deliver per stage
  static constexpr int kNS = n_stats(D);
  static constexpr int kSlotBytes = kSlots * kCWarps * kNS * 8;
  // the DMMA kernels at d <= 8 (~110 registers) are latency-bound at 2 CTAs/SM: run 3
  static constexpr int kMinBlocks = kSmallBlocks ? CAVI_MMA_SMALL_BLOCKS
                                   : (sizeof(T) == 4 && sizeof(M) == 4 && D <= CAVI_F32_BLOCKS_MAXD) ? CAVI_F32M_BLOCKS
                                   : (sizeof(T) == 4 && D <= CAVI_F32_BLOCKS_MAXD) ? (D >= 3 ? CAVI_F32_D3_BLOCKS : CAVI_F32_BLOCKS)
                                   : D <= 1     ? CAVI_TINY_BLOCKS
                                   : D == 2     ? CAVI_D2_BLOCKS
                                   : D == 4     ? CAVI_D4_BLOCKS
                                                : CAVI_MIN_BLOCKS;
  // A reducer warp takes each chunk's slot sum and the reduction cascade off the consumers
  // (the finishing consumer's cascade work -- at d >= 5 the acquire/release arrival's fence --
  // stalled it and, through the shared stage ring, the whole CTA).  Where the 32 extra threads
  // fit the register budget: 2 CTAs/SM (V=1e8: N=4 2240 -> 2253 sweeps/s, 1.25e7 genes 70.0 ->
  // 67.9 us; N=6 1395 -> 1444, N=7 1124 -> 1216, N=8 871 -> 920; DMMA d = 10..14 +0.5..4%).  At
  // 3-4 CTAs/SM (d = 1, 2, DMMA d <= 9) it forces spills: -2 to -16% (profiles/r02_reducer_*).
  static constexpr bool kReducer =
      CAVI_REDUCER_WARP && (!kMma || D <= CAVI_REDUCER_MMA_MAXD) && D >= CAVI_REDUCER_MIN_D && kMinBlocks <= 2;
  static constexpr int kCtaThreads = kCons + 32 + (kReducer ? 32 : 0);  // + 1 TMA producer warp (+ reducer)
  static constexpr int kBudget = (kMinBlocks > 2 ? 210000 / kMinBlocks : CAVI_SMEM_BUDGET) - kSlotBytes;
  static constexpr int kFit = kBudget / (int)kStageBytes;
  static constexpr int kDrift = (kSlots - 1) * kTilesPerChunk;
  static constexpr int kStages = kFit < 8 ? (kFit < kDrift ? kFit : kDrift) : (8 < kDrift ? 8 : kDrift);
  // [stages][1+D][tile] | full[stages] | empty[stages] | stage chunk id[stages] | slots
  static constexpr int kOffBar = kStages * kStageBytes;
  static constexpr int kOffChunk = kOffBar + 2 * kStages * 8;
  static constexpr int kOffSlots = kOffChunk + kStages * 8;
  static constexpr int kSmem = kOffSlots + kSlotBytes;
  static_assert(kStages >= 2, "stage too large");
  static_assert(kTile % kCons == 0, "tile must split evenly across consumers");
  static_assert(kStages <= (kSlots - 1) * kTilesPerChunk, "warp drift could lap the reduction slots");
};

template <int D, typename T, typename M = double>
__global__ void __launch_bounds__(Geometry<D, T, M>::kCtaThreads, Geometry<D, T, M>::kMinBlocks)
    pass_kernel(PassArgs a) {
  using G = Geometry<D, T, M>;
  // fp32 per-gene math on the register path (CV_STORE_F32M); the DMMA path stays fp64
  constexpr bool kF32Math = sizeof(M) == 4 && !G::kMma;
  constexpr int NS = n_stats(D);
  constexpr int kWarps = G::kCWarps;
  constexpr int kThreads = G::kCons;
  constexpr int kProducerWarp = G::kProducerWarp;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double s_red[kWarps + 1][NS];  // per-warp chunk sum / final totals (+ the reducer's)
  __shared__ unsigned int s_cnt[kSlots];
  // reducer hand-off (G::kReducer): slot q holds chunk red_chunk[q] once red_full[q] completes
  // (one arrival per consumer warp); the reducer releases it through red_empty[q]
  __shared__ uint64_t red_full[kSlots], red_empty[kSlots];
  __shared__ int64_t red_chunk[kSlots];
  T* stage_base = reinterpret_cast<T*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G::kOffBar);
  uint64_t* empty = full + G::kStages;
  int64_t* stage_chunk = reinterpret_cast<int64_t*>(smem + G::kOffChunk);
  double* slots = reinterpret_cast<double*>(smem + G::kOffSlots);  // [kSlots][kWarps][NS]

  const Ctl* ctl = a.ctl;
  ptx::griddep_launch_dependents();  // the tail may launch and wait on this grid now
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (a.cta_trace && threadIdx.x == 0) a.cta_trace[blockIdx.x * 8 + 7] = globaltimer_ns();  // resident (pre-wait)
  if (threadIdx.x == 0) {
    for (int q = 0; q < G::kStages; ++q) {
      ptx::mbar_init(&full[q], 1);
      ptx::mbar_init(&empty[q], kWarps);
    }
    for (int q = 0; q < kSlots; ++q) s_cnt[q] = 0u;
    if constexpr (G::kReducer)
      for (int q = 0; q < kSlots; ++q) {
        ptx::mbar_init(&red_full[q], kWarps);
        ptx::mbar_init(&red_empty[q], 1);
      }
    ptx::fence_mbar_init();
  }
  if constexpr (G::kCols > D) {  // zero the padding columns once: TMA never writes them
    for (int q = 0; q < G::kStages; ++q) {
      T* st = stage_base + (size_t)q * (G::kStageBytes / sizeof(T)) + (size_t)(1 + D) * G::kColStride;
      for (int i = threadIdx.x; i < (G::kCols - D) * G::kColStride; i += blockDim.x) st[i] = (T)0;
    }
  }
  __syncthreads();  // barriers initialised
  // Chunk schedule: CTA b's first chunk is chunk b (static); the rest go out as tickets from a
  // counter that is monotone across sweeps (dynamic load balance).  A sweep consumes exactly
  // `period` tickets: the n_chunks - S dynamic chunks plus one end ticket per CTA.
  const int64_t n_static = a.n_chunks < (int64_t)gridDim.x ? a.n_chunks : (int64_t)gridDim.x;
  const unsigned long long period = (unsigned long long)(a.n_chunks - n_static) + gridDim.x;
  const bool has_static = (int64_t)blockIdx.x < n_static;
  // The stream never depends on the previous kernel (the dataset is immutable during a fit),
  // so the producer issues the first stages of its static chunk BEFORE griddepcontrol.wait:
  // under PDL this CTA is resident while the previous sweep's cascade and tail still run, and
  // HBM keeps streaming through them.
  constexpr int kPre = G::kStages < G::kTilesPerChunk ? G::kStages : G::kTilesPerChunk;
  const int tiles_per_chunk = a.chunk_genes / G::kTile;  // >= G::kTilesPerChunk
  const bool producer = warp == kProducerWarp && lane == 0;
  const T* xs = static_cast<const T*>(a.x);
  const T* Ds = static_cast<const T*>(a.D);
  const uint64_t pol = a.l2_keep ? ptx::policy_evict_last() : ptx::policy_evict_first();
  auto issue = [&](int stage, int64_t chunk, int t) {
    stage_chunk[stage] = chunk;
    ptx::mbar_arrive_expect_tx(&full[stage], G::kTxBytes);
    const int64_t g0 = chunk * a.chunk_genes + (int64_t)t * G::kTile;
    T* dst = stage_base + (size_t)stage * (G::kStageBytes / sizeof(T));
    ptx::bulk_g2s(dst, xs + g0, G::kColBytes, &full[stage], pol);
#pragma unroll
    for (int j = 0; j < D; ++j)
      ptx::bulk_g2s(dst + (size_t)(j + 1) * G::kColStride, Ds + (int64_t)j * a.Vp + g0, G::kColBytes, &full[stage],
                    pol);
  };
  if (producer && has_static)
    for (int t = 0; t < kPre; ++t) issue(t, (int64_t)blockIdx.x, t);  // fresh stages: no empty-wait
  // ...and pulls the first dynamic chunks (handed out right after the static ones, to whichever
  // CTA asks first) into L2: the HBM would otherwise idle through the previous sweep's last
  // chunks, its reduction cascade and tail; the stage loads of those chunks then hit in L2.
  if (producer && !a.l2_keep) {
#pragma unroll 1
    for (int p = 0; p < CAVI_L2_PREFETCH_CHUNKS; ++p) {
      const int64_t pc = n_static + (int64_t)p * gridDim.x + blockIdx.x;
      if (pc >= a.n_chunks) break;
      const uint64_t pn = ptx::policy_evict_normal();
      ptx::bulk_prefetch_l2(xs + pc * a.chunk_genes, (uint32_t)(a.chunk_genes * sizeof(T)), pn);
#pragma unroll
      for (int j = 0; j < D; ++j)
        ptx::bulk_prefetch_l2(Ds + (int64_t)j * a.Vp + pc * a.chunk_genes, (uint32_t)(a.chunk_genes * sizeof(T)), pn);
    }
  }
  // everything above reads only the immutable stream or is CTA-local
  ptx::griddep_wait();
  // the done flag is loaded together with the consumers' coefficients (one L2 round trip) and
  // tested once they are in flight
  const int fit_done = *(volatile const int*)&ctl->done;
  if (a.cta_trace && threadIdx.x == 0) a.cta_trace[blockIdx.x * 8] = globaltimer_ns();

  if (warp == kProducerWarp) {
    if (fit_done) {
      if (producer && has_static)  // no bulk copy may still target this CTA's smem when it exits
        for (int t = 0; t < kPre; ++t) ptx::mbar_wait(&full[t], 0u);
      return;
    }
    // ---------------- TMA producer: the rest of the static chunk, then chunk tickets, each
    // chunk tile by tile into the stage ring; a -1 chunk id ends the consumers.
    if (lane == 0) {
      int stage = 0;
      uint32_t parity = 1;  // fresh "empty" barriers count as released
      auto advance = [&]() {
        if (++stage == G::kStages) {
          stage = 0;
          parity ^= 1u;
        }
      };
      if (has_static) {
        for (int t = 0; t < kPre; ++t) advance();  // issued before the wait
        for (int t = kPre; t < tiles_per_chunk; ++t) {
          ptx::mbar_wait(&empty[stage], parity);
          issue(stage, (int64_t)blockIdx.x, t);
          advance();
        }
      }
      // (a ticket is taken only when the previous chunk is fully issued: fetching it one chunk
      // ahead deepens every CTA's queue by a chunk and costs ~4.5 us of end-of-pass imbalance
      // per sweep at d = 3 -- profiles/r02_tpf_ab.log)
      for (;;) {
        const int64_t idx = (int64_t)(atomicAdd(a.ticket, 1ull) % period);
        const int64_t chunk = n_static + idx;
        const bool end = chunk >= a.n_chunks;
        for (int t = 0; t < (end ? 1 : tiles_per_chunk); ++t) {
          ptx::mbar_wait(&empty[stage], parity);
          if (end) {
            stage_chunk[stage] = -1;
            ptx::mbar_arrive(&full[stage]);
          } else {
            issue(stage, chunk, t);
          }
          advance();
        }
        if (end) break;
      }
      if (a.cta_trace) a.cta_trace[blockIdx.x * 8 + 1] = globaltimer_ns();
    }
    return;
  }

  const uint32_t tag = *(volatile const unsigned int*)a.pass_seq;  // LL tag of this pass
  if constexpr (G::kReducer) {
    if (warp == G::kReducerWarp) {
      // ---------------- reducer: chunk n's slot -> warp-order sum -> the cascade (finish_chunk)
      if (fit_done) return;
      double* mine = s_red[kWarps];
#pragma unroll 1
      for (int n = 0;; ++n) {
        const int q = n % kSlots;
        ptx::mbar_wait(&red_full[q], (uint32_t)((n / kSlots) & 1));
        const int64_t chunk = red_chunk[q];
        if (chunk < 0) break;
        const double* slot = slots + (size_t)q * kWarps * NS;
        for (int st = lane; st < NS; st += 32) {
          double v = slot[st];
#pragma unroll
          for (int w = 1; w < kWarps; ++w) v += slot[w * NS + st];
          mine[st] = v;
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&red_empty[q]);  // the slot may be refilled
        finish_chunk<D>(a, chunk, mine, tag, lane);
        __syncwarp();
      }
      return;
    }
  }

  // ---------------- consumers: independent warps, no CTA barrier in the steady state
  constexpr bool kSmemCoef = !G::kMma && D >= CAVI_SMEM_COEF_MIN_D;
  __shared__ GeneCoef<kSmemCoef ? D : 1> s_coef[kSmemCoef ? kWarps : 1];
  GeneCoef<(G::kMma || kSmemCoef || kF32Math ? 1 : D)> k;
  MmaConsumer<D> mc;
  if constexpr (G::kMma) {
    mc.load(ctl->pass, lane);
  } else if constexpr (kSmemCoef) {
    if (lane == 0) load_coef<D>(*reinterpret_cast<GeneCoef<D>*>(&s_coef[warp]), ctl->pass);
    __syncwarp();
  } else if constexpr (!kF32Math) {
    load_coef<D>(*reinterpret_cast<GeneCoef<D>*>(&k), ctl->pass);
  }
  GeneCoefF<kF32Math ? D : 1> kf;
  if constexpr (kF32Math) load_coef_f<D>(kf, ctl->pass);
  const double k_erho = ctl->pass.e_rho;
  if (fit_done) return;
  const int tid = threadIdx.x;  // 0 .. kThreads-1
  int stage = 0;
  uint32_t parity = 0;
  int n_done = 0;
  for (;;) {
    ptx::mbar_wait(&full[stage], parity);
    const int64_t chunk = stage_chunk[stage];
    if (chunk < 0) break;
    double* slot = slots + (size_t)(n_done % kSlots) * kWarps * NS;
    if constexpr (G::kReducer)  // the reducer has read this slot's previous chunk (fresh: free)
      ptx::mbar_wait(&red_empty[n_done % kSlots], (uint32_t)(((n_done / kSlots) & 1) ^ 1));
    if constexpr (G::kMma) {
      mc.reset();
#pragma unroll 1
      for (int t = 0; t < tiles_per_chunk; ++t) {
        if (t) ptx::mbar_wait(&full[stage], parity);
        const T* tile = stage_base + (size_t)stage * (G::kStageBytes / sizeof(T));
        mc.template tile<T, G::kColStride>(tile, warp * (G::kTile / kWarps), G::kTile / kWarps / 8, lane);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[stage]);
        if (++stage == G::kStages) {
          stage = 0;
          parity ^= 1u;
        }
      }
      mc.publish(slot + warp * NS, lane);
    } else {
      double acc[NS];
#pragma unroll
      for (int i = 0; i < NS; ++i) acc[i] = 0.0;
      LogAcc lg;
      lg.init();
#pragma unroll 1
      for (int t = 0; t < tiles_per_chunk; ++t) {
        if (t) ptx::mbar_wait(&full[stage], parity);
        const T* tile = stage_base + (size_t)stage * (G::kStageBytes / sizeof(T));
        double prod = 1.0;
        if constexpr (kF32Math) {  // fp32 per gene, the tile's sums promoted to the fp64 accumulators
          // 16-byte shared loads: this thread's genes come in runs of 4 (a warp reads 512
          // contiguous bytes per column: conflict-free), 4x fewer load instructions per gene
          static_assert(G::kGenesPerThread % 4 == 0, "vector loads need runs of 4 genes");
          float a32[NS];
#pragma unroll
          for (int i = 0; i < NS; ++i) a32[i] = 0.f;
#pragma unroll
          for (int u4 = 0; u4 < G::kGenesPerThread / 4; ++u4) {
            const int g4 = (u4 * kThreads + tid) * 4;
            const float4 xv = *reinterpret_cast<const float4*>(tile + g4);
            float4 dv[D];
#pragma unroll
            for (int j = 0; j < D; ++j) dv[j] = *reinterpret_cast<const float4*>(tile + (j + 1) * G::kColStride + g4);
            const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              float Dv[D];
#pragma unroll
              for (int j = 0; j < D; ++j) Dv[j] = v == 0 ? dv[j].x : v == 1 ? dv[j].y : v == 2 ? dv[j].z : dv[j].w;
              prod *= (double)gene_f<D>(kf, xs[v], Dv, a32);
            }
          }
#pragma unroll
          for (int i = 0; i < NS; ++i)
            if (i != stat_Ld(D)) acc[i] += (double)a32[i];
        } else {
          auto one = [&](double x, const double (&Dv)[D]) {
            if constexpr (kSmemCoef)
              prod *= gene_rows<D>(SmemCoef<D>{reinterpret_cast<const volatile GeneCoef<D>*>(&s_coef[warp]), k_erho},
                                   x, Dv, acc);
            else if constexpr (D >= CAVI_ROWFORM_MIN_D)
              prod *= gene_rows<D>(RegCoef<D>{*reinterpret_cast<const GeneCoef<D>*>(&k)}, x, Dv, acc);
            else
              prod *= gene<D>(*reinterpret_cast<const GeneCoef<D>*>(&k), x, Dv, acc);
          };
          if constexpr (sizeof(T) == 4 && G::kGenesPerThread % 4 == 0) {
            // fp32 stream, fp64 math: 16-byte shared loads as on the fp32-math path
#pragma unroll
            for (int u4 = 0; u4 < G::kGenesPerThread / 4; ++u4) {
              const int g4 = (u4 * kThreads + tid) * 4;
              const float4 xv = *reinterpret_cast<const float4*>(tile + g4);
              float4 dv[D];
#pragma unroll
              for (int j = 0; j < D; ++j)
                dv[j] = *reinterpret_cast<const float4*>(tile + (j + 1) * G::kColStride + g4);
              const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
              for (int v = 0; v < 4; ++v) {
                double Dv[D];
#pragma unroll
                for (int j = 0; j < D; ++j)
                  Dv[j] = (double)(v == 0 ? dv[j].x : v == 1 ? dv[j].y : v == 2 ? dv[j].z : dv[j].w);
                one((double)xs[v], Dv);
              }
            }
          } else {
#pragma unroll
            for (int u = 0; u < G::kGenesPerThread; ++u) {
              const int gi = u * kThreads + tid;
              double Dv[D];
#pragma unroll
              for (int j = 0; j < D; ++j) Dv[j] = (double)tile[(j + 1) * G::kColStride + gi];
              one((double)tile[gi], Dv);
            }
          }
        }
        lg.mul(prod);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[stage]);
        if (++stage == G::kStages) {
          stage = 0;
          parity ^= 1u;
        }
      }
      acc[stat_Ld(D)] = lg.log_value();
      // warp sum (fixed butterfly) -> this warp's slot of the chunk
#pragma unroll
      for (int i = 0; i < NS; ++i) {
        double v = acc[i];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == (i & 31)) slot[warp * NS + i] = v;
      }
    }
    if constexpr (G::kReducer) {  // hand the chunk to the reducer warp and carry on streaming
      __syncwarp();
      if (lane == 0) {
        if (warp == 0) red_chunk[n_done % kSlots] = chunk;
        ptx::mbar_arrive(&red_full[n_done % kSlots]);
      }
      ++n_done;
      continue;
    }
    // the last warp to finish the chunk sums the 8 warp slots (warp order) and carries on up
    unsigned int last = 0;
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      last = atomicAdd(&s_cnt[n_done % kSlots], 1u) == kWarps - 1;
      if (last) {
        s_cnt[n_done % kSlots] = 0u;
        __threadfence_block();
      }
    }
    if (__shfl_sync(0xffffffffu, last, 0)) {
      double* mine = s_red[warp];
      for (int st = lane; st < NS; st += 32) {
        double v = slot[st];
#pragma unroll
        for (int w = 1; w < kWarps; ++w) v += slot[w * NS + st];
        mine[st] = v;
      }
      __syncwarp();
      finish_chunk<D>(a, chunk, mine, tag, lane);
    }
    ++n_done;
  }
  if constexpr (G::kReducer) {  // end of the stream: a chunk id of -1 ends the reducer
    const int q = n_done % kSlots;
    ptx::mbar_wait(&red_empty[q], (uint32_t)(((n_done / kSlots) & 1) ^ 1));
    __syncwarp();
    if (lane == 0) {
      if (warp == 0) red_chunk[q] = -1;
      ptx::mbar_arrive(&red_full[q]);
    }
  }
  if (a.cta_trace && tid == 0) {
    a.cta_trace[blockIdx.x * 8 + 2] = globaltimer_ns();
    a.cta_trace[blockIdx.x * 8 + 3] = smid();
  }
}

}  // namespace cavi
