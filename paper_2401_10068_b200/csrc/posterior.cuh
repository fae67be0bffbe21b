// posterior.cuh -- joint (K, Lambda, rho) draws from the fitted Q on the device:
// vb_posterior_sample (reference vb.py:357-393) with the reference's Philox stream
// layout, so the same RngStream position yields the same draws (uniforms exact,
// normals to libm ulps, sums to fp64 reordering).
//
//   Lambda_k ~ Wishart(nu = n0 + V, S = lam0l_inv^-1): sum over nu outer products of
//              R u_i (R = chol(S)), u_i ~ N(0, I) -- nu*d normals per draw, consumed in
//              the reference's chunks of max(1, min(n, 4e6 // (nu d))) draws;
//   K_k     = k0k + chol((qv Lambda_k)^-1) u_k;
//   rho     ~ Gamma(a_rho, b_rho) by the vectorised cubed-normal rejection rounds
//              (samplers.py:220-261).
// The Wishart part is the cost (O(n nu d) normals): a grid of CTAs per draw, each
// summing u u^T over a fixed row segment; segments are combined in index order.
#pragma once

#include "gen.cuh"

namespace cavi {

constexpr int kPostThreads = 256;
constexpr int64_t kPostRowsPerThread = 64;
constexpr int64_t kPostSegRows = kPostThreads * kPostRowsPerThread;  // rows of u per CTA segment

// both Box-Muller normals of one block (samplers.py:104-109)
__device__ __forceinline__ double2 block_normals(uint4 w) {
  const double u0 = block_uniform(w, 0), u1 = block_uniform(w, 1);
  const double rad = sqrt(__dmul_rn(-2.0, log(u0)));
  const double ang = __dmul_rn(6.283185307179586, u1);
  double sn, cs;
  sincos(ang, &sn, &cs);
  return make_double2(__dmul_rn(rad, cs), __dmul_rn(rad, sn));
}

struct WishartArgs {
  uint64_t seed, stream_id;
  int d;
  int64_t nu;
  int64_t n_draws;       // draws in this launch (whole reference chunks but possibly the last)
  int64_t k_base;        // first draw (within the launch) of this grid slice
  uint64_t block0;       // first block of the launch's first reference chunk
  int64_t rchunk;        // the reference's draws per RNG request (vb.py:378)
  uint64_t chunk_blocks; // blocks a full chunk consumes: u = normals(rchunk nu d), then normals(rchunk d)
  int64_t n_seg;         // segments per draw
  double* seg_out;       // [n_draws][n_seg][d(d+1)/2]
};

// Stream position of draw k of a launch: its reference chunk c, index j inside it, the
// chunk's first block and its draw count.
struct DrawPos {
  int64_t j, m;
  uint64_t base;
};
__device__ __forceinline__ DrawPos draw_pos(const WishartArgs& a, int64_t k) {
  const int64_t c = k / a.rchunk;
  DrawPos p;
  p.j = k - c * a.rchunk;
  p.m = a.n_draws - c * a.rchunk < a.rchunk ? a.n_draws - c * a.rchunk : a.rchunk;
  p.base = a.block0 + (uint64_t)c * a.chunk_blocks;
  return p;
}

__device__ __forceinline__ uint4 philox_block_s(uint64_t seed, uint64_t sid, uint64_t blk) {
  return philox4x32_10(make_uint4((unsigned)blk, (unsigned)(blk >> 32), (unsigned)sid, (unsigned)(sid >> 32)),
                       make_uint2((unsigned)seed, (unsigned)(seed >> 32)));
}

// grid (n_seg, n_draws): CTA (s, k) sums u_i u_i^T for rows i of segment s of draw k
template <int D>
__global__ void __launch_bounds__(kPostThreads) wishart_segment_kernel(WishartArgs a) {
  constexpr int NP = D * (D + 1) / 2;
  const int64_t k = a.k_base + blockIdx.y, s = blockIdx.x;
  const int64_t row_lo = s * kPostSegRows + (int64_t)threadIdx.x * kPostRowsPerThread;
  const int64_t row_hi = row_lo + kPostRowsPerThread < a.nu ? row_lo + kPostRowsPerThread : a.nu;
  double acc[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) acc[p] = 0.0;
  if (row_lo < a.nu) {
    // elements of this thread: [e0, e1) of its reference chunk's normals
    const DrawPos dp = draw_pos(a, k);
    const uint64_t e0 = ((uint64_t)dp.j * a.nu + row_lo) * D, e1 = ((uint64_t)dp.j * a.nu + row_hi) * D;
    const uint64_t base = dp.base;
    double row[D];
    int j = 0;
    auto push = [&](double v) {
      row[j++] = v;
      if (j == D) {  // a full row u_i: W += u_i u_i^T
        int p = 0;
#pragma unroll
        for (int q = 0; q < D; ++q)
#pragma unroll
          for (int r = q; r < D; ++r) {
            acc[p] = fma(row[q], row[r], acc[p]);
            ++p;
          }
        j = 0;
      }
    };
    uint64_t e = e0;
    if (e & 1) {  // first element is the second half of a block
      push(block_normals(philox_block_s(a.seed, a.stream_id, base + (e >> 1))).y);
      ++e;
    }
    for (; e < e1; e += 2) {
      const double2 nn = block_normals(philox_block_s(a.seed, a.stream_id, base + (e >> 1)));
      push(nn.x);
      if (e + 1 < e1) push(nn.y);
    }
  }
  // fixed-order CTA reduction
  __shared__ double red[kPostThreads / 32][NP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    double v = acc[p];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) red[warp][p] = v;
  }
  __syncthreads();
  if (threadIdx.x < NP) {
    double v = red[0][threadIdx.x];
    for (int w = 1; w < kPostThreads / 32; ++w) v += red[w][threadIdx.x];
    a.seg_out[((size_t)k * a.n_seg + s) * NP + threadIdx.x] = v;
  }
}

// one thread per draw: W = sum of segments (index order); Lambda = R W R^T;
// K = k0k + chol(inv(qv Lambda)) u_k with u_k = normals(m d) of the chunk
template <int D>
__global__ void wishart_finish_kernel(WishartArgs a, const double* R, const double* k0k, double qv, uint64_t,
                                      double* lam_out, double* k_out) {
  constexpr int NP = D * (D + 1) / 2;
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= a.n_draws) return;
  double W[D * D];
  {
    double w[NP];
    for (int p = 0; p < NP; ++p) w[p] = 0.0;
    for (int64_t s = 0; s < a.n_seg; ++s)
      for (int p = 0; p < NP; ++p) w[p] += a.seg_out[((size_t)k * a.n_seg + s) * NP + p];
    int p = 0;
    for (int q = 0; q < D; ++q)
      for (int r = q; r < D; ++r) {
        W[q * D + r] = w[p];
        W[r * D + q] = w[p];
        ++p;
      }
  }
  double L[D * D];  // Lambda = R W R^T
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j) {
      double t = 0.0;
      for (int q = 0; q < D; ++q) {
        double u = 0.0;
        for (int r = 0; r < D; ++r) u += W[q * D + r] * R[j * D + r];
        t += R[i * D + q] * u;
      }
      L[i * D + j] = t;
    }
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < i; ++j) L[i * D + j] = L[j * D + i] = 0.5 * (L[i * D + j] + L[j * D + i]);
  for (int i = 0; i < D * D; ++i) lam_out[k * D * D + i] = L[i];
  // cov_k = inv(qv Lambda), Lk = chol(cov_k)  (Cholesky of the precision, then triangular inverse)
  double P[D * D], C[D * D], ld;
  for (int i = 0; i < D * D; ++i) P[i] = qv * L[i];
  if (!spd_inv_logdet_chol_t<D>(P, C, &ld)) {
    for (int i = 0; i < D; ++i) k_out[k * D + i] = qnan();
    return;
  }
  double Lk[D * D];
  if (!chol_t<D>(C, Lk)) {
    for (int i = 0; i < D; ++i) k_out[k * D + i] = qnan();
    return;
  }
  double uk[D];
  const DrawPos dp = draw_pos(a, k);
  const uint64_t block_k = dp.base + (uint64_t)((dp.m * a.nu * D + 1) / 2);  // after the chunk's u
  for (int j = 0; j < D; ++j) {
    const uint64_t e = (uint64_t)dp.j * D + j;
    const double2 nn = block_normals(philox_block_s(a.seed, a.stream_id, block_k + (e >> 1)));
    uk[j] = (e & 1) ? nn.y : nn.x;
  }
  for (int i = 0; i < D; ++i) {
    double t = 0.0;
    for (int j = 0; j < D; ++j) t += Lk[i * D + j] * uk[j];
    k_out[k * D + i] = k0k[i] + t;
  }
}

// one rejection round of _gamma_ge1_many: u = uniforms(todo) from block bu, x = normals(todo)
// from block bx; flags[i] = accepted; val[i] = dd * v
static __global__ void gamma_round_kernel(uint64_t seed, uint64_t sid, uint64_t bu, uint64_t bx, int64_t todo, double dd,
                                   double cc, double* val, char* flags) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= todo) return;
  const double u = block_uniform(philox_block_s(seed, sid, bu + (i >> 1)), (int)(i & 1));
  const double2 nn = block_normals(philox_block_s(seed, sid, bx + (i >> 1)));
  const double x = (i & 1) ? nn.y : nn.x;
  const double t = 1.0 + cc * x;
  const double v = t * t * t;
  bool ok = false;
  if (v > 0.0) ok = log(u) < 0.5 * x * x + dd - dd * v + dd * log(v);
  flags[i] = ok ? 1 : 0;
  val[i] = dd * v;
}

// raw -> rho = raw / b  (boost path for a < 1: raw = boost * u^(1/a), u = uniforms(n) from bu)
static __global__ void gamma_finish_kernel(const double* raw, int64_t n, int boosted, uint64_t seed, uint64_t sid, uint64_t bu,
                                    double a, double b, double* rho) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double r = raw[i];
  if (boosted) r = r * pow(block_uniform(philox_block_s(seed, sid, bu + (i >> 1)), (int)(i & 1)), 1.0 / a);
  rho[i] = r / b;
}

}  // namespace cavi
