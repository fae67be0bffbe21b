// gen.cuh -- device-side dataset construction: the Philox4x32-10 synthetic
// generator (stream-exact with reference samplers.py:47-147 + model.py:224-270),
// the host-upload transform (model.py:174-189: x = r - mu, D columns), and the
// lazy per-gene moment materialisation (VbState.mu_beta / lam_beta / e_bbt).
#pragma once

#include "engine.cuh"

namespace cavi {

// ------------------------------------------------------------------ Philox4x32-10
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned int hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const unsigned int hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// block `blk` of stream 0 under `seed` (counter = [blk_lo, blk_hi, 0, 0], key = seed words)
__device__ __forceinline__ uint4 philox_block(uint64_t seed, uint64_t blk) {
  return philox4x32_10(make_uint4((unsigned)blk, (unsigned)(blk >> 32), 0u, 0u),
                       make_uint2((unsigned)seed, (unsigned)(seed >> 32)));
}

// element `which` (0/1) of the block's two (0,1] uniforms (samplers.py:95-101)
__device__ __forceinline__ double block_uniform(uint4 w, int which) {
  const uint64_t v = which == 0 ? (((uint64_t)w.x << 32) | w.y) : (((uint64_t)w.z << 32) | w.w);
  return __dmul_rn(__dadd_rn((double)(v >> 11), 1.0), 1.1102230246251565e-16);
}

// element `which` of the block's Box-Muller pair (samplers.py:104-109)
__device__ __forceinline__ double block_normal(uint4 w, int which) {
  const double u0 = block_uniform(w, 0), u1 = block_uniform(w, 1);
  const double rad = sqrt(__dmul_rn(-2.0, log(u0)));
  const double ang = __dmul_rn(6.283185307179586, u1);
  return which == 0 ? __dmul_rn(rad, cos(ang)) : __dmul_rn(rad, sin(ang));
}

// value #e of a draw that started at block `b0`
__device__ __forceinline__ double stream_normal(uint64_t seed, uint64_t b0, uint64_t e) {
  return block_normal(philox_block(seed, b0 + (e >> 1)), (int)(e & 1));
}

struct GenArgs {
  uint64_t seed;
  int64_t gene_lo, V, V_total, Vp;
  int N, d, storage;
  double K[kMaxD];
  double L[kMaxD2];  // chol(inv(Lam)), computed by gen_prep_kernel
  double sqrt_rho;  // eps = normal / sqrt(rho)  (model.py:268)
  void* x;
  void* D;
  double* r_raw;   // optional
  double* mu_raw;  // optional
};

// reference model.py:264-265: cov = inverse_batched(Lam); L = cholesky_batched(cov),
// in the reference's operation order (no FMA contraction).
static __global__ void gen_prep_kernel(const double* Lam, double* Lout, int d, int* status) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double C[kMaxD2];
  *status = CV_OK;
  if (d == 1) {
    C[0] = __ddiv_rn(1.0, Lam[0]);
  } else if (d == 2) {
    const double a = Lam[0], b = Lam[1], c = Lam[2], e = Lam[3];
    const double det = __dsub_rn(__dmul_rn(a, e), __dmul_rn(b, c));
    const double r = __ddiv_rn(1.0, det);
    C[0] = __dmul_rn(e, r);
    C[1] = __dmul_rn(-b, r);
    C[2] = __dmul_rn(-c, r);
    C[3] = __dmul_rn(a, r);
  } else if (d == 3) {
#define M(i, j) Lam[(i)*3 + (j)]
    const double c00 = __dsub_rn(__dmul_rn(M(1, 1), M(2, 2)), __dmul_rn(M(1, 2), M(2, 1)));
    const double c01 = __dsub_rn(__dmul_rn(M(1, 2), M(2, 0)), __dmul_rn(M(1, 0), M(2, 2)));
    const double c02 = __dsub_rn(__dmul_rn(M(1, 0), M(2, 1)), __dmul_rn(M(1, 1), M(2, 0)));
    const double det = __dadd_rn(__dadd_rn(__dmul_rn(M(0, 0), c00), __dmul_rn(M(0, 1), c01)), __dmul_rn(M(0, 2), c02));
    const double c10 = __dsub_rn(__dmul_rn(M(0, 2), M(2, 1)), __dmul_rn(M(0, 1), M(2, 2)));
    const double c11 = __dsub_rn(__dmul_rn(M(0, 0), M(2, 2)), __dmul_rn(M(0, 2), M(2, 0)));
    const double c12 = __dsub_rn(__dmul_rn(M(0, 1), M(2, 0)), __dmul_rn(M(0, 0), M(2, 1)));
    const double c20 = __dsub_rn(__dmul_rn(M(0, 1), M(1, 2)), __dmul_rn(M(0, 2), M(1, 1)));
    const double c21 = __dsub_rn(__dmul_rn(M(0, 2), M(1, 0)), __dmul_rn(M(0, 0), M(1, 2)));
    const double c22 = __dsub_rn(__dmul_rn(M(0, 0), M(1, 1)), __dmul_rn(M(0, 1), M(1, 0)));
#undef M
    const double r = __ddiv_rn(1.0, det);
    C[0] = __dmul_rn(c00, r); C[1] = __dmul_rn(c10, r); C[2] = __dmul_rn(c20, r);
    C[3] = __dmul_rn(c01, r); C[4] = __dmul_rn(c11, r); C[5] = __dmul_rn(c21, r);
    C[6] = __dmul_rn(c02, r); C[7] = __dmul_rn(c12, r); C[8] = __dmul_rn(c22, r);
  } else {
    // Gauss-Jordan with partial pivoting (the reference uses LAPACK here; ulp-level agreement)
    double W[kMaxD2];
    for (int i = 0; i < d * d; ++i) {
      W[i] = Lam[i];
      C[i] = 0.0;
    }
    for (int i = 0; i < d; ++i) C[i * d + i] = 1.0;
    for (int col = 0; col < d; ++col) {
      int piv = col;
      for (int i = col + 1; i < d; ++i)
        if (fabs(W[i * d + col]) > fabs(W[piv * d + col])) piv = i;
      if (W[piv * d + col] == 0.0) {
        *status = CV_ERR_NUMERIC;
        return;
      }
      if (piv != col)
        for (int j = 0; j < d; ++j) {
          double t = W[col * d + j]; W[col * d + j] = W[piv * d + j]; W[piv * d + j] = t;
          t = C[col * d + j]; C[col * d + j] = C[piv * d + j]; C[piv * d + j] = t;
        }
      const double p = W[col * d + col];
      for (int j = 0; j < d; ++j) {
        W[col * d + j] /= p;
        C[col * d + j] /= p;
      }
      for (int i = 0; i < d; ++i) {
        if (i == col) continue;
        const double f = W[i * d + col];
        for (int j = 0; j < d; ++j) {
          W[i * d + j] -= f * W[col * d + j];
          C[i * d + j] -= f * C[col * d + j];
        }
      }
    }
  }
  // Cholesky, column by column (linalg.py:214-227)
  for (int i = 0; i < d * d; ++i) Lout[i] = 0.0;
  for (int j = 0; j < d; ++j) {
    double ss = 0.0;
    for (int k = 0; k < j; ++k) ss = __dadd_rn(ss, __dmul_rn(Lout[j * d + k], Lout[j * d + k]));
    const double s = __dsub_rn(C[j * d + j], ss);
    if (!(s > 0.0)) {
      *status = CV_ERR_NUMERIC;
      return;
    }
    const double ljj = __dsqrt_rn(s);
    Lout[j * d + j] = ljj;
    for (int i = j + 1; i < d; ++i) {
      double dot = 0.0;
      for (int k = 0; k < j; ++k) dot = __dadd_rn(dot, __dmul_rn(Lout[i * d + k], Lout[j * d + k]));
      Lout[i * d + j] = __ddiv_rn(__dsub_rn(C[i * d + j], dot), ljj);
    }
  }
}

template <typename T>
__global__ void gen_kernel(GenArgs a, const double* Ldev) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // local gene
  if (i >= a.Vp) return;
  T* xs = static_cast<T*>(a.x);
  T* Ds = static_cast<T*>(a.D);
  const int d = a.d;
  if (i >= a.V) {  // zero padding genes contribute exactly 0 to every statistic
    xs[i] = (T)0;
    for (int j = 0; j < d; ++j) Ds[(int64_t)j * a.Vp + i] = (T)0;
    return;
  }
  const uint64_t gi = (uint64_t)(a.gene_lo + i);
  const uint64_t Vt = (uint64_t)a.V_total;
  // random_profiles: uniforms(V_total) from block 0
  const double u = block_uniform(philox_block(a.seed, gi >> 1), (int)(gi & 1));
  const int64_t ncodes = (int64_t)1 << a.N;
  int64_t code = (int64_t)__dmul_rn(u, (double)ncodes);
  if (code > ncodes - 1) code = ncodes - 1;
  const double mu = (double)((code >> (a.N - 1)) & 1);
  // synth_generate: z = normals(V*d), then eps = normals(V)
  const uint64_t b_z = (Vt + 1) >> 1;
  const uint64_t b_e = b_z + ((Vt * (uint64_t)d + 1) >> 1);
  double z[kMaxD], Dv[kMaxD];
  for (int j = 0; j < d; ++j) {
    z[j] = stream_normal(a.seed, b_z, gi * (uint64_t)d + j);
    Dv[j] = __dsub_rn((double)((code >> j) & 1), mu);
  }
  // beta = K + z @ L^T ; r = D . beta + mu + eps
  double dot = 0.0;
  for (int j = 0; j < d; ++j) {
    double zl = 0.0;
    for (int k = 0; k < d; ++k) zl = __dadd_rn(zl, __dmul_rn(z[k], Ldev[j * d + k]));
    const double beta = __dadd_rn(a.K[j], zl);
    dot = j == 0 ? __dmul_rn(Dv[j], beta) : __dadd_rn(dot, __dmul_rn(Dv[j], beta));
  }
  const double eps = __ddiv_rn(stream_normal(a.seed, b_e, gi), a.sqrt_rho);
  const double r = __dadd_rn(__dadd_rn(dot, mu), eps);
  xs[i] = (T)__dsub_rn(r, mu);
  for (int j = 0; j < d; ++j) Ds[(int64_t)j * a.Vp + i] = (T)Dv[j];
  if (a.r_raw) a.r_raw[i] = r;
  if (a.mu_raw) a.mu_raw[i] = mu;
}

// ------------------------------------------------------------------ host upload transform
template <typename T>
__global__ void upload_kernel(const double* r, const double* mu, const double* Drow, int64_t V, int64_t Vp, int d,
                              T* xs, T* Ds, int* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= Vp) return;
  if (i >= V) {
    xs[i] = (T)0;
    for (int j = 0; j < d; ++j) Ds[(int64_t)j * Vp + i] = (T)0;
    return;
  }
  xs[i] = (T)__dsub_rn(r[i], mu[i]);  // rm = r - mu (vb.py:118)
  int nonfinite = 0;
  for (int j = 0; j < d; ++j) {
    const double v = Drow[i * d + j];
    nonfinite |= !isfinite(v);
    Ds[(int64_t)j * Vp + i] = (T)v;
  }
  if (nonfinite) atomicOr(bad, 1);
}

template <typename T>
__global__ void download_kernel(const T* xs, const T* Ds, int64_t V, int64_t Vp, int d, double* x, double* Drow) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  if (x) x[i] = (double)xs[i];
  if (Drow)
    for (int j = 0; j < d; ++j) Drow[i * d + j] = (double)Ds[(int64_t)j * Vp + i];
}

// ------------------------------------------------------------------ per-gene materialisation
// mu_beta_i = c + w u ; Sigma_i = Ainv - (e_rho/den) u u^T ; lam_beta_i = A + e_rho D D^T ;
// e_bbt_i = mu mu^T + Sigma_i   (vb.py:150-156);  S_i = (x - t - s w)^2 + s/den, the per-gene
// expected squared residual (em.py:56-60)
template <typename T>
__global__ void materialize_kernel(const T* xs, const T* Ds, int64_t Vp, int d, int64_t lo, int64_t n,
                                   const Ctl* ctl, double* mu_out, double* lam_out, double* ebb_out,
                                   double* sig_out, double* res_out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t i = lo + k;
  const cv_state& s = ctl->cur;
  double Dv[kMaxD], u[kMaxD], m[kMaxD];
  const double x = (double)xs[i];
  for (int j = 0; j < d; ++j) Dv[j] = (double)Ds[(int64_t)j * Vp + i];
  double sq = 0.0, t = 0.0;
  for (int j = 0; j < d; ++j) {
    double acc = 0.0;
    for (int q = 0; q < d; ++q) acc += s.gen_Ainv[j * d + q] * Dv[q];
    u[j] = acc;
    sq += Dv[j] * acc;
    t += s.gen_c[j] * Dv[j];
  }
  const double er = s.gen_e_rho;
  const double den = 1.0 + er * sq;
  const double w = er * (x - t) / den;
  for (int j = 0; j < d; ++j) m[j] = s.gen_c[j] + w * u[j];
  if (mu_out)
    for (int j = 0; j < d; ++j) mu_out[k * d + j] = m[j];
  for (int j = 0; j < d; ++j)
    for (int q = 0; q < d; ++q) {
      const double sg = s.gen_Ainv[j * d + q] - (er / den) * u[j] * u[q];
      if (lam_out) lam_out[(k * d + j) * d + q] = s.gen_A[j * d + q] + er * Dv[j] * Dv[q];
      if (ebb_out) ebb_out[(k * d + j) * d + q] = m[j] * m[q] + sg;
      if (sig_out) sig_out[(k * d + j) * d + q] = sg;
    }
  if (res_out) {
    const double e = x - t - sq * w;
    res_out[k] = e * e + sq / den;
  }
}

}  // namespace cavi
