// kde.cu -- posterior summaries on the GPU: the reference's
// analysis.kde_fit / kde_density / kde_grid / kde_mode / summarize (analysis.py:58-188).
//
// The work is O(columns x grid x samples) Gaussian-kernel terms plus a golden-section
// refinement whose six density evaluations are each a reduction over all samples.
// Every column is independent:
//   kde_stats_kernel    one CTA per column: mean, sample sd (ddof=1), min, max with
//                       compensated (TwoSum) sums -- the reference's np.mean / np.std
//   cub segmented sort  order statistics for the central interval (np.quantile 'linear')
//   kde_setup_kernel    bandwidth (explicit or Scott's rule), grid range, quantiles
//   kde_partial_kernel  grid points x sample splits: sum exp(-z^2/2), z = (x - s)/h, per
//                       split with TwoSum compensation (the reference's chunked einsum)
//   kde_mode_kernel     one CTA per column: combine splits in fixed order, argmax with the
//                       1e-12 near-tie rule, three golden-section steps (analysis.py:98-139)
// Arithmetic mirrors the reference's operation order (no FMA contraction where numpy
// rounds twice: linspace, golden section, quantile lerp); the sums are compensated, so
// densities agree with numpy's pairwise sums to ~1e-15 relative.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "../../include/cavi.h"

namespace cavi {
int set_error(int code, const char* msg);
}

namespace {

constexpr int kStatThreads = 512;
constexpr int kPartThreads = 256;   // grid points per partial block
constexpr int kSplit = 2048;        // samples per partial block
constexpr int kModeThreads = 512;

struct Acc {  // compensated sum: value = s + c
  double s = 0.0, c = 0.0;
  __device__ __forceinline__ void add(double x) {
    const double t = __dadd_rn(s, x);
    const double bp = __dsub_rn(t, s);
    const double err = __dadd_rn(__dsub_rn(s, __dsub_rn(t, bp)), __dsub_rn(x, bp));
    s = t;
    c = __dadd_rn(c, err);
  }
  __device__ __forceinline__ void merge(const Acc& o) {
    c = __dadd_rn(c, o.c);
    add(o.s);
  }
  __device__ __forceinline__ double value() const { return __dadd_rn(s, c); }
};

__device__ __forceinline__ Acc warp_merge(Acc a) {
  for (int off = 16; off; off >>= 1) {
    Acc o;
    o.s = __shfl_xor_sync(0xffffffffu, a.s, off);
    o.c = __shfl_xor_sync(0xffffffffu, a.c, off);
    a.merge(o);
  }
  return a;
}

// deterministic block reduction (fixed tree), result broadcast to all threads
template <int T>
__device__ Acc block_merge(Acc a, Acc* sh) {
  a = warp_merge(a);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = a;
  __syncthreads();
  if (w == 0) {
    Acc b = l < T / 32 ? sh[l] : Acc();
    b = warp_merge(b);
    if (l == 0) sh[0] = b;
  }
  __syncthreads();
  return sh[0];
}

struct ColOut {  // per column results (see cv_kde_summary)
  double mean, sd, h, mode, multimodal, qlo, qhi, trivial, lo, hi;
};

__global__ void __launch_bounds__(kStatThreads) kde_stats_kernel(const double* cols, int64_t n, ColOut* out) {
  __shared__ Acc sh[kStatThreads / 32];
  __shared__ double smin[kStatThreads / 32], smax[kStatThreads / 32];
  const double* x = cols + (int64_t)blockIdx.x * n;
  Acc a;
  double mn = INFINITY, mx = -INFINITY;
  for (int64_t i = threadIdx.x; i < n; i += kStatThreads) {
    const double v = x[i];
    a.add(v);
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  }
  const double sum = block_merge<kStatThreads>(a, sh).value();
  const double mean = sum / (double)n;  // np.mean: add.reduce(x) / n
  Acc q;
  for (int64_t i = threadIdx.x; i < n; i += kStatThreads) {
    const double dv = __dsub_rn(x[i], mean);
    q.add(__dmul_rn(dv, dv));
  }
  const double ss = block_merge<kStatThreads>(q, sh).value();
  for (int off = 16; off; off >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, off));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  }
  if ((threadIdx.x & 31) == 0) {
    smin[threadIdx.x >> 5] = mn;
    smax[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kStatThreads / 32; ++w) {
      mn = fmin(mn, smin[w]);
      mx = fmax(mx, smax[w]);
    }
    ColOut& o = out[blockIdx.x];
    o.mean = mean;
    o.sd = n > 1 ? sqrt(ss / (double)(n - 1)) : 0.0;  // np.std(ddof=1)
    o.lo = mn;  // sample min / max (the default grid range)
    o.hi = mx;
  }
}

struct SetupArgs {
  const double* cols;
  const double* sorted;
  int64_t n;
  int C;
  const double* bw;     // [C] > 0: explicit bandwidth; else Scott (sd * scott)
  double scott;         // n ** (-1/5), computed as the reference does
  const double* range;  // [2C] explicit grid range or null
  double qlo, qhi;      // central-interval quantiles
  int summarize;        // trivial columns (sd == 0) take mode = x[0] (analysis.py:163-164)
  ColOut* out;
  int* status;
};

__device__ double quantile_linear(const double* s, int64_t n, double q) {
  // np.quantile(method='linear'): v = (n-1) q, lerp of the neighbours (numpy _lerp)
  const double v = __dmul_rn((double)(n - 1), q);
  double prev = floor(v);
  int64_t ip = (int64_t)prev, in = ip + 1;
  if (v >= (double)(n - 1)) ip = in = n - 1;
  if (v < 0) ip = in = 0;
  const double g = __dsub_rn(v, prev);
  const double a = s[ip], b = s[in];
  const double diff = __dsub_rn(b, a);
  if (g >= 0.5) return __dsub_rn(b, __dmul_rn(diff, __dsub_rn(1.0, g)));
  return __dadd_rn(a, __dmul_rn(diff, g));
}

__global__ void kde_setup_kernel(SetupArgs a) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.C) return;
  ColOut& o = a.out[c];
  const double* s = a.sorted + (int64_t)c * a.n;
  o.qlo = quantile_linear(s, a.n, a.qlo);
  o.qhi = quantile_linear(s, a.n, a.qhi);
  o.trivial = o.sd == 0.0 ? 1.0 : 0.0;
  o.multimodal = 0.0;
  double h;
  if (a.bw && a.bw[c] > 0) {
    h = a.bw[c];
  } else {
    if (o.sd == 0.0 && !a.summarize) atomicExch(a.status, 1);  // kde_fit's zero-variance error
    h = __dmul_rn(o.sd, a.scott);
  }
  o.h = h;
  if (a.range) {
    o.lo = a.range[2 * c];
    o.hi = a.range[2 * c + 1];
  } else {
    o.lo = __dsub_rn(o.lo, __dmul_rn(4.0, h));  // samples.min() - 4 h
    o.hi = __dadd_rn(o.hi, __dmul_rn(4.0, h));  // samples.max() + 4 h
  }
  o.mode = a.cols[(int64_t)c * a.n];  // x[0]: the trivial-column mode
}

// np.linspace(lo, hi, m)[g]: g * step + lo (two roundings), last point exactly hi
__device__ __forceinline__ double grid_x(double lo, double hi, int m, int g) {
  if (g == m - 1) return hi;
  const double step = __ddiv_rn(__dsub_rn(hi, lo), (double)(m - 1));
  return __dadd_rn(__dmul_rn((double)g, step), lo);
}

__device__ __forceinline__ double kterm(double x, double s, double h) {
  const double z = __ddiv_rn(__dsub_rn(x, s), h);
  return exp(__dmul_rn(-0.5, __dmul_rn(z, z)));
}

// blockIdx: x = grid-point block, y = sample split, z = column
__global__ void __launch_bounds__(kPartThreads) kde_partial_kernel(const double* cols, int64_t n, const ColOut* outc,
                                                                  const double* xq, int m, int skip_trivial,
                                                                  double2* part) {
  __shared__ double sm[kSplit];
  const int c = blockIdx.z;
  const ColOut& o = outc[c];
  if (skip_trivial && o.trivial != 0.0) return;
  const int64_t s0 = (int64_t)blockIdx.y * kSplit;
  const int64_t s1 = s0 + kSplit < n ? s0 + kSplit : n;
  const double* x = cols + (int64_t)c * n;
  for (int64_t i = s0 + threadIdx.x; i < s1; i += kPartThreads) sm[i - s0] = x[i];
  __syncthreads();
  const int g = blockIdx.x * kPartThreads + threadIdx.x;
  if (g >= m) return;
  const double xv = xq ? xq[(int64_t)c * m + g] : grid_x(o.lo, o.hi, m, g);
  const double h = o.h;
  Acc a;
  const int cnt = (int)(s1 - s0);
  for (int i = 0; i < cnt; ++i) a.add(kterm(xv, sm[i], h));
  part[((int64_t)c * gridDim.y + blockIdx.y) * m + g] = make_double2(a.s, a.c);
}

__device__ double point_density(const double* x, int64_t n, double h, double norm, double at, Acc* sh) {
  Acc a;
  for (int64_t i = threadIdx.x; i < n; i += kModeThreads) a.add(kterm(at, x[i], h));
  return __dmul_rn(norm, block_merge<kModeThreads>(a, sh).value());
}

struct ModeArgs {
  const double* cols;
  int64_t n;
  ColOut* out;
  const double2* part;
  int splits;
  int m;
  double sqrt2pi;
  double golden;
  int skip_trivial;
  int find_mode;
  double* dens;  // [C][m] or null
};

__global__ void __launch_bounds__(kModeThreads) kde_mode_kernel(ModeArgs a) {
  __shared__ Acc sh[kModeThreads / 32];
  __shared__ double sval[kModeThreads / 32];
  __shared__ int sidx[kModeThreads / 32], sfirst[kModeThreads / 32], slast[kModeThreads / 32],
      scnt[kModeThreads / 32];
  const int c = blockIdx.x;
  ColOut& o = a.out[c];
  if (a.skip_trivial && o.trivial != 0.0) return;
  const double h = o.h;
  // norm = 1 / (n h sqrt(2 pi))   (analysis.py:81)
  const double norm = __ddiv_rn(1.0, __dmul_rn(__dmul_rn((double)a.n, h), a.sqrt2pi));
  const int m = a.m;
  extern __shared__ double dens_sm[];  // [m]
  for (int g = threadIdx.x; g < m; g += kModeThreads) {
    Acc t;
    for (int sp = 0; sp < a.splits; ++sp) {
      const double2 p = a.part[((int64_t)c * a.splits + sp) * m + g];
      Acc q;
      q.s = p.x;
      q.c = p.y;
      if (sp == 0) t = q;
      else t.merge(q);
    }
    const double d = __dmul_rn(norm, t.value());
    dens_sm[g] = d;
    if (a.dens) a.dens[(int64_t)c * m + g] = d;
  }
  __syncthreads();
  if (!a.find_mode) return;
  // argmax (first occurrence)
  double bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int g = threadIdx.x; g < m; g += kModeThreads) {
    const double d = dens_sm[g];
    if (d > bv || (d == bv && g < bi)) {
      bv = d;
      bi = g;
    }
  }
  for (int off = 16; off; off >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sval[w] = bv;
    sidx[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < kModeThreads / 32; ++k)
      if (sval[k] > bv || (sval[k] == bv && sidx[k] < bi)) {
        bv = sval[k];
        bi = sidx[k];
      }
    sval[0] = bv;
    sidx[0] = bi;
  }
  __syncthreads();
  const double thr = __dsub_rn(sval[0], 1e-12);
  // near ties: first, last, count
  int first = 0x7fffffff, last = -1, cnt = 0;
  for (int g = threadIdx.x; g < m; g += kModeThreads)
    if (dens_sm[g] >= thr) {
      first = min(first, g);
      last = max(last, g);
      ++cnt;
    }
  for (int off = 16; off; off >>= 1) {
    first = min(first, __shfl_xor_sync(0xffffffffu, first, off));
    last = max(last, __shfl_xor_sync(0xffffffffu, last, off));
    cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
  }
  __syncthreads();
  if (l == 0) {
    sfirst[w] = first;
    slast[w] = last;
    scnt[w] = cnt;
  }
  __syncthreads();
  first = 0x7fffffff;
  last = -1;
  cnt = 0;
  for (int k = 0; k < kModeThreads / 32; ++k) {
    first = min(first, sfirst[k]);
    last = max(last, slast[k]);
    cnt += scnt[k];
  }
  const bool multimodal = cnt != last - first + 1;  // any gap between near-tie cells
  const int best = first;
  double lo_ = grid_x(o.lo, o.hi, m, best > 0 ? best - 1 : 0);
  double hi_ = grid_x(o.lo, o.hi, m, best + 1 < m ? best + 1 : m - 1);
  const double G = a.golden;
  const double* x = a.cols + (int64_t)c * a.n;
  double cc = __dsub_rn(hi_, __dmul_rn(G, __dsub_rn(hi_, lo_)));
  double dd = __dadd_rn(lo_, __dmul_rn(G, __dsub_rn(hi_, lo_)));
  double fc = point_density(x, a.n, h, norm, cc, sh);
  double fd = point_density(x, a.n, h, norm, dd, sh);
  for (int it = 0; it < 3; ++it) {
    if (fc > fd) {
      hi_ = dd;
      dd = cc;
      fd = fc;
      cc = __dsub_rn(hi_, __dmul_rn(G, __dsub_rn(hi_, lo_)));
      fc = point_density(x, a.n, h, norm, cc, sh);
    } else {
      lo_ = cc;
      cc = dd;
      fc = fd;
      dd = __dadd_rn(lo_, __dmul_rn(G, __dsub_rn(hi_, lo_)));
      fd = point_density(x, a.n, h, norm, dd, sh);
    }
  }
  if (threadIdx.x == 0) {
    o.mode = __dmul_rn(0.5, __dadd_rn(lo_, hi_));
    o.multimodal = multimodal ? 1.0 : 0.0;
  }
}

// row-major (n, d) K / Lambda draws -> the column-major work matrix
__global__ void gather_kernel(const double* K, const double* rho, const double* Lam, int64_t n, int d, double* cols) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* k = K + i * d;
  // full_weights: (K, 1 - K.sum()) with numpy's summation order for d < 16 (model.py:218-221)
  double s;
  if (d < 8) {
    s = 0.0;
    for (int j = 0; j < d; ++j) s = __dadd_rn(s, k[j]);
  } else {
    const double r01 = __dadd_rn(k[0], k[1]), r23 = __dadd_rn(k[2], k[3]);
    const double r45 = __dadd_rn(k[4], k[5]), r67 = __dadd_rn(k[6], k[7]);
    s = __dadd_rn(__dadd_rn(r01, r23), __dadd_rn(r45, r67));
    for (int j = 8; j < d; ++j) s = __dadd_rn(s, k[j]);
  }
  int c = 0;
  for (int j = 0; j < d; ++j) cols[(int64_t)(c++) * n + i] = k[j];  // K_1..K_d
  for (int j = 0; j < d; ++j) cols[(int64_t)(c++) * n + i] = k[j];  // w_1..w_d
  cols[(int64_t)(c++) * n + i] = __dsub_rn(1.0, s);                  // w_{d+1}
  cols[(int64_t)(c++) * n + i] = rho[i];
  if (Lam)
    for (int q = 0; q < d * d; ++q) cols[(int64_t)(c++) * n + i] = Lam[i * d * d + q];
}

#define KCK(call)                                                                                   \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess)                                                                          \
      return cavi::set_error(CV_ERR_CUDA, (std::string(#call) + ": " + cudaGetErrorString(e_)).c_str()); \
  } while (0)

struct Scratch {
  std::vector<void*> p;
  ~Scratch() {
    for (void* q : p) cudaFree(q);
  }
  template <typename T>
  cudaError_t alloc(T** out, size_t bytes) {
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, bytes ? bytes : 8);
    if (e == cudaSuccess) p.push_back(q);
    *out = (T*)q;
    return e;
  }
};

// columns already on the device (C x n, column-major)
int summary_device(const double* dcols, int64_t n, int C, int C_kde, const double* bw, double scott, double sqrt2pi,
                   double golden, int grid_n, const double* range, double qlo, double qhi, int summarize,
                   int find_mode, double* out, double* grid_out, cudaStream_t st, Scratch& sc) {
  ColOut* dout = nullptr;
  KCK(sc.alloc(&dout, sizeof(ColOut) * C));
  kde_stats_kernel<<<C, kStatThreads, 0, st>>>(dcols, n, dout);
  KCK(cudaGetLastError());
  if (C_kde > 0) {
    double* sorted = nullptr;
    int64_t* offs = nullptr;
    KCK(sc.alloc(&sorted, sizeof(double) * n * C_kde));
    KCK(sc.alloc(&offs, sizeof(int64_t) * (C_kde + 1)));
    std::vector<int64_t> ho(C_kde + 1);
    for (int c = 0; c <= C_kde; ++c) ho[c] = (int64_t)c * n;
    KCK(cudaMemcpyAsync(offs, ho.data(), sizeof(int64_t) * ho.size(), cudaMemcpyHostToDevice, st));
    size_t tb = 0;
    KCK(cub::DeviceSegmentedRadixSort::SortKeys(nullptr, tb, dcols, sorted, n * C_kde, C_kde, offs, offs + 1, 0, 64,
                                                st));
    void* tmp = nullptr;
    KCK(sc.alloc(&tmp, tb));
    KCK(cub::DeviceSegmentedRadixSort::SortKeys(tmp, tb, dcols, sorted, n * C_kde, C_kde, offs, offs + 1, 0, 64, st));
    double *dbw = nullptr, *drange = nullptr;
    int* dstatus = nullptr;
    if (bw) {
      KCK(sc.alloc(&dbw, sizeof(double) * C_kde));
      KCK(cudaMemcpyAsync(dbw, bw, sizeof(double) * C_kde, cudaMemcpyHostToDevice, st));
    }
    if (range) {
      KCK(sc.alloc(&drange, sizeof(double) * 2 * C_kde));
      KCK(cudaMemcpyAsync(drange, range, sizeof(double) * 2 * C_kde, cudaMemcpyHostToDevice, st));
    }
    KCK(sc.alloc(&dstatus, sizeof(int)));
    KCK(cudaMemsetAsync(dstatus, 0, sizeof(int), st));
    SetupArgs sa{dcols, sorted, n, C_kde, dbw, scott, drange, qlo, qhi, summarize, dout, dstatus};
    kde_setup_kernel<<<(C_kde + 63) / 64, 64, 0, st>>>(sa);
    KCK(cudaGetLastError());
    int hstatus = 0;
    KCK(cudaMemcpyAsync(&hstatus, dstatus, sizeof(int), cudaMemcpyDeviceToHost, st));
    KCK(cudaStreamSynchronize(st));
    if (hstatus) return cavi::set_error(CV_ERR_ARG, "zero-variance samples: pass an explicit bandwidth");
    if (grid_n > 0) {
      const int splits = (int)((n + kSplit - 1) / kSplit);
      double2* part = nullptr;
      KCK(sc.alloc(&part, sizeof(double2) * (size_t)C_kde * splits * grid_n));
      dim3 grid((grid_n + kPartThreads - 1) / kPartThreads, splits, C_kde);
      kde_partial_kernel<<<grid, kPartThreads, 0, st>>>(dcols, n, dout, nullptr, grid_n, summarize, part);
      KCK(cudaGetLastError());
      double* ddens = nullptr;
      if (grid_out) KCK(sc.alloc(&ddens, sizeof(double) * (size_t)C_kde * grid_n));
      ModeArgs ma{dcols, n, dout, part, splits, grid_n, sqrt2pi, golden, summarize, find_mode, ddens};
      const size_t smem = sizeof(double) * grid_n;
      if (smem > 48 * 1024) KCK(cudaFuncSetAttribute(kde_mode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)smem));
      kde_mode_kernel<<<C_kde, kModeThreads, smem, st>>>(ma);
      KCK(cudaGetLastError());
      if (grid_out)
        KCK(cudaMemcpyAsync(grid_out, ddens, sizeof(double) * (size_t)C_kde * grid_n, cudaMemcpyDeviceToHost, st));
    }
  }
  std::vector<ColOut> h(C);
  KCK(cudaMemcpyAsync(h.data(), dout, sizeof(ColOut) * C, cudaMemcpyDeviceToHost, st));
  KCK(cudaStreamSynchronize(st));
  for (int c = 0; c < C; ++c) {
    double* o = out + (size_t)c * 10;
    const ColOut& q = h[c];
    o[0] = q.mean;
    o[1] = q.sd;
    o[2] = q.h;
    o[3] = q.mode;
    o[4] = q.multimodal;
    o[5] = q.qlo;
    o[6] = q.qhi;
    o[7] = q.trivial;
    o[8] = q.lo;
    o[9] = q.hi;
  }
  return CV_OK;
}

}  // namespace

extern "C" {

int32_t cv_kde_columns(const double* cols, int64_t n, int32_t C, const double* bw, double scott, double sqrt2pi,
                       double golden, int32_t grid_n, const double* range, double qlo, double qhi, int32_t find_mode,
                       int32_t device, double* out, double* grid_out) {
  if (!cols || !out || n < 2 || C < 1) return cavi::set_error(CV_ERR_ARG, "need at least 2 samples per column");
  KCK(cudaSetDevice(device));
  Scratch sc;
  double* dcols = nullptr;
  KCK(sc.alloc(&dcols, sizeof(double) * n * C));
  KCK(cudaMemcpy(dcols, cols, sizeof(double) * n * C, cudaMemcpyHostToDevice));
  return summary_device(dcols, n, C, C, bw, scott, sqrt2pi, golden, grid_n, range, qlo, qhi, 0, find_mode, out,
                        grid_out, 0, sc);
}

int32_t cv_kde_density(const double* samples, int64_t n, double h, double sqrt2pi, const double* x, int64_t m,
                       int32_t device, double* out) {
  if (!samples || !x || !out || n < 1 || m < 0 || !(h > 0)) return cavi::set_error(CV_ERR_ARG, "bad arguments");
  if (m == 0) return CV_OK;
  KCK(cudaSetDevice(device));
  Scratch sc;
  double *ds = nullptr, *dx = nullptr, *dd = nullptr;
  double2* part = nullptr;
  ColOut* dout = nullptr;
  const int splits = (int)((n + kSplit - 1) / kSplit);
  KCK(sc.alloc(&ds, sizeof(double) * n));
  KCK(sc.alloc(&dx, sizeof(double) * m));
  KCK(sc.alloc(&dd, sizeof(double) * m));
  KCK(sc.alloc(&part, sizeof(double2) * (size_t)splits * m));
  KCK(sc.alloc(&dout, sizeof(ColOut)));
  ColOut o{};
  o.h = h;
  KCK(cudaMemcpy(ds, samples, sizeof(double) * n, cudaMemcpyHostToDevice));
  KCK(cudaMemcpy(dx, x, sizeof(double) * m, cudaMemcpyHostToDevice));
  KCK(cudaMemcpy(dout, &o, sizeof o, cudaMemcpyHostToDevice));
  // points in chunks of 8192 (the combine kernel keeps one chunk of densities in shared memory)
  for (int64_t p0 = 0; p0 < m; p0 += 8192) {
    const int mm = (int)(m - p0 < 8192 ? m - p0 : 8192);
    dim3 grid((mm + kPartThreads - 1) / kPartThreads, splits, 1);
    kde_partial_kernel<<<grid, kPartThreads>>>(ds, n, dout, dx + p0, mm, 0, part);
    KCK(cudaGetLastError());
    ModeArgs ma{ds, n, dout, part, splits, mm, sqrt2pi, 0.0, 0, 0, dd + p0};
    KCK(cudaFuncSetAttribute(kde_mode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 8));
    kde_mode_kernel<<<1, kModeThreads, sizeof(double) * mm>>>(ma);
    KCK(cudaGetLastError());
  }
  KCK(cudaMemcpy(out, dd, sizeof(double) * m, cudaMemcpyDeviceToHost));
  return CV_OK;
}

int32_t cv_summarize(const double* K, const double* rho, const double* Lam, int64_t n, int32_t d, double bandwidth,
                     double scott, double sqrt2pi, double golden, double qlo, double qhi, int32_t device,
                     double* out, double* lam_mean) {
  if (!K || !rho || !out || n < 2 || d < 1) return cavi::set_error(CV_ERR_ARG, "bad arguments");
  KCK(cudaSetDevice(device));
  Scratch sc;
  const int C_kde = 2 * d + 2;
  const int C = C_kde + (Lam ? d * d : 0);
  double *dK = nullptr, *drho = nullptr, *dL = nullptr, *dcols = nullptr;
  KCK(sc.alloc(&dK, sizeof(double) * n * d));
  KCK(sc.alloc(&drho, sizeof(double) * n));
  KCK(sc.alloc(&dcols, sizeof(double) * n * C));
  KCK(cudaMemcpy(dK, K, sizeof(double) * n * d, cudaMemcpyHostToDevice));
  KCK(cudaMemcpy(drho, rho, sizeof(double) * n, cudaMemcpyHostToDevice));
  if (Lam) {
    KCK(sc.alloc(&dL, sizeof(double) * n * d * d));
    KCK(cudaMemcpy(dL, Lam, sizeof(double) * n * d * d, cudaMemcpyHostToDevice));
  }
  gather_kernel<<<(unsigned)((n + 255) / 256), 256>>>(dK, drho, dL, n, d, dcols);
  KCK(cudaGetLastError());
  std::vector<double> bw(C_kde, bandwidth > 0 ? bandwidth : 0.0);
  std::vector<double> all((size_t)C * 10);
  int rc = summary_device(dcols, n, C, C_kde, bw.data(), scott, sqrt2pi, golden, 512, nullptr, qlo, qhi, 1, 1,
                          all.data(), nullptr, 0, sc);
  if (rc) return rc;
  for (int c = 0; c < C_kde * 10; ++c) out[c] = all[c];
  if (Lam && lam_mean)
    for (int q = 0; q < d * d; ++q) lam_mean[q] = all[(size_t)(C_kde + q) * 10];
  return CV_OK;
}

}  // extern "C"
