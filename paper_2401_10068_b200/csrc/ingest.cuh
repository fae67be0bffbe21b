// ingest.cuh -- the dataset CSV reader on the GPU, replacing the
// reference's `cli.read_dataset_csv` (cli.py:58-75) + `model.transform` (model.py:174-189),
// which build one Python object per row.
//
// The file body (after the header) is copied into HBM once and parsed there:
//   1. term_count_kernel / term_write_kernel: line terminators ('\n', '\r\n', lone '\r',
//      as the csv module with newline='' splits), per 4 KiB tile, positions written in
//      file order after a scan of the per-tile counts;
//   2. line_flag_kernel: a line is a row unless it is empty (csv yields [] -> skipped);
//      a scan of the flags gives each line its row index;
//   3. row_parse_kernel<T>: one thread per line splits on ',', converts every field with
//      numparse.cuh (Python float() syntax, correctly rounded) and writes the working
//      transform straight into the dataset's stream layout:
//        r_raw = r, mu_raw = d_N, x = r - d_N, D_j = d_j - d_N      (model.py:185-188)
//      Errors are reduced to the FIRST offending row with an atomicMin on
//      (line << 3 | kind), kinds ordered as the reference raises them within a row.
#pragma once

#include <stdint.h>

#include "numparse.cuh"

namespace cavi {
namespace ingest {

constexpr int kTile = 4096;        // bytes per scan tile
constexpr int kTileThreads = 256;  // 16 bytes per thread
constexpr int kMaxFields = 17;     // r + up to 16 networks

// error kinds, in the order the reference checks one row (cli.py:67-73, model.py:64-86)
enum : int {
  kErrFields = 0,    // UsageError: row has k fields, expected N+1
  kErrParseR = 1,    // ValueError from float(row[0])
  kErrParseD = 2,    // ValueError from np.array(row[1:], dtype=float)
  kErrNonfiniteD = 3,  // ExpressionProfile: profile contains non-finite entries
  kErrNonfiniteR = 4,  // RawRecord: expression reading must be finite
};

// any '"' in the body: such files go to the host reader (csv.reader's quoting rules span
// commas and line breaks, which the line-parallel split cannot see)
static __global__ void quote_any_kernel(const char* t, int64_t n, int* flag) {
  const int64_t n16 = n / 16;
  int hit = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = reinterpret_cast<const uint4*>(t)[i];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // SWAR: a zero byte of w ^ 0x22222222 is a quote
      const uint32_t x = w[k] ^ 0x22222222u;
      hit |= ((x - 0x01010101u) & ~x & 0x80808080u) != 0;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int64_t i = n16 * 16; i < n; ++i) hit |= t[i] == '"';
  if (__syncthreads_or(hit) && threadIdx.x == 0) atomicOr(flag, 1);
}

__device__ __forceinline__ bool is_term(const char* t, int64_t n, int64_t i) {
  const char c = t[i];
  return c == '\n' || (c == '\r' && (i + 1 >= n || t[i + 1] != '\n'));
}

__device__ __forceinline__ int tile_terms(const char* t, int64_t n, int64_t base, int lane16, bool* mine) {
  // this thread's 16 bytes: [base + 16*lane16, +16)
  int c = 0;
  const int64_t p = base + 16 * (int64_t)lane16;
  if (p < n) {
    const uint4 v = *reinterpret_cast<const uint4*>(t + p);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const char ch = (char)((w[k >> 2] >> (8 * (k & 3))) & 0xFF);
      bool m = false;
      if (p + k < n) {
        if (ch == '\n') m = true;
        else if (ch == '\r') m = (p + k + 1 >= n) || t[p + k + 1] != '\n';
      }
      mine[k] = m;
      c += m;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k) mine[k] = false;
  }
  return c;
}

__global__ void __launch_bounds__(kTileThreads) term_count_kernel(const char* t, int64_t n, int64_t* tile_count) {
  __shared__ int s_sum[kTileThreads / 32];
  const int64_t tile = blockIdx.x;
  bool mine[16];
  int c = tile_terms(t, n, tile * kTile, threadIdx.x, mine);
  for (int off = 16; off; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
  if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t s = 0;
    for (int w = 0; w < kTileThreads / 32; ++w) s += s_sum[w];
    tile_count[tile] = s;
  }
}

__global__ void __launch_bounds__(kTileThreads) term_write_kernel(const char* t, int64_t n, const int64_t* tile_base,
                                                                   int64_t* term) {
  __shared__ int s_warp[kTileThreads / 32];
  const int64_t tile = blockIdx.x;
  bool mine[16];
  const int c = tile_terms(t, n, tile * kTile, threadIdx.x, mine);
  // block-wide exclusive scan of c in thread order (= byte order)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = c;
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += y;
  }
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  int before = 0;
  for (int w = 0; w < warp; ++w) before += s_warp[w];
  int64_t o = tile_base[tile] + before + inc - c;
  const int64_t p = tile * kTile + 16 * (int64_t)threadIdx.x;
#pragma unroll
  for (int k = 0; k < 16; ++k)
    if (mine[k]) term[o++] = p + k;
}

// line l spans [start, end): start = term[l-1] + 1, end = term[l] minus a '\r' of "\r\n"
__device__ __forceinline__ void line_span(const char* t, const int64_t* term, int64_t l, int64_t* s, int64_t* e) {
  const int64_t a = l ? term[l - 1] + 1 : 0;
  int64_t b = term[l];
  if (t[b] == '\n' && b > a && t[b - 1] == '\r') --b;
  *s = a;
  *e = b;
}

__global__ void line_flag_kernel(const char* t, const int64_t* term, int64_t L, int64_t* flag) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  int64_t s, e;
  line_span(t, term, l, &s, &e);
  flag[l] = e > s ? 1 : 0;
}

// a field as the csv module hands it to float(): "..." quoting removed when it wraps the field
__device__ __forceinline__ void unquote(const char*& s, const char*& e) {
  if (e - s >= 2 && *s == '"' && e[-1] == '"') {
    ++s;
    --e;
  }
}

template <typename T>
__global__ void row_parse_kernel(const char* t, const int64_t* term, const int64_t* rowidx, int64_t L, int N,
                                 int64_t Vp, double* r_raw, double* mu_raw, T* xs, T* Ds,
                                 unsigned long long* err_key, int64_t* slow, unsigned long long* slow_n,
                                 int64_t slow_cap) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  int64_t a, b;
  line_span(t, term, l, &a, &b);
  if (b <= a) return;  // blank line: no row
  const char* s = t + a;
  const char* e = t + b;
  // field count first (the reference checks len(row) before converting)
  int nf = 1;
  for (const char* p = s; p < e; ++p) nf += *p == ',';
  auto report = [&](int kind) { atomicMin(err_key, ((unsigned long long)l << 3) | (unsigned long long)kind); };
  if (nf != N + 1) {
    report(kErrFields);
    return;
  }
  double v[kMaxFields];
  int bad_r = 0, bad_d = 0, slow_any = 0;
  const char* fs = s;
  for (int f = 0; f <= N; ++f) {
    const char* fe = fs;
    while (fe < e && *fe != ',') ++fe;
    const char* qs = fs;
    const char* qe = fe;
    unquote(qs, qe);
    const int st = num::parse_double(qs, qe, &v[f]);
    if (st == num::kParseBad) {
      if (f == 0) bad_r = 1;
      else bad_d = 1;
    } else if (st == num::kParseSlow) {
      slow_any = 1;
    }
    fs = fe + 1;
  }
  if (bad_r) return report(kErrParseR);
  if (slow_any) {  // > 19 significant digits at a rounding boundary: the host converts this row
    const unsigned long long k = atomicAdd(slow_n, 1ull);
    if ((int64_t)k < slow_cap) slow[k] = l;
    return;
  }
  if (bad_d) return report(kErrParseD);
  bool fin_d = true;
  for (int j = 1; j <= N; ++j) fin_d &= isfinite(v[j]);
  if (!fin_d) return report(kErrNonfiniteD);
  if (!isfinite(v[0])) return report(kErrNonfiniteR);
  const int64_t row = rowidx[l];
  const double mu = v[N];
  r_raw[row] = v[0];
  mu_raw[row] = mu;
  xs[row] = (T)__dsub_rn(v[0], mu);
  for (int j = 0; j < N - 1; ++j) Ds[(int64_t)j * Vp + row] = (T)__dsub_rn(v[1 + j], mu);
}

}  // namespace ingest
}  // namespace cavi
