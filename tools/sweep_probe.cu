// sweep_probe.cu -- clock64 cycles of the tail's rate inversion (spd_sweep_warp /
// ref_inv_once_warp / the serial ref_inv_once_t) on one warp, cold and warm, per d.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 --expt-relaxed-constexpr \
//        -I/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/include -o /tmp/sweep_probe tools/sweep_probe.cu
#include <cstdio>
#include "../paper_2401_10068_b200/csrc/tail.cuh"

using namespace cavi;

// rolled symmetric sweep with register rotation: after each pivot every lane rotates its column
// half left by one, so the pivot's column is always register 0 (static index, no selects)
template <int D>
__device__ bool sweep_rot(const double* A, double* Ainv, double* logabs, int lane) {
  constexpr int H = (D + 1) / 2;
  const int r = lane & 15, h = lane >> 4;
  double w[H];
#pragma unroll
  for (int t = 0; t < H; ++t) {
    const int j = h * H + t;
    w[t] = (r < D && j < D) ? A[r * D + j] : 0.0;
  }
  double prod = 1.0;
  int ex = 0;
#pragma unroll 1
  for (int k = 0; k < D; ++k) {
    const int hk = k >= H ? 1 : 0;
    const int rot = k % H;  // rotations done so far within the cycle: register t holds column (t + rot) % H
    const double p = __shfl_sync(0xffffffffu, w[0], k + 16 * hk);
    const double wik = __shfl_sync(0xffffffffu, w[0], r + 16 * hk);
    double wkj[H];
#pragma unroll
    for (int t = 0; t < H; ++t) wkj[t] = __shfl_sync(0xffffffffu, w[t], k + 16 * h);
    if (!(p > 0.0)) return false;
    const double rp = 1.0 / p;
#pragma unroll
    for (int t = 0; t < H; ++t) {
      int c = t + rot;
      c = c >= H ? c - H : c;
      const int j = h * H + c;
      const double gen = fma(-wik * rp, wkj[t], w[t]);
      const double rowcol = (r == k ? wkj[t] : wik) * rp;
      w[t] = (r == k && j == k) ? -rp : ((r == k || j == k) ? rowcol : gen);
    }
    // rotate left by one
    const double w0 = w[0];
#pragma unroll
    for (int t = 0; t + 1 < H; ++t) w[t] = w[t + 1];
    w[H - 1] = w0;
    if (lane == 0) {
      prod *= p;
      const int hi = __double2hiint(prod);
      ex += ((hi >> 20) & 0x7ff) - 1023;
      prod = __hiloint2double((hi & 0x800fffff) | 0x3ff00000, __double2loint(prod));
    }
  }
  const int rot = D % H;
#pragma unroll
  for (int t = 0; t < H; ++t) {
    int c = t + rot;
    c = c >= H ? c - H : c;
    const int j = h * H + c;
    if (r < D && j < D) Ainv[r * D + j] = -w[t];
  }
  if (lane == 0) *logabs = log(prod) + (double)ex * kLn2;
  __syncwarp();
  return true;
}

template <int D>
__global__ void __launch_bounds__(32, 1) probe(const double* A, double* out, long long* cyc) {
  __shared__ double sA[D * D], sW[2 * D * D], sI[D * D];
  const int lane = threadIdx.x;
  for (int e = lane; e < D * D; e += 32) sA[e] = A[e];
  __syncwarp();
  double ld = 0;
  for (int rep = 0; rep < 3; ++rep) {
    long long t0 = clock64();
    bool ok = spd_sweep_warp<D>(sA, sW, sI, &ld, lane);
    long long t1 = clock64();
    bool ok2 = sweep_rot<D>(sA, sW, &ld, lane);
    long long t2 = clock64();
    if (lane == 0) {
      cyc[rep * 2] = t1 - t0;
      cyc[rep * 2 + 1] = t2 - t1;
      out[0] = ld + ok + ok2;
      double md = 0;
      for (int e = 0; e < D * D; ++e) md = fmax(md, fabs(sI[e] - sW[e]) / fmax(fabs(sI[e]), 1e-300));
      out[1] = md;
    }
  }
}

template <int D>
__global__ void __launch_bounds__(32, 1) probe_tail(const double* A, double* out, long long* cyc) {
  __shared__ TailSm<D> sm;
  const int lane = threadIdx.x;
  for (int rep = 0; rep < 3; ++rep) {
    for (int e = lane; e < D * D; e += 32) sm.C[e] = A[e];
    __syncwarp();
    double l = 0.0;
    long long t0 = clock64();
    const bool ok = tail_inverse<D>(sm, &l, lane);
    long long t1 = clock64();
    if (lane == 0) {
      cyc[rep] = t1 - t0;
      out[0] = l + ok;
    }
  }
}

__global__ void stream_kernel(const double4* x, size_t n, double* out) {
  double acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double4 v = x[i];
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1.2345) out[0] = acc;
}

template <int D>
void run_tail(const double* h) {
  double *A, *out;
  long long* cyc;
  cudaMalloc(&A, D * D * 8);
  cudaMalloc(&out, 8);
  cudaMallocManaged(&cyc, 6 * sizeof(long long));
  cudaMemcpy(A, h, D * D * 8, cudaMemcpyHostToDevice);
  probe_tail<D><<<1, 32>>>(A, out, cyc);
  cudaDeviceSynchronize();
  printf("d=%2d tail_inverse on TailSm: %6lld %6lld %6lld\n", D, cyc[0], cyc[1], cyc[2]);
  const size_t n = (size_t)1 << 28;  // 8 GB
  double4* big;
  if (cudaMalloc(&big, n * sizeof(double4)) == cudaSuccess) {
    cudaMemset(big, 0, n * sizeof(double4));
    for (int rep = 0; rep < 3; ++rep) {
      stream_kernel<<<148 * 8, 256>>>(big, n, out);
      probe_tail<D><<<1, 32>>>(A, out, cyc);
      cudaDeviceSynchronize();
      printf("d=%2d tail_inverse right after an 8 GB stream: %6lld %6lld %6lld\n", D, cyc[0], cyc[1], cyc[2]);
    }
    cudaFree(big);
  }
}

template <int D>
void run(double scale) {
  double h[D * D];
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j) h[i * D + j] = scale * ((i == j ? D + 1.0 : 0.0) + 1.0 / (1.0 + i + j));
  double *A, *out;
  long long* cyc;
  cudaMalloc(&A, sizeof h);
  cudaMalloc(&out, 16);
  cudaMallocManaged(&cyc, 6 * sizeof(long long));
  cudaMemcpy(A, h, sizeof h, cudaMemcpyHostToDevice);
  probe<D><<<1, 32>>>(A, out, cyc);
  cudaDeviceSynchronize();
  printf("scale %g d=%2d sweep cold %6lld warm %6lld %6lld | rotated cold %6lld warm %6lld %6lld\n", scale, D, cyc[0], cyc[2], cyc[4],
         cyc[1], cyc[3], cyc[5]);
}

int main(int argc, char** argv) {
  if (argc > 1) {  // a d = 15 rate matrix from a file (raw float64)
    double h[15 * 15];
    FILE* f = fopen(argv[1], "rb");
    if (!f || fread(h, sizeof(double), 225, f) != 225) return 1;
    fclose(f);
    double *A, *out;
    long long* cyc;
    cudaMalloc(&A, sizeof h);
    cudaMalloc(&out, 16);
    cudaMallocManaged(&cyc, 6 * sizeof(long long));
    cudaMemcpy(A, h, sizeof h, cudaMemcpyHostToDevice);
    probe<15><<<1, 32>>>(A, out, cyc);
    cudaDeviceSynchronize();
    run_tail<15>(h);
    double o2[2];
    cudaMemcpy(o2, out, 16, cudaMemcpyDeviceToHost);
    printf("rotated vs sweep max rel diff %g\n", o2[1]);
    printf("file d=15 sweep cold %6lld warm %6lld %6lld | rotated cold %6lld warm %6lld %6lld\n", cyc[0], cyc[2], cyc[4],
           cyc[1], cyc[3], cyc[5]);
    return 0;
  }
  for (double scale : {1.0, 1e6, 1e12}) {
    run<4>(scale);
    run<9>(scale);
    run<15>(scale);
  }
  return 0;
}
