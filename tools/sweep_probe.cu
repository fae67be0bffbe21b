// sweep_probe.cu -- clock64 cycles of the tail's rate inversion (spd_sweep_warp /
// ref_inv_once_warp / the serial ref_inv_once_t) on one warp, cold and warm, per d.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 --expt-relaxed-constexpr \
//        -I/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/include -o /tmp/sweep_probe tools/sweep_probe.cu
#include <cstdio>
#include "../paper_2401_10068_b200/csrc/tail.cuh"

using namespace cavi;

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
    bool ok2 = ref_inv_once_warp<D>(sA, sW, sI, &ld, lane);
    long long t2 = clock64();
    if (lane == 0) {
      cyc[rep * 2] = t1 - t0;
      cyc[rep * 2 + 1] = t2 - t1;
      out[0] = ld + ok + ok2;
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
  cudaMalloc(&out, 8);
  cudaMallocManaged(&cyc, 6 * sizeof(long long));
  cudaMemcpy(A, h, sizeof h, cudaMemcpyHostToDevice);
  probe<D><<<1, 32>>>(A, out, cyc);
  cudaDeviceSynchronize();
  printf("scale %g d=%2d sweep cold %6lld warm %6lld %6lld | pivoted GJ cold %6lld warm %6lld %6lld\n", scale, D, cyc[0], cyc[2], cyc[4],
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
    cudaMalloc(&out, 8);
    cudaMallocManaged(&cyc, 6 * sizeof(long long));
    cudaMemcpy(A, h, sizeof h, cudaMemcpyHostToDevice);
    probe<15><<<1, 32>>>(A, out, cyc);
    cudaDeviceSynchronize();
    run_tail<15>(h);
    printf("file d=15 sweep cold %6lld warm %6lld %6lld | pivoted GJ cold %6lld warm %6lld %6lld\n", cyc[0], cyc[2], cyc[4],
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
