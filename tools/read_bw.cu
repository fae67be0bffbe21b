// read_bw.cu -- the pure-read HBM ceiling the fused pass is compared against: a grid-stride
// 16-byte-load (ld.global.cs) reduction over 3.2 GB (the d=3 stream size), several unroll depths, best of 20.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/read_bw tools/read_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(256) rd(const double2* __restrict__ x, size_t n, double* out) {
  double acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(x + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
  }
  for (; i < n; i += stride) {
    const double2 v = __ldcs(x + i);
    acc += v.x + v.y;
  }
  if (acc == 1.2345) *out = acc;
}

template <int U>
void run(const double2* x, size_t n, double* out, int blocks_per_sm) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 20; ++r) {
    cudaEventRecord(a);
    rd<U><<<148 * blocks_per_sm, 256>>>(x, n, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r > 2 && ms < best) best = ms;
  }
  printf("unroll %d, %d CTAs/SM: %.3f ms = %.0f GB/s\n", U, blocks_per_sm, best, n * 16.0 / (best * 1e-3) / 1e9);
}

int main() {
  const size_t n = 200000000;  // 3.2 GB of 16-byte words
  double2* x;
  double* out;
  if (cudaMalloc(&x, n * sizeof(double2)) != cudaSuccess) return 1;
  cudaMalloc(&out, 8);
  cudaMemset(x, 0, n * sizeof(double2));
  for (int bps : {4, 8}) {
    run<1>(x, n, out, bps);
    run<2>(x, n, out, bps);
    run<4>(x, n, out, bps);
    run<8>(x, n, out, bps);
  }
  return 0;
}
