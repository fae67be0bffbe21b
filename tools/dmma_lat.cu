// dmma_lat.cu -- DMMA (mma.sync m8n8k4 f64) dependent-chain latency and per-SMSP issue
// interval, one warp (and 2-4 warps on one SM sub-partition set), for the pass kernel's
// accumulation-chain scheduling.   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/dmma_lat tools/dmma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int CH>
__global__ void chain(double* out, long long* cyc, double seed) {
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = seed * i;
  const double a = seed + threadIdx.x, b = seed - threadIdx.x;
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 256; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c[i], a, b);
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int CH>
void run(int warps) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMallocManaged(&cyc, 8);
  for (int r = 0; r < 2; ++r) chain<CH><<<1, 32 * warps>>>(out, cyc, 1e-3);
  cudaDeviceSynchronize();
  printf("chains/warp %d, warps/CTA %2d: %6.1f cycles per DMMA per warp (%s)\n", CH, warps, (double)*cyc / (256.0 * CH),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  run<1>(1);
  run<2>(1);
  run<4>(1);
  run<8>(1);
  run<1>(4);
  run<2>(4);
  run<1>(8);
  run<2>(8);
  run<4>(8);
  run<1>(16);
  return 0;
}
