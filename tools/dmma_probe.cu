// dmma_probe.cu -- measured FP64 tensor-core throughput of the mma.sync f64 shapes on
// this GPU (m8n8k4 vs the sm_90+ m16n8k4 / m16n8k8 / m16n8k16) and of scalar DFMA.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

__global__ void k_m8n8k4(double* out, double seed) {
  double c[kChains][2];
  for (int i = 0; i < kChains; ++i) c[i][0] = c[i][1] = seed * i;
  double a = seed + threadIdx.x, b = seed - threadIdx.x;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < kChains; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int i = 0; i < kChains; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_m16n8k4(double* out, double seed) {
  double c[kChains][4];
  for (int i = 0; i < kChains; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = seed * i;
  double a0 = seed + threadIdx.x, a1 = seed * 2, b = seed - threadIdx.x;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < kChains; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  double s = 0;
  for (int i = 0; i < kChains; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_m16n8k8(double* out, double seed) {
  double c[kChains][4];
  for (int i = 0; i < kChains; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = seed * i;
  double a0 = seed + threadIdx.x, a1 = seed * 2, a2 = seed * 3, a3 = seed * 4, b0 = seed - threadIdx.x, b1 = seed;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < kChains; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
          : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  double s = 0;
  for (int i = 0; i < kChains; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_m16n8k16(double* out, double seed) {
  double c[kChains][4];
  for (int i = 0; i < kChains; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = seed * i;
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = seed + i + threadIdx.x;
  for (int i = 0; i < 4; ++i) b[i] = seed - i;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < kChains; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
          "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
          : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
            "d"(b[1]), "d"(b[2]), "d"(b[3]));
  double s = 0;
  for (int i = 0; i < kChains; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double* out, double seed) {
  double c[kChains * 2];
  for (int i = 0; i < kChains * 2; ++i) c[i] = seed * i;
  const double a = seed + threadIdx.x, b = 0.999999;
  for (int it = 0; it < kIters * 4; ++it)
#pragma unroll
    for (int i = 0; i < kChains * 2; ++i) c[i] = fma(c[i], b, a);
  double s = 0;
  for (int i = 0; i < kChains * 2; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
void run(const char* name, K kern, double flops_per_warp_iter, int iters, int threads) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4;
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  kern<<<blocks, threads>>>(out, 1e-3);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(out, 1e-3);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = (double)blocks * threads / 32;
  const double flops = 5.0 * warps * iters * flops_per_warp_iter;
  printf("%-10s %8.2f TFLOP/s  (%s)\n", name, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  run("m8n8k4", k_m8n8k4, 2.0 * 8 * 8 * 4 * kChains, kIters, 256);
  run("m16n8k4", k_m16n8k4, 2.0 * 16 * 8 * 4 * kChains, kIters, 256);
  run("m16n8k8", k_m16n8k8, 2.0 * 16 * 8 * 8 * kChains, kIters, 256);
  run("m16n8k16", k_m16n8k16, 2.0 * 16 * 8 * 16 * kChains, kIters, 256);
  run("dfma", k_dfma, 2.0 * 32 * kChains * 2, kIters * 4, 256);
  return 0;
}
