// lat_probe.cu -- dependent-chain latencies seen by ONE warp (the sweep tail's regime: no other
// warps to hide behind): DFMA, DMUL, fp64 division, fp64 reciprocal via rcp + Newton, double
// shuffles, shared-memory load, log().
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/lat_probe tools/lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kN = 256;

__global__ void probe(double seed, double* out, long long* cyc) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  sm[lane] = seed + lane;
  sm[lane + 32] = seed - lane;
  __syncwarp();
  double x = seed + lane * 1e-3, acc = 0;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < kN; ++i) x = fma(x, 0.999999, 1e-7);
  t1 = clock64();
  if (lane == 0) cyc[0] = t1 - t0;
  acc += x;
  // division chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < kN; ++i) x = 1.0 / (x + 1.0);
  t1 = clock64();
  if (lane == 0) cyc[1] = t1 - t0;
  acc += x;
  // __drcp_rn chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < kN; ++i) x = __drcp_rn(x + 1.0);
  t1 = clock64();
  if (lane == 0) cyc[2] = t1 - t0;
  acc += x;
  // shuffle chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < kN; ++i) x = __shfl_sync(0xffffffffu, x, (lane + i) & 31) + 1e-9;
  t1 = clock64();
  if (lane == 0) cyc[3] = t1 - t0;
  acc += x;
  // shared load chain (address depends on the loaded value)
  int idx = lane;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < kN; ++i) idx = ((int)sm[idx & 63] + i) & 63;
  t1 = clock64();
  if (lane == 0) cyc[4] = t1 - t0;
  acc += idx;
  // log chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < kN; ++i) x = log(x + 2.0);
  t1 = clock64();
  if (lane == 0) cyc[5] = t1 - t0;
  acc += x;
  // DADD chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < kN; ++i) x = x + 1e-9;
  t1 = clock64();
  if (lane == 0) cyc[6] = t1 - t0;
  acc += x;
  // shared store -> load (same address) chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < kN; ++i) {
    sm[lane] = x;
    __syncwarp();
    x = sm[(lane + 1) & 31] + 1e-9;
    __syncwarp();
  }
  t1 = clock64();
  if (lane == 0) cyc[7] = t1 - t0;
  acc += x;
  // empty loop
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < kN; ++i) asm volatile("" ::: "memory");
  t1 = clock64();
  if (lane == 0) cyc[8] = t1 - t0;
  out[lane] = acc;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  const char* names[] = {"dfma", "ddiv", "drcp_rn", "shfl.f64", "lds", "log", "dadd", "sts->lds+2 syncwarp", "empty loop"};
  for (int rep = 0; rep < 3; ++rep) {
    probe<<<1, 32>>>(1.5, out, cyc);
    cudaDeviceSynchronize();
  }
  for (int i = 0; i < 9; ++i) printf("%-22s %7.1f cycles/iter\n", names[i], (double)cyc[i] / kN);
  return 0;
}
