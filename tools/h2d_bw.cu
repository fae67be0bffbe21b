// h2d_bw.cu -- pinned host -> device copy bandwidth for a 4 GB upload (the e2e call's H2D):
// one cudaMemcpyAsync vs the same bytes in 64 MiB pieces over 1, 2 and 4 streams.
//   nvcc -O3 -o /tmp/h2d_bw tools/h2d_bw.cu
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

int main() {
  const size_t bytes = (size_t)4 << 30, piece = (size_t)64 << 20;
  void *h, *d;
  if (cudaMallocHost(&h, bytes) != cudaSuccess || cudaMalloc(&d, bytes) != cudaSuccess) return 1;
  memset(h, 1, bytes);
  cudaStream_t s[4];
  for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int ns : {0, 1, 2, 4}) {
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(a, s[0]);
      if (ns == 0) {
        cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s[0]);
      } else {
        for (int i = 1; i < ns; ++i) cudaStreamWaitEvent(s[i], a, 0);
        for (size_t off = 0, k = 0; off < bytes; off += piece, ++k)
          cudaMemcpyAsync((char*)d + off, (char*)h + off, piece, cudaMemcpyHostToDevice, s[k % ns]);
        for (int i = 1; i < ns; ++i) {
          cudaEvent_t e;
          cudaEventCreate(&e);
          cudaEventRecord(e, s[i]);
          cudaStreamWaitEvent(s[0], e, 0);
        }
      }
      cudaEventRecord(b, s[0]);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%s %d stream(s): %.1f ms = %.1f GB/s\n", ns ? "64 MiB pieces," : "one copy,", ns ? ns : 1, best,
           bytes / (best * 1e-3) / 1e9);
  }
  return 0;
}
