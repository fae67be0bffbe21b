// pass_inst.cu -- one explicit instantiation set of the fused pass per
// dimension; the Makefile compiles this file once per CAVI_D in 1..15 so the
// builds run in parallel.
#include "batched.cuh"
#include "posterior.cuh"

#ifndef CAVI_D
#error "compile with -DCAVI_D=<1..15>"
#endif

#define CAVI_CAT2(a, b) a##b
#define CAVI_CAT(a, b) CAVI_CAT2(a, b)

template <typename T, typename M = double>
static cavi::PassKernel make_kernel() {
  using G = cavi::Geometry<CAVI_D, T, M>;
  cavi::PassKernel k;
  k.fn = cavi::pass_kernel<CAVI_D, T, M>;
  k.threads = G::kCtaThreads;
  k.smem = G::kSmem;
  k.tail = cavi::tail_kernel<CAVI_D>;
  k.batched = cavi::batched_fit_kernel<CAVI_D>;
  k.rate_inverse_test = cavi::rate_inverse_test_kernel<CAVI_D>;
  k.wishart_seg = cavi::wishart_segment_kernel<CAVI_D>;
  k.wishart_fin = cavi::wishart_finish_kernel<CAVI_D>;
  cudaFuncSetAttribute((const void*)k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, k.smem);
  return k;
}

cavi::PassKernel CAVI_CAT(cavi_pass_d, CAVI_D)(int storage) {
  if (storage == CV_STORE_F32M) return make_kernel<float, float>();
  return storage == CV_STORE_F32 ? make_kernel<float>() : make_kernel<double>();
}
