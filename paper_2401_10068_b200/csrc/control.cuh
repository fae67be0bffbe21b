// control.cuh -- one-thread kernels around the fused pass (setup, generator
// hand-over, the multi-GPU tail).  Included by cavi.cu only.
#pragma once

#include "batched.cuh"

namespace cavi {

// One-CTA kernels around the pass --------------------------------------------
__global__ void setup_kernel(Hyp* h) {
  if (threadIdx.x == 0 && blockIdx.x == 0) hyp_setup(*h);
}

// Generator of the next pass from ctl->cur (used after a host-provided state).
__global__ void derive_kernel(const Hyp* h, Ctl* c) {
  if (threadIdx.x == 0 && blockIdx.x == 0) derive_pass_rt(*h, *c);
}

// Set the generator of vb_init's state (K0, Lambda0, e_rho = 0).
__global__ void init_gen_kernel(const Hyp* h, Ctl* c) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const int d = h->d;
    for (int i = 0; i < d; ++i) c->pass.c[i] = h->K0[i];
    for (int i = 0; i < d * d; ++i) {
      c->pass.A[i] = h->L0[i];
      c->pass.Ainv[i] = h->L0inv[i];
    }
    c->pass.lnA = h->lnL0;
    c->pass.e_rho = 0.0;
    c->mode = MODE_INIT;
  }
}

// Set the generator of an arbitrary state's own moments (for vb_elbo of it).
__global__ void state_gen_kernel(Ctl* c, int d) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const cv_state& s = c->cur;
    for (int i = 0; i < d; ++i) c->pass.c[i] = s.gen_c[i];
    for (int i = 0; i < d * d; ++i) {
      c->pass.A[i] = s.gen_A[i];
      c->pass.Ainv[i] = s.gen_Ainv[i];
    }
    c->pass.lnA = s.gen_lnA;
    c->pass.e_rho = s.gen_e_rho;
  }
}

// EM: the generator of theta_0 = (K, Lambda, rho) given by the caller (em.py:112-114).
__global__ void em_init_kernel(Hyp* h, Ctl* c, const double* K, const double* Lam, double rho) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int d = h->d;
  double ld;
  for (int i = 0; i < d; ++i) c->pass.c[i] = K[i];
  for (int i = 0; i < d * d; ++i) c->pass.A[i] = Lam[i];
  if (!spd_inv_logdet_rt(Lam, c->pass.Ainv, &ld, d, h->wL, h->wJ, h->wM)) {
    c->status = CV_ERR_NUMERIC;
    c->done = 1;
    return;
  }
  c->pass.lnA = ld;
  c->pass.e_rho = rho;
  c->mode = MODE_EM;
}

// Per-fit hyperparameter constants and control blocks of a batched fit.
__global__ void batched_setup_kernel(const Hyp* base, Hyp* hyps, Ctl* ctls, const int64_t* offsets, int64_t n_fits,
                                     int max_iter, double rel_tol, int compute_elbo, double param_tol,
                                     double* traces) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n_fits) return;
  Hyp& h = hyps[f];
  h = *base;
  h.V = (double)(offsets[f + 1] - offsets[f]);
  hyp_setup(h);
  Ctl& c = ctls[f];
  c.max_iter = max_iter;
  c.rel_tol = rel_tol;
  c.param_tol = param_tol;
  c.compute_elbo = compute_elbo;
  c.tr_cap = max_iter;
  double* t = traces + (size_t)f * 4 * max_iter;
  c.tr_elbo = t;
  c.tr_dk = t + max_iter;
  c.tr_drho = t + 2 * (size_t)max_iter;
  c.tr_dlam = t + 3 * (size_t)max_iter;
  if (h.setup_status != CV_OK) {
    c.status = h.setup_status;
    c.done = 1;
  }
}

}  // namespace cavi
