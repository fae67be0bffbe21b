/*
 * cavi.h -- C ABI of the B200-native CAVI engine (libcavi.so).
 *
 * Drop-in boundary for the reference's variational path, `tissuemix.vb`
 * (reference pkg/src/tissuemix/vb.py:26-34 `__all__`).  The reference has no
 * FFI of its own (it is pure Python); these are the entry points a ctypes
 * binding of that module binds (paper_2401_10068_b200/_lib.py; INTEGRATION.md
 * shows the stub).  Plain pointers and sizes only; all host buffers are
 * borrowed for the duration of the call; every call is blocking and returns
 * a status code (CV_OK on success), with the message in cv_last_error().
 *
 *   cv_dataset_create    <- tissuemix.model.Dataset construction (model.py:89-123)
 *                           uploaded into HBM (one-time, per dataset)
 *   cv_dataset_generate  <- model.random_profiles + model.synth_generate
 *                           (model.py:224-270), Philox4x32-10 stream-exact
 *   cv_init              <- vb.vb_init (vb.py:82-111)
 *   cv_step              <- vb.vb_step (vb.py:129-198)  (+ vb_elbo of the result)
 *   cv_elbo              <- vb.vb_elbo (vb.py:216-304)
 *   cv_fit               <- vb.vb_fit  (vb.py:312-354)
 *   cv_materialize       <- the per-gene VbState fields mu_beta / lam_beta /
 *                           e_beta / e_bbt (vb.py:49-54), produced on demand
 *   cv_batched_fit       <- many independent vb_fit calls (config 4)
 *
 * Status codes map to the reference's exceptions (linalg.py:46-69):
 *   CV_ERR_NUMERIC   -> linalg.NumericError   (non-PD / singular after retry)
 *   CV_ERR_NONFINITE -> FloatingPointError    (non-finite input)
 *   CV_ERR_ARG       -> ValueError            (bad arguments)
 *   CV_ERR_CUDA      -> RuntimeError          (CUDA / NCCL failure)
 */
#ifndef CAVI_H
#define CAVI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CV_MAX_DIM 15 /* N <= 16 networks (d = N - 1) */
#define CV_MAX_D2 (CV_MAX_DIM * CV_MAX_DIM)

enum {
  CV_OK = 0,
  CV_ERR_NUMERIC = 1,
  CV_ERR_NONFINITE = 2,
  CV_ERR_ARG = 3,
  CV_ERR_CUDA = 4,
  CV_ERR_IMPROPER = 5, /* NumericError("Q(Lambda) is improper; dataset too small") */
  CV_ERR_FORMAT = 6,   /* cli.UsageError: malformed dataset file (header / field count) */
  CV_ERR_PEER = 7,     /* multi-GPU: a peer's statistics did not arrive within CAVI_PEER_TIMEOUT_S */
  CV_ERR_SINGULAR = 8  /* linalg.BatchItemError: a d <= 3 item with |det| < 1e-300 (vb_init's Lambda0) */
};

/* storage layouts of the measurement stream in HBM */
enum {
  CV_STORE_F64 = 0, /* x = r - mu and D as fp64 (exact) */
  CV_STORE_F32 = 1, /* x and D stored as fp32, fp64 math (the optional fp32 path) */
  CV_STORE_F32M = 2 /* fp32 storage and fp32 per-gene math, fp64 sums (d <= 7; fp64 math above) */
};

/* Prior constants (reference model.py:126-151).  Host pointers, borrowed. */
typedef struct cv_hyper {
  double a0, b0, q0;
  int32_t n0;
  int32_t d;
  const double* K0;      /* (d,) */
  const double* Lambda0; /* (d,d) row-major, SPD */
} cv_hyper;

/* A variational state (reference VbState, vb.py:39-66) minus the per-gene
 * arrays, which are a pure function of the dataset and the `gen_*` fields
 * ("generator": the expectations the sweep that produced the state used),
 * plus the sums the next sweep and the bound need.  Fixed-size, so it can be
 * checkpointed by value.  Matrices are row-major d x d inside the arrays. */
typedef struct cv_state {
  int32_t d;
  int32_t n_iter;      /* sweeps taken to reach this state (0 = vb_init) */
  int32_t status;      /* CV_OK or the error the producing call hit */
  int32_t elbo_status; /* CV_OK, or the error vb_elbo of this state raises */
  int64_t V;
  double a_rho, b_rho, e_rho;
  double k0k[CV_MAX_DIM];
  double lam0l_inv[CV_MAX_D2];
  double e_lam[CV_MAX_D2];
  double e_lamk[CV_MAX_DIM];
  double ln_det_lam0l_inv;
  double elbo;  /* vb_elbo(state) */
  double resid; /* sum_i (r-mu)^2 - 2(r-mu) D.E[b] + D.E[bb^T].D under this state */
  double gen_c[CV_MAX_DIM];
  double gen_A[CV_MAX_D2];    /* per-gene precision base: lam_beta_i = A + e_rho D D^T */
  double gen_Ainv[CV_MAX_D2];
  double gen_lnA;
  double gen_e_rho;
} cv_state;

typedef struct cv_dataset cv_dataset;
typedef struct cv_comm cv_comm;
typedef struct cv_batch cv_batch;

/* ---- library ---------------------------------------------------------- */
int32_t cv_abi_version(void);
const char* cv_last_error(void);
int32_t cv_device_count(int32_t* n);

/* ---- datasets (device-resident measurement streams) -------------------- */
/* Upload genes [0, V) of (r, mu, D) (D row-major (V, d)) to `device`.
 * `gene_lo`/`V_total` place this shard in a dataset of V_total genes
 * (gene_lo = 0, V_total = V for a whole dataset). */
int32_t cv_dataset_create(const double* r, const double* mu, const double* D, int64_t V, int32_t d,
                          int64_t gene_lo, int64_t V_total, int32_t storage, int32_t device,
                          cv_dataset** out);
/* Genes [gene_lo, gene_lo+V) of the dataset random_profiles(RngStream(seed), V_total, N) +
 * synth_generate(truth=(K, Lam, rho)) would produce, generated on the device. */
int32_t cv_dataset_generate(uint64_t seed, int64_t gene_lo, int64_t V, int64_t V_total, int32_t n_networks,
                            const double* K, const double* Lam, double rho, int32_t storage,
                            int32_t device, cv_dataset** out);
/* ---- dataset files ------------------------------------ */
/* cli.read_dataset_csv (cli.py:58-75) + model.transform (model.py:174-189): the file body
 * is copied to HBM and parsed there (one thread per line, Python float() syntax, correctly
 * rounded) straight into the dataset's stream layout.  Errors as the reference raises them
 * for the first offending row: CV_ERR_FORMAT (UsageError: header, field count) or
 * CV_ERR_ARG (ValueError: unparsable / non-finite value, no records).  A file holding any
 * quote character is read on the host with csv.reader's quoting rules instead (a field may
 * then contain commas and line breaks), with the same checks and messages. */
int32_t cv_dataset_load_csv(const char* path, int32_t storage, int32_t device, cv_dataset** out,
                            int32_t* n_networks);
/* Binary dataset files (SURVEY 8(f) row 2's binary loader): the working arrays r (V,), mu (V,),
 * D (V, d) as np.savez writes them (an uncompressed ZIP of '<f8' C-order .npy members, ZIP64
 * for members over 4 GiB), streamed into HBM through pinned buffers and transformed on the
 * device.  CV_ERR_FORMAT for anything else (compressed, other dtypes, missing members, shapes).
 * cv_npz_probe validates the file on the host only (V, d). */
int32_t cv_dataset_load_npz(const char* path, int32_t storage, int32_t device, cv_dataset** out,
                            int32_t* n_networks);
int32_t cv_npz_probe(const char* path, int64_t* V, int32_t* d);
/* cli.write_dataset_csv (cli.py:47-56): header r,d_1..d_N, rows repr(r), untransformed profile
 * (D_j + mu, mu), every value formatted exactly as Python's repr(float).  threads <= 0: all cores. */
int32_t cv_write_dataset_csv(const char* path, const double* r, const double* mu, const double* D, int64_t V,
                             int32_t d, int32_t threads);
/* test hooks: the shared decimal parser / repr formatter run on the host
 * (0 ok, 1 syntax error, 2 needs strtod; repr returns the length written, <= 32 chars) */
int32_t cv_parse_number_host(const char* s, int64_t n, double* out);
int32_t cv_format_repr(double x, char* out);
/* test hook: the host csv.reader restatement that files containing a quote character take
 * (quoted fields may span commas and lines): records of text[0..n) serialised into out as
 * 0x1d + fields separated by 0x1f (nothing for the empty record []), each record ended by
 * 0x1e; *used = bytes written (CV_ERR_ARG if cap is too small). */
int32_t cv_csv_records_host(const char* text, int64_t n, char* out, int64_t cap, int64_t* used);

/* Copy back x = r - mu, r, mu and D (row-major) of the shard; any pointer may be
 * NULL (r and mu exist for datasets made by create/generate/load_csv, which keep them). */
int32_t cv_dataset_download(cv_dataset* ds, double* x, double* r, double* mu, double* D);
int32_t cv_dataset_info(cv_dataset* ds, int64_t* V, int32_t* d, int64_t* gene_lo, int64_t* V_total,
                        int32_t* storage, int64_t* device_bytes);
void cv_dataset_destroy(cv_dataset* ds);

/* ---- multi-GPU (one process per GPU; NCCL over NVLink) ---------------- */
/* The dataset is split into 8 octants of whole 64x4096-gene groups; rank r of a
 * world of 1/2/4/8 owns octants [8r/world, 8(r+1)/world) (the gene range the
 * Python planner `dist.shard_ranges` computes).  Per sweep the ranks exchange
 * one n_stats(d)-double partial (ncclAllGather) and all run the identical tail,
 * so states, traces and stop decisions agree bit-for-bit on every rank, and
 * with the single-GPU result for any world size.  Every shard call (cv_init, cv_step,
 * cv_elbo, cv_fit, cv_em_*) begins with a collective (an NCCL allreduce used as a barrier
 * and to resync the fused exchange's sequence counter), so all ranks must make the same
 * shard calls in the same order, as with any NCCL collective. */
int32_t cv_nccl_unique_id(uint8_t* out /* 128 bytes */);
int32_t cv_comm_create(const uint8_t* id, int32_t rank, int32_t world, int32_t device, cv_comm** out);
void cv_comm_destroy(cv_comm* c);
/* 1 when the exchange is fused into the pass (peer stores into NCCL symmetric windows over
 * NVLink, checked by a collective self-test at cv_comm_create); 0: ncclAllGather per sweep.
 * CAVI_NO_LSA=1 forces the NCCL path; a world of one uses neither (CAVI_LSA_WORLD1=1: fused). */
int32_t cv_comm_fused(cv_comm* c);
/* Fault injection (tests): this rank skips publishing its partial `ahead` sweeps after the
 * next shard call's entry resync, so every rank's tail times out (CV_ERR_PEER after
 * CAVI_PEER_TIMEOUT_S).  The following shard call resyncs and runs normally. */
int32_t cv_comm_drop_publish(cv_comm* c, int32_t ahead);
int32_t cv_dataset_set_comm(cv_dataset* ds, cv_comm* comm);
/* Mark a shard as rank `rank` of `world` without a communicator (single-GPU
 * emulation of the multi-GPU reduction for tests) and return the shard's
 * octant-subtree statistics of the sweep that would follow state `st`:
 * out holds d + d(d+1)/2 + 3 doubles [g | G upper | R | Q | Ld]. */
int32_t cv_dataset_set_shard(cv_dataset* ds, int32_t rank, int32_t world);
int32_t cv_shard_stats(cv_dataset* ds, const cv_hyper* hp, const cv_state* st, double* out);

/* ---- the CAVI path --------------------------------------------------- */
int32_t cv_init(cv_dataset* ds, const cv_hyper* hp, cv_state* out);
int32_t cv_step(cv_dataset* ds, const cv_hyper* hp, const cv_state* in, cv_state* out);
int32_t cv_elbo(cv_dataset* ds, const cv_hyper* hp, const cv_state* st, double* elbo);
/* Trace arrays have room for max_iter entries; *n_iter receives the count. */
int32_t cv_fit(cv_dataset* ds, const cv_hyper* hp, int32_t max_iter, double rel_tol, int32_t compute_elbo,
               double param_tol, cv_state* out, double* tr_elbo, double* tr_dk, double* tr_drho,
               double* tr_dlam, int32_t* n_iter);
/* Per-gene moments of genes [lo, hi) of state `st`; any output may be NULL.
 * mu_beta (n,d), lam_beta (n,d,d), e_bbt (n,d,d), sigma = lam_beta^-1 (n,d,d) and the
 * expected squared residual resid (n) (EM's Sigma, M, S: em.py:22-29), n = hi - lo. */
int32_t cv_materialize(cv_dataset* ds, const cv_hyper* hp, const cv_state* st, int64_t lo, int64_t hi,
                       double* mu_beta, double* lam_beta, double* e_bbt, double* sigma, double* resid);

/* ---- EM point estimation on the same fused pass (reference em.py) ------- */
/* em_fit (em.py:97-124) from theta_0 = (K, Lam, rho): one pass per iteration yields the
 * marginal log-likelihood of theta_n (model.py:278-287) and the E-step sums for
 * theta_{n+1}.  Traces have room for max_iter entries (tr_K: max_iter x d). */
int32_t cv_em_fit(cv_dataset* ds, const double* K, const double* Lam, double rho, int32_t max_iter, double rel_tol,
                  double* K_out, double* Lam_out, double* rho_out, double* tr_loglik, double* tr_K, double* tr_rho,
                  int32_t* n_iter);
/* em_step (em.py:80-94): theta -> theta'; optionally Lambda^-1 and ll of the input theta. */
int32_t cv_em_step(cv_dataset* ds, const double* K, const double* Lam, double rho, double* K_out, double* Lam_out,
                   double* rho_out, double* Lam_inv_in, double* loglik_in);

/* ---- posterior summaries (reference analysis.py) -------- */
/* Per column of `cols` (C columns of n samples, column-major): out[c*10 + k] =
 * {mean, sd (ddof=1), bandwidth, mode, multimodal, q(qlo), q(qhi), trivial (sd == 0),
 *  grid lo, grid hi}.  bw[c] > 0 is an explicit bandwidth, else Scott's rule sd * scott
 * (scott = n ** (-1/5), analysis.py:69-71; zero variance -> CV_ERR_ARG).  range[2c..2c+1]
 * overrides the grid [min - 4h, max + 4h].  grid_n > 0 evaluates the density on
 * linspace(lo, hi, grid_n) (grid_out: C x grid_n, optional) and, with find_mode, the
 * grid argmax + near-tie flag + 3 golden-section steps (kde_mode, analysis.py:98-139). */
int32_t cv_kde_columns(const double* cols, int64_t n, int32_t C, const double* bw, double scott, double sqrt2pi,
                       double golden, int32_t grid_n, const double* range, double qlo, double qhi, int32_t find_mode,
                       int32_t device, double* out, double* grid_out);
/* kde_density (analysis.py:74-85) at m points. */
int32_t cv_kde_density(const double* samples, int64_t n, double h, double sqrt2pi, const double* x, int64_t m,
                       int32_t device, double* out);
/* summarize (analysis.py:147-188) of n posterior draws K (n x d), rho (n), Lambda (n x d x d,
 * optional): out[c*10 + k] as cv_kde_columns for the 2d+2 columns K_1..K_d, w_1..w_{d+1}
 * (full_weights), rho (trivial columns keep mode = first draw); lam_mean: d x d. */
int32_t cv_summarize(const double* K, const double* rho, const double* Lam, int64_t n, int32_t d, double bandwidth,
                     double scott, double sqrt2pi, double golden, double qlo, double qhi, int32_t device,
                     double* out, double* lam_mean);

/* ---- many independent fits (BASELINE config 4) --------------------------- */
/* vb_fit on each of n_fits datasets (genes [offsets[f], offsets[f+1]) of r, mu, D),
 * all with hyperparameters hp, on `device` (a group of 8 lanes per fit: genes split across
 * the group, the tail on its first lane).  cv_batch_run leaves the results in HBM, owned by
 * the returned handle, and writes each fit's sweep count to n_iter (optional, [n_fits]);
 * cv_batch_states copies the states of fits [lo, hi), cv_batch_traces their traces
 * ([hi-lo][4][max_iter] = elbo, delta_k0k, delta_rho, delta_lam per sweep, NaN past n_iter).
 * cv_batched_fit = run + copy everything + destroy (out: n_fits states; traces optional). */
int32_t cv_batch_run(const double* r, const double* mu, const double* D, const int64_t* offsets, int64_t n_fits,
                     int32_t d, const cv_hyper* hp, int32_t max_iter, double rel_tol, int32_t compute_elbo,
                     double param_tol, int32_t device, int32_t* n_iter, cv_batch** out);
int32_t cv_batch_states(cv_batch* b, int64_t lo, int64_t hi, cv_state* out);
int32_t cv_batch_traces(cv_batch* b, int64_t lo, int64_t hi, double* out);
void cv_batch_destroy(cv_batch* b);
int32_t cv_batched_fit(const double* r, const double* mu, const double* D, const int64_t* offsets, int64_t n_fits,
                       int32_t d, const cv_hyper* hp, int32_t max_iter, double rel_tol, int32_t compute_elbo,
                       double param_tol, int32_t device, cv_state* out, double* traces);

/* ---- posterior draws (vb_posterior_sample, vb.py:357-393) -------------- */
/* n joint draws of (K, Lambda, rho) from the fitted Q of a state with globals
 * (a_rho, b_rho, k0k, lam0l_inv), consuming the Philox stream (seed, stream_id)
 * from block `block0` exactly as the reference RngStream does; *block_end is the
 * stream position afterwards.  K_out (n,d), Lam_out (n,d,d), rho_out (n). */
int32_t cv_posterior_sample(uint64_t seed, uint64_t stream_id, uint64_t block0, int32_t d, int32_t n0, double q0,
                            int64_t V, double a_rho, double b_rho, const double* k0k, const double* lam0l_inv,
                            int64_t n, int32_t device, double* K_out, double* Lam_out, double* rho_out,
                            uint64_t* block_end);

/* test hook: the sweep tail's rate inversion (the reference's inverse_batched semantics --
 * adjugate with the |det| >= 1e-300 guard for d <= 3, pivoted elimination above -- with the
 * jitter-once retry) on one d x d matrix on `device`: *ok = 0 where the reference raises
 * NumericError after the retry; *logdet = ln|det| of the matrix inverted. */
int32_t cv_test_rate_inverse(const double* A, int32_t d, int32_t device, double* Ainv, double* logdet, int32_t* ok);

/* ---- pinned host memory (for end-to-end uploads at DMA speed) --------- */
int32_t cv_host_alloc(int64_t bytes, void** out);
void cv_host_free(void* p);

/* ---- measurement hooks (bench.py) ------------------------------------ */
/* Run `warmup` then `sweeps` CAVI sweeps (ELBO on, no stop rule) from `st`
 * on the dataset's stream; *ms_total = CUDA-event time of the timed sweeps run back to
 * back as the fit loop runs them; *ms_kernel = summed CUDA-event time of the fused-pass
 * kernels alone, from a second run of `sweeps` sweeps with events bracketing each pass. */
int32_t cv_bench_sweeps(cv_dataset* ds, const cv_hyper* hp, const cv_state* st, int32_t warmup,
                        int32_t sweeps, double* ms_total, double* ms_kernel, int32_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* CAVI_H */
