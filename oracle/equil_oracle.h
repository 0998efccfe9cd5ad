/*
 * equil_oracle.h -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * This header and equil_oracle.c are the parity checker for the B200 product
 * (paper_1602_06621_b200/).  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  It is never
 * linked into, or called by, the product library.
 *
 * Every function restates one reference routine; the file:line it follows is
 * given beside it (paths relative to the reference's proj/ tree).
 *
 * The three operations the reference delegates to Eigen (which is absent in
 * this image) are defined here once, as a
 * numerics contract that the CUDA kernels restate independently:
 *   eo_det_exp        -- Eigen .array().exp()      (src/equilibrate.cpp:162-163,203-204)
 *   eo_canon_sum      -- Eigen .norm()/.dot()/...  (src/lsqr.cpp:23,26,40,50,97,131)
 *   eo_dense_rowdot / eo_dense_coldot -- Eigen dense GEMV (src/explicit_matrix.cpp:69,84)
 * Parity of those three is "shim-defined".
 */
#ifndef EQUIL_ORACLE_H
#define EQUIL_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG: src/rng.cpp:9-64, include/equil/rng.hpp:15-44 ------------------ */
typedef struct {
  uint64_t mt[312];
  int mti;
  double spare;
  int has_spare;
} eo_rng;

void eo_rng_init(eo_rng* r, uint64_t seed, uint64_t stream); /* rng.cpp:19-27 */
uint64_t eo_rng_next_u64(eo_rng* r);                         /* rng.cpp:29 */
double eo_rng_uniform01(eo_rng* r);                          /* rng.cpp:31-34 */
double eo_rng_sign(eo_rng* r);                               /* rng.cpp:36 */
double eo_rng_normal(eo_rng* r);                             /* rng.cpp:38-49 */
uint64_t eo_rng_uniform_index(eo_rng* r, uint64_t n);        /* rng.cpp:51-57 */
/* Standard-seeded mt19937_64 (seed(v)), for the C++ standard's KAT. */
void eo_mt64_seed(eo_rng* r, uint64_t v);
/* Seeding of SeededRng: the splitmix64-mixed value handed to mt19937_64. */
uint64_t eo_mixed_seed(uint64_t seed, uint64_t stream);
/* Raw 312-word state right after seeding (before the first twist). */
void eo_rng_state(uint64_t seed, uint64_t stream, uint64_t* out312);
/* Outputs [start, start+count) of SeededRng(seed, stream).next_u64(). */
void eo_raw_outputs(uint64_t seed, uint64_t stream, uint64_t start,
                    uint64_t count, uint64_t* out);
/* Sign bits of outputs [start, start+count): bit k of the packed little-endian
 * u32 words is 1 iff output (start+k) has its MSB set (sign() == +1.0). */
void eo_sign_bits(uint64_t seed, uint64_t stream, uint64_t start,
                  uint64_t count, uint32_t* bits_out);

/* ---- numerics contract (shim-defined, see header comment) ----------------- */
double eo_det_exp(double x);
double eo_canon_sum(const double* p, int64_t len);     /* sum, canonical tree */
double eo_canon_sumsq(const double* p, int64_t len);   /* sum of squares */
double eo_canon_dot(const double* a, const double* b, int64_t len);

/* ---- matrix store: src/explicit_matrix.cpp ------------------------------- */
/* CSR of A^T exactly as ExplicitMatrix::transposed() (:117-125) builds it. */
void eo_csr_transpose(int64_t m, int64_t n, const int64_t* row_ptr,
                      const int32_t* col, const double* val, int64_t* t_row_ptr,
                      int32_t* t_col, double* t_val);
/* y = A x, sparse (:67-79) */
void eo_csr_apply(int64_t m, const int64_t* row_ptr, const int32_t* col,
                  const double* val, const double* x, double* y);
/* x = A^T y as the reference's ascending-row scatter (:81-93) */
void eo_csr_apply_adjoint(int64_t m, int64_t n, const int64_t* row_ptr,
                          const int32_t* col, const double* val,
                          const double* y, double* x);
/* dense row-major A (m x n): y = A x and x = A^T y in the canonical order */
void eo_dense_apply(int64_t m, int64_t n, const double* A, const double* x,
                    double* y);
void eo_dense_apply_adjoint(int64_t m, int64_t n, const double* A,
                            const double* y, double* x);

/* ---- params: src/params.cpp:7-44 ----------------------------------------- */
typedef struct {
  double alpha, beta, gamma, max_log_scale;
  int iterations;
  uint64_t seed;
} eo_params;

/* returns 0 ok, 1 = invalid_argument (message in eo_last_error()) */
int eo_resolve_targets(const eo_params* p, int64_t m, int64_t n, double* alpha,
                       double* beta);
int eo_validate_params(const eo_params* p);
const char* eo_last_error(void);

/* ---- operator: CSR (dense==NULL) or dense row-major (row_ptr==NULL) ------- */
typedef struct {
  int64_t m, n;
  const int64_t* row_ptr;
  const int32_t* col;
  const double* val;
  const double* dense; /* row-major m x n, or NULL */
} eo_matrix;

/* ---- SGD engine: src/equilibrate.cpp:79-221 ------------------------------ */
typedef struct {
  double* u;
  double* v;
  double* d;
  double* e;
  double alpha, beta;
  int box_feasible, iterate_bound_ok;
  long long apply_count, adjoint_count;
  /* history: iter 0 and every stride (src/equilibrate.cpp:174-195); arrays
   * sized >= iterations/stride + 1 by the caller, or NULL when stride == 0. */
  int* hist_iter;
  double* hist_objective;
  double* hist_rms;
  int hist_len;
  /* optional full trajectory dump: per-iteration x_u (m*T) and x_v (n*T) */
  double* traj_u;
  double* traj_v;
} eo_scaling;

/* sgd_equilibrate_targets (src/variants.cpp:105-118): r (m), c (n) */
int eo_sgd_equilibrate_targets(const eo_matrix* A, const double* r, const double* c,
                               const eo_params* p, int diag_stride, eo_scaling* out);
int eo_sgd_equilibrate(const eo_matrix* A, const eo_params* p, int diag_stride,
                       eo_scaling* out);
/* sgd_equilibrate_symmetric (src/variants.cpp:35-103): square A, one scaling
 * u applied on both sides; symmetry spot check on stream 18 (:14-33). */
int eo_sgd_equilibrate_symmetric(const eo_matrix* A, const eo_params* p, int diag_stride,
                                 eo_scaling* out);
/* sgd_equilibrate_block (src/variants.cpp:156-240): row i shares u_{rb[i]},
 * column j shares v_{cb[j]}; R row blocks, C column blocks. */
int eo_sgd_equilibrate_block(const eo_matrix* A, const int64_t* rb, const int64_t* cb,
                             int64_t R, int64_t C, const eo_params* p, int diag_stride,
                             eo_scaling* out);

/* diagnostics at (u, v): src/equilibrate.cpp:10-22 and src/metrics.cpp:24-56 */
double eo_objective(const eo_matrix* A, const double* u, const double* v,
                    double alpha2, double beta2, double gamma);
double eo_rms_error(const eo_matrix* A, const double* u, const double* v,
                    double alpha, double beta);

/* ---- LSQR: src/lsqr.cpp:17-138 ------------------------------------------- */
typedef struct {
  double* x;                /* n */
  double* residual_history; /* capacity max_iters + 1 (+ T for preconditioned) */
  int hist_len;
  int iterations, equil_iterations, reached_tol, breakdown;
  long long apply_count, adjoint_count;
  double* d; /* optional (preconditioned): scaling used, m */
  double* e; /* optional (preconditioned): n */
} eo_lsqr_run;

int eo_lsqr(const eo_matrix* A, const double* b, int max_iters, double tol,
            eo_lsqr_run* out);
int eo_lsqr_preconditioned(const eo_matrix* A, const double* b,
                           const eo_params* p, int max_iters, double tol,
                           eo_lsqr_run* out);

/* stochastic_gradient_estimate (src/equilibrate.cpp:60-71): probes are outputs
 * [offset, offset + n + m) of SeededRng(seed, stream) */
int eo_stochastic_gradient_estimate(const eo_matrix* A, const double* u, const double* v,
                                    const eo_params* p, uint64_t seed, uint64_t stream,
                                    uint64_t offset, double* g_u, double* g_v);

/* ---- spectral_norm (src/lsqr.cpp:140-163) and the Chambolle-Pock lasso
 * (src/ccp.cpp:28-160) --------------------------------------------------- */
int eo_spectral_norm(const eo_matrix* A, int max_iters, double rel_tol, uint64_t seed,
                     double* out);
double eo_lasso_objective(const eo_matrix* A, const double* b, double lambda, const double* x);
typedef struct {
  int max_iters;
  double tau, sigma, theta; /* tau, sigma <= 0: auto 0.9 / |K|_2 */
  double p_star;            /* NaN: no gap history */
  double gap_tol;
} eo_ccp_options;
typedef struct {
  double* x;        /* n */
  double* obj_hist; /* capacity max_iters + 1 (+ T) */
  double* gap_hist; /* same capacity, or NULL */
  int hist_len, gap_len;
  double tau, sigma, theta;
  int iterations, equil_iterations, reached_tol;
  long long apply_count, adjoint_count;
} eo_ccp_run;
int eo_ccp_lasso(const eo_matrix* A, const double* b, double lambda, const eo_ccp_options* o,
                 eo_ccp_run* out);
int eo_ccp_lasso_preconditioned(const eo_matrix* A, const double* b, double lambda,
                                const eo_params* p, const eo_ccp_options* o, eo_ccp_run* out);

#ifdef __cplusplus
}
#endif

#endif
