/*
 * equil_b200.h -- C ABI of the B200 equilibration hot path (libequil_b200.so).
 *
 * Drop-in boundary for the reference's algorithm-level entry points
 * (SURVEY.md §8(b)).  Each function names the reference interface it replaces.
 * Plain pointers and sizes only; host pointers unless stated otherwise.
 * Reference paths are relative to the reference's proj/ tree.
 *
 * Error convention (include/equil/common.hpp:16-22): precondition failures
 * (detail::require -> std::invalid_argument) return EQUIL_EINVAL, runtime
 * failures (detail::check -> std::runtime_error) return EQUIL_ERUNTIME; CUDA /
 * NCCL / allocation failures have their own codes.  The message of the last
 * failure on the calling thread is available from equil_last_error().
 */
#ifndef EQUIL_B200_H
#define EQUIL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  EQUIL_OK = 0,
  EQUIL_EINVAL = 1,   /* std::invalid_argument */
  EQUIL_ERUNTIME = 2, /* std::runtime_error */
  EQUIL_ECUDA = 3,
  EQUIL_ENCCL = 4,
  EQUIL_ENOMEM = 5
} equil_status;

/* Opaque device-resident matrix: CSR(A), CSR(A^T) built on device, traversal
 * plans, workspaces.  Replaces ExplicitMatrix (include/equil/explicit_matrix.hpp:13-86)
 * as the operand of the entry points below. */
typedef struct equil_matrix equil_matrix;

/* EquilibrationParams (include/equil/params.hpp:14-23).  alpha/beta == 0 means
 * "auto" (src/params.cpp:7-33). */
typedef struct {
  double alpha;
  double beta;
  double gamma;
  double max_log_scale;
  int iterations;
  uint64_t seed;
} equil_params;

/* Device placement.  world_size > 1 row-shards A and A^T across one process per
 * GPU and all-gathers e.*s and d.*w with NCCL each iteration (SGD), and the
 * gathered LSQR vectors after every update (LSQR; norms are reduced over the
 * whole vector in global order, so every rank sees the single-GPU scalars);
 * nccl_id points to the 128-byte ncclUniqueId shared by all ranks (ignored
 * when world_size == 1).  Every rank calls every entry point collectively and
 * receives the full-length results. */
typedef struct {
  int device;
  int rank;
  int world_size;
  const void* nccl_id;
} equil_device_cfg;

/* DiagnosticsConfig (include/equil/equilibrate.hpp:63-67): history at t = 0
 * and every `stride` iterations; condition numbers are out of scope. */
typedef struct {
  int stride; /* 0 disables history */
  int want_objective;
  int want_rms;
} equil_diag_cfg;

/* ScalingResult (include/equil/equilibrate.hpp:69-78).  Caller-allocated
 * buffers; u,d have m entries and v,e n entries (full length on every rank).
 * hist_* have capacity hist_cap (>= iterations/stride + 1). */
typedef struct {
  double* u;
  double* v;
  double* d;
  double* e;
  int outputs_on_device; /* nonzero: u,v,d,e are device pointers */
  double alpha, beta;
  int box_feasible;
  int iterate_bound_ok;
  long long apply_count;
  long long adjoint_count;
  int* hist_iter;
  double* hist_objective;
  double* hist_rms;
  int hist_cap;
  int hist_len;
} equil_scaling_out;

/* LsqrRun (include/equil/lsqr.hpp:10-23).  x has n entries; residual_history
 * capacity residual_cap (>= max_iters + 1, + iterations for preconditioned). */
typedef struct {
  double* x;
  double* residual_history;
  int residual_cap;
  int hist_len;
  int iterations;
  int equil_iterations;
  int reached_tol;
  int breakdown;
  long long apply_count;
  long long adjoint_count;
} equil_lsqr_out;

/* ---- defaults / params (src/params.cpp) -------------------------------- */
void equil_params_default(equil_params* p); /* params.hpp:14-23 defaults */
/* resolve_targets (src/params.cpp:7-33) */
equil_status equil_resolve_targets(const equil_params* p, int64_t rows,
                                   int64_t cols, double* alpha, double* beta);
/* validate_params (src/params.cpp:35-44) */
equil_status equil_validate_params(const equil_params* p);

/* ---- matrix store ------------------------------------------------------- */
/* ExplicitMatrix::sparse (src/explicit_matrix.cpp:19-57) for input that is
 * already canonical CSR (rows ascending, columns strictly ascending): uploads,
 * validates on device, and builds CSR(A^T) on device bit-identically to
 * ExplicitMatrix::transposed() (:117-125).  Non-canonical input -> EINVAL. */
equil_status equil_matrix_create_csr(int64_t m, int64_t n, const int64_t* row_ptr,
                                     const int32_t* col, const double* val,
                                     const equil_device_cfg* cfg,
                                     equil_matrix** out);
/* ExplicitMatrix::sparse(rows, cols, entries) (src/explicit_matrix.cpp:19-57)
 * from COO triplets in any order, on device: range check in input order, sort
 * by (row, col), duplicate rejection in sorted order (same messages), CSR. */
equil_status equil_matrix_create_coo(int64_t m, int64_t n, int64_t nnz,
                                     const int64_t* rows, const int64_t* cols,
                                     const double* vals, const equil_device_cfg* cfg,
                                     equil_matrix** out);
/* ExplicitMatrix::dense (src/explicit_matrix.cpp:8-17); input row-major. */
equil_status equil_matrix_create_dense(int64_t m, int64_t n, const double* rowmajor,
                                       const equil_device_cfg* cfg,
                                       equil_matrix** out);
void equil_matrix_destroy(equil_matrix* A);
equil_status equil_matrix_shape(const equil_matrix* A, int64_t* m, int64_t* n,
                                int64_t* nnz);
/* read_matrix_market_file (include/equil/matrix_market.hpp:17-18,
 * src/matrix_market.cpp:63-204): real general coordinate or array files;
 * parse errors are EQUIL_ERUNTIME with the reference's message
 * "matrix market: line N: ...". */
equil_status equil_matrix_read_matrix_market(const char* path, const equil_device_cfg* cfg,
                                             equil_matrix** out);
/* write_matrix_market_file (include/equil/matrix_market.hpp:20-21,
 * src/matrix_market.cpp:209-243): "%.17g", byte-identical to the reference. */
equil_status equil_matrix_write_matrix_market(equil_matrix* A, const char* path);
/* Binary CSR ("EQBCSR01": int64 m, n, nnz, dense flag; row_ptr int64, col int32,
 * val f64 -- or m*n f64 row-major): fast reload path, no reference equivalent. */
equil_status equil_matrix_save_binary(equil_matrix* A, const char* path);
equil_status equil_matrix_load_binary(const char* path, const equil_device_cfg* cfg,
                                      equil_matrix** out);
/* CSR(A) (sparse) or row-major A (dense) back on the host; single GPU. */
equil_status equil_matrix_export_csr(equil_matrix* A, int64_t* row_ptr, int32_t* col,
                                     double* val);
equil_status equil_matrix_export_dense(equil_matrix* A, double* rowmajor);
int equil_matrix_is_dense(const equil_matrix* A);
/* Host-only Matrix Market access (no GPU needed): parse a file into an
 * opaque handle (entries 0-based in file order, with their line numbers; or a
 * dense row-major array), fetch, free; write a host CSR / dense array. */
equil_status equil_mm_parse(const char* path, int64_t* m, int64_t* n, int64_t* nnz, int* dense,
                            void** handle);
equil_status equil_mm_fetch(void* handle, int64_t* rows, int64_t* cols, double* vals,
                            int64_t* lines);
void equil_mm_free(void* handle);
equil_status equil_mm_write_csr(const char* path, int64_t m, int64_t n, const int64_t* row_ptr,
                                const int32_t* col, const double* val);
equil_status equil_mm_write_dense(const char* path, int64_t m, int64_t n,
                                  const double* rowmajor);
/* The cudaStream_t all work on this handle is issued on (for event timing). */
void* equil_matrix_stream(equil_matrix* A);
/* Device time (CUDA events on the handle's stream) of the T-iteration loop of
 * the last equil_sgd_equilibrate call; *iterations receives T. */
double equil_last_loop_ms(equil_matrix* A, int* iterations);
/* How the SGD loop of a sharded handle exchanges the next gathered vectors:
 * 0 single GPU / not yet negotiated, 1 padded all-gathers (NCCL or host
 * exchange), 2 fused peer stores from the SGD epilogue + one-word barrier. */
int equil_exchange_mode(const equil_matrix* A);
/* How the SGD passes traverse the rows of A longer than 512 entries: 0 the
 * warp-specialised long-slice kernel (or no such rows), 1 the column sweep
 * (one persistent CTA per SM, gathered vector in shared-memory panels).  No
 * reference counterpart (the result is the same bit for bit). */
int equil_sweep_active(const equil_matrix* A);
/* Number of this library's kernels launched so far in the process. */
long long equil_kernel_launches(void);
/* Build flags of the loaded library: bit 0 = checked build (EQ_CHECK device
 * assertions, libequil_b200_checked.so).  No reference counterpart. */
int equil_build_flags(void);

/* LinearOperator::apply / apply_adjoint (include/equil/linop.hpp:13-25,
 * src/explicit_matrix.cpp:67-93): y = A x or x = A^T y, host vectors. */
equil_status equil_apply(equil_matrix* A, const double* x, double* y, int adjoint);

/* ---- the hot path -------------------------------------------------------- */
/* sgd_equilibrate(op, params, diag) (include/equil/equilibrate.hpp:89-91,
 * src/equilibrate.cpp:138-221).  diag may be NULL. */
equil_status equil_sgd_equilibrate(equil_matrix* A, const equil_params* p,
                                   const equil_diag_cfg* diag,
                                   equil_scaling_out* out);
/* sgd_equilibrate_targets(op, r, c, params, diag) (include/equil/variants.hpp:24-27,
 * src/variants.cpp:105-118): per-row squared-norm targets r (m entries) and
 * per-column targets c (n entries), positive, sum(r) == sum(c) to 1e-8; the
 * same engine with per-coordinate linear terms (history: objective only). */
equil_status equil_sgd_equilibrate_targets(equil_matrix* A, const double* r, const double* c,
                                           const equil_params* p, const equil_diag_cfg* diag,
                                           equil_scaling_out* out);
/* sgd_equilibrate_symmetric(op, params, diag) (include/equil/variants.hpp:16-18,
 * src/variants.cpp:35-103): square symmetric A, one scaling u = v on both
 * sides, one apply and no adjoint per iteration; the symmetry spot check of
 * :14-33 runs first.  Single GPU. */
equil_status equil_sgd_equilibrate_symmetric(equil_matrix* A, const equil_params* p,
                                             const equil_diag_cfg* diag,
                                             equil_scaling_out* out);
/* sgd_equilibrate_block(op, BlockStructure, params, diag)
 * (include/equil/variants.hpp:30-50, src/variants.cpp:120-240): row i shares
 * u_{row_block[i]}, column j shares v_{col_block[j]}; results expanded to full
 * length.  Single GPU. */
equil_status equil_sgd_equilibrate_block(equil_matrix* A, const int64_t* row_block,
                                         const int64_t* col_block, int64_t row_blocks,
                                         int64_t col_blocks, const equil_params* p,
                                         const equil_diag_cfg* diag, equil_scaling_out* out);
/* CcpOptions / CcpRun (include/equil/ccp.hpp:24-48).  tau, sigma <= 0 select
 * the automatic 0.9 / |K|_2; p_star NaN disables the gap history.  Histories
 * are caller-allocated with capacity hist_cap >= max_iters + 1 (+ iterations
 * of the equilibration for the preconditioned run). */
typedef struct {
  int max_iters;
  double tau;
  double sigma;
  double theta;
  double p_star;
  double gap_tol;
} equil_ccp_options;
typedef struct {
  double* x; /* n */
  double* objective_history;
  double* gap_history; /* required when p_star is finite */
  int hist_cap;
  int hist_len;
  int gap_len;
  double tau, sigma, theta;
  int iterations;
  int equil_iterations;
  int reached_tol;
  long long apply_count;
  long long adjoint_count;
} equil_ccp_out;
/* ccp_lasso(LassoProblem{A, b, lambda}, options) (include/equil/ccp.hpp:57,
 * src/ccp.cpp:125-132): min |Ax - b|^2/sqrt(lambda) + sqrt(lambda)|x|_1.  Single GPU. */
equil_status equil_ccp_lasso(equil_matrix* A, const double* b, double lambda,
                             const equil_ccp_options* options, equil_ccp_out* out);
/* ccp_lasso_preconditioned (include/equil/ccp.hpp:65-67, src/ccp.cpp:134-141) */
equil_status equil_ccp_lasso_preconditioned(equil_matrix* A, const double* b, double lambda,
                                            const equil_params* p,
                                            const equil_ccp_options* options,
                                            equil_ccp_out* out);
/* spectral_norm(op, max_iters, rel_tol, seed) (include/equil/lsqr.hpp:44-48,
 * src/lsqr.cpp:140-163): power iteration, normals on stream 19. */
equil_status equil_spectral_norm(equil_matrix* A, int max_iters, double rel_tol, uint64_t seed,
                                 double* out);
/* lasso_objective(LassoProblem{A, b, lambda}, x) (include/equil/ccp.hpp:21,
 * src/ccp.cpp:115-123) */
equil_status equil_lasso_objective(equil_matrix* A, const double* b, double lambda,
                                   const double* x, double* out);
/* Public helpers of include/equil/equilibrate.hpp:15-48 and metrics.hpp:14-15 on the
 * device matrix (single GPU; sparse, except the estimate).  u (m), v (n), lin_u (m),
 * lin_v (n), gradients are host arrays.  exp and whole-vector sums follow the
 * numerics contract, so objective / gradient / rms agree with the
 * reference to ~1e-12 relative; the estimate is bit-exact. */
equil_status equil_objective(equil_matrix* A, const double* u, const double* v,
                             const equil_params* p, double* out);
equil_status equil_objective_weighted(equil_matrix* A, const double* u, const double* v,
                                      const double* lin_u, const double* lin_v, double gamma,
                                      double* out);
equil_status equil_gradient(equil_matrix* A, const double* u, const double* v,
                            const equil_params* p, double* grad_u, double* grad_v);
equil_status equil_gradient_weighted(equil_matrix* A, const double* u, const double* v,
                                     const double* lin_u, const double* lin_v, double gamma,
                                     double* grad_u, double* grad_v);
/* stochastic_gradient_estimate(op, u, v, params, rng, g_u, g_v): the SeededRng is
 * (seed, stream) advanced by `offset` draws; the call consumes n + m draws. */
equil_status equil_stochastic_gradient_estimate(equil_matrix* A, const double* u,
                                                const double* v, const equil_params* p,
                                                uint64_t seed, uint64_t stream, uint64_t offset,
                                                double* g_u, double* g_v);
equil_status equil_rms_error(equil_matrix* A, const double* u, const double* v, double alpha,
                             double beta, double* out);
equil_status equil_project_box(const double* x, int64_t n, double bound, double* out);
/* lsqr(op, b, max_iters, tol) (include/equil/lsqr.hpp:30-31, src/lsqr.cpp:85-103) */
equil_status equil_lsqr(equil_matrix* A, const double* b, int max_iters, double tol,
                        equil_lsqr_out* out);
/* lsqr_preconditioned(op, b, params, max_iters, tol)
 * (include/equil/lsqr.hpp:38-40, src/lsqr.cpp:105-138) */
equil_status equil_lsqr_preconditioned(equil_matrix* A, const double* b,
                                       const equil_params* p, int max_iters,
                                       double tol, equil_lsqr_out* out);

/* One-shot convenience for callers that only hold host CSR: create + equilibrate
 * + destroy (all host<->device traffic inside the call). */
equil_status equil_sgd_equilibrate_csr(int64_t m, int64_t n, const int64_t* row_ptr,
                                       const int32_t* col, const double* val,
                                       const equil_params* p,
                                       const equil_device_cfg* cfg,
                                       equil_scaling_out* out);

/* ---- matrix-free operators ------------------------------------------------
 * The reference's plugin interface is LinearOperator (include/equil/linop.hpp:
 * 13-25): rows(), cols(), apply(x), apply_adjoint(y).  On the device it is a
 * pair of callbacks: apply(ctx, x, y, stream) computes y = A x (x: cols
 * doubles, y: rows doubles, device pointers); apply_adjoint(ctx, y, x, stream)
 * computes x = A^T y.  They are called from the calling thread and must
 * enqueue their work on `stream` (a cudaStream_t) or finish it before
 * returning. */
typedef void (*equil_device_apply_fn)(void* ctx, const double* in, double* out, void* stream);
typedef struct {
  int64_t rows;
  int64_t cols;
  equil_device_apply_fn apply;
  equil_device_apply_fn apply_adjoint;
  void* ctx;
  int device;
} equil_device_operator;
/* sgd_equilibrate(op, params) on a matrix-free operator (include/equil/
 * equilibrate.hpp:89-91, src/equilibrate.cpp:138-221): T applies and T
 * adjoints of op, probes, estimate, update and averaging on the device.
 * Single GPU; no history (the reference needs the explicit matrix for it). */
equil_status equil_sgd_equilibrate_operator(const equil_device_operator* op,
                                            const equil_params* p, equil_scaling_out* out);
/* lsqr(op, b, max_iters, tol) (p == NULL) or lsqr_preconditioned(op, b, *p,
 * max_iters, tol) (src/lsqr.cpp:85-138) on a matrix-free operator: b and
 * out->x on the host; three operator calls per iteration (B v, B^T u and the
 * uncharged residual probe A x).  Single GPU. */
equil_status equil_lsqr_operator(const equil_device_operator* op, const double* b,
                                 const equil_params* p, int max_iters, double tol,
                                 equil_lsqr_out* out);
/* y = A x (adjoint: x = A^T y) on device pointers, ordered on `stream`:
 * an explicit matrix's own traversal, usable as a device operator
 * (LinearOperator::apply / apply_adjoint, include/equil/linop.hpp:20-24). */
equil_status equil_apply_device(equil_matrix* A, const double* x, double* y, int adjoint,
                                void* stream);

/* ---- verification hooks -------------------------------------------------- */
/* Sign bits of SeededRng(seed, stream) outputs [start, start+count), generated
 * on device (K1); bit k of the packed u32 words = MSB of output start+k. */
equil_status equil_sign_bits(uint64_t seed, uint64_t stream, uint64_t start,
                             uint64_t count, uint32_t* bits_out, int device);
/* CSR(A^T) as built on device (K2); arrays sized n+1, nnz, nnz. */
equil_status equil_export_transpose(equil_matrix* A, int64_t* t_row_ptr,
                                    int32_t* t_col, double* t_val);
/* det_exp evaluated on device, elementwise (numerics contract). */
equil_status equil_det_exp_device(const double* x, double* y, int64_t n, int device);
/* Host side of the same contract (for ABI tests without a GPU). */
double equil_det_exp_host(double x);
/* Canonical sum of squares on device. */
equil_status equil_canon_sumsq_device(const double* x, int64_t n, double* out,
                                      int device);
/* Row partition used for world_size > 1: splits [0, rows) into `parts`
 * contiguous ranges balanced by nnz + rows; bounds has parts + 1 entries. */
equil_status equil_partition_rows(const int64_t* row_ptr, int64_t rows, int parts,
                                  int64_t* bounds);

/* ncclGetUniqueId for rank 0 of a multi-GPU run (128 bytes). */
equil_status equil_nccl_unique_id(void* out128);

const char* equil_last_error(void);
const char* equil_version(void);

#ifdef __cplusplus
}
#endif

#endif /* EQUIL_B200_H */
