// ref_harness.cpp -- extern "C" wrapper over the REFERENCE's own hot-path
// translation units (TEST INFRASTRUCTURE).  oracle/Makefile compiles
// /root/reference/proj/src/{rng,params,linop,estimator,explicit_matrix,
// equilibrate,lsqr,metrics}.cpp unmodified against oracle/eigen_lite and links
// this file, producing oracle/_ref/libequil_ref.so.  Tests use it to pin the C
// restatement (equil_oracle.c) and bench.py --impl reference times it.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "equil/ccp.hpp"
#include "equil/equilibrate.hpp"
#include "equil/explicit_matrix.hpp"
#include "equil/lsqr.hpp"
#include "equil/matrix_market.hpp"
#include "equil/metrics.hpp"
#include "equil/rng.hpp"
#include "equil/variants.hpp"

using namespace equil;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

Vec to_vec(const double* p, int64_t n) {
  Vec v(n);
  std::memcpy(v.data(), p, static_cast<std::size_t>(n) * sizeof(double));
  return v;
}
void from_vec(const Vec& v, double* p) {
  if (p) std::memcpy(p, v.data(), static_cast<std::size_t>(v.size()) * sizeof(double));
}
}  // namespace

extern "C" {

const char* er_last_error() { return g_err.c_str(); }

void er_rng_outputs(uint64_t seed, uint64_t stream, uint64_t count, uint64_t* out) {
  SeededRng r(seed, stream);
  for (uint64_t k = 0; k < count; ++k) out[k] = r.next_u64();
}

void er_rng_draws(uint64_t seed, uint64_t stream, int kind, uint64_t count,
                  double* out) {
  SeededRng r(seed, stream);
  for (uint64_t k = 0; k < count; ++k)
    out[k] = kind == 0 ? r.uniform01() : (kind == 1 ? r.normal() : r.sign());
}

// Matrix handle: ExplicitMatrix::sparse from the CSR arrays (construction is
// the reference's own sort + duplicate check, explicit_matrix.cpp:19-57).
int er_matrix_csr(int64_t m, int64_t n, const int64_t* row_ptr,
                  const int32_t* col, const double* val, void** out) {
  return guarded([&] {
    std::vector<ExplicitMatrix::Entry> ent;
    ent.reserve(static_cast<std::size_t>(row_ptr[m]));
    for (int64_t i = 0; i < m; ++i)
      for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k)
        ent.push_back({i, static_cast<Index>(col[k]), val[k]});
    *out = new ExplicitMatrix(ExplicitMatrix::sparse(m, n, std::move(ent)));
  });
}

int er_matrix_coo(int64_t m, int64_t n, int64_t nnz, const int64_t* rows,
                  const int64_t* cols, const double* vals, void** out) {
  return guarded([&] {
    std::vector<ExplicitMatrix::Entry> ent(static_cast<std::size_t>(nnz));
    for (int64_t k = 0; k < nnz; ++k) ent[k] = {rows[k], cols[k], vals[k]};
    *out = new ExplicitMatrix(ExplicitMatrix::sparse(m, n, std::move(ent)));
  });
}

int er_matrix_dense(int64_t m, int64_t n, const double* rowmajor, void** out) {
  return guarded([&] {
    Mat A(m, n);
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < n; ++j) A(i, j) = rowmajor[i * n + j];
    *out = new ExplicitMatrix(ExplicitMatrix::dense(std::move(A)));
  });
}

void er_matrix_free(void* h) { delete static_cast<ExplicitMatrix*>(h); }

int64_t er_matrix_nnz(void* h) {
  return static_cast<ExplicitMatrix*>(h)->stored_entries();
}

// CSR export (for_each_entry order = CSR order); row_ptr m+1.
void er_matrix_export(void* h, int64_t* row_ptr, int32_t* col, double* val) {
  const auto& A = *static_cast<ExplicitMatrix*>(h);
  int64_t k = 0;
  row_ptr[0] = 0;
  Index last = 0;
  A.for_each_entry([&](Index i, Index j, double v) {
    while (last < i) row_ptr[++last] = k;
    col[k] = static_cast<int32_t>(j);
    val[k] = v;
    ++k;
  });
  while (last < A.rows()) row_ptr[++last] = k;
}

void* er_matrix_transposed(void* h) {
  return new ExplicitMatrix(static_cast<ExplicitMatrix*>(h)->transposed());
}

int er_apply(void* h, const double* x, double* y, int adjoint) {
  return guarded([&] {
    const auto& A = *static_cast<ExplicitMatrix*>(h);
    if (adjoint)
      from_vec(A.apply_adjoint(to_vec(x, A.rows())), y);
    else
      from_vec(A.apply(to_vec(x, A.cols())), y);
  });
}

struct er_sgd_out {
  double* u;
  double* v;
  double* d;
  double* e;
  double alpha, beta;
  int box_feasible, iterate_bound_ok;
  long long apply_count, adjoint_count;
  int* hist_iter;
  double* hist_objective;
  double* hist_rms;
  int hist_len;
};

int er_sgd_equilibrate(void* h, double alpha, double beta, double gamma,
                       double max_log_scale, int iterations, uint64_t seed,
                       int diag_stride, er_sgd_out* out) {
  return guarded([&] {
    const auto& A = *static_cast<ExplicitMatrix*>(h);
    EquilibrationParams p;
    p.alpha = alpha;
    p.beta = beta;
    p.gamma = gamma;
    p.max_log_scale = max_log_scale;
    p.iterations = iterations;
    p.seed = seed;
    DiagnosticsConfig diag;
    if (diag_stride > 0) {
      diag.matrix = &A;
      diag.stride = diag_stride;
    }
    const ScalingResult r = sgd_equilibrate(A, p, diag);
    from_vec(r.u, out->u);
    from_vec(r.v, out->v);
    from_vec(r.d, out->d);
    from_vec(r.e, out->e);
    out->alpha = r.alpha;
    out->beta = r.beta;
    out->box_feasible = r.box_feasible;
    out->iterate_bound_ok = r.iterate_bound_ok;
    out->apply_count = r.apply_count;
    out->adjoint_count = r.adjoint_count;
    out->hist_len = static_cast<int>(r.history.size());
    for (std::size_t k = 0; k < r.history.size(); ++k) {
      if (out->hist_iter) out->hist_iter[k] = r.history[k].iter;
      if (out->hist_objective)
        out->hist_objective[k] = r.history[k].objective.value_or(0.0);
      if (out->hist_rms) out->hist_rms[k] = r.history[k].rms.value_or(0.0);
    }
  });
}

// sgd_equilibrate_targets (include/equil/variants.hpp:24-27)
int er_sgd_targets(void* h, const double* r, const double* c, double gamma,
                   double max_log_scale, int iterations, uint64_t seed, int diag_stride,
                   er_sgd_out* out) {
  return guarded([&] {
    const auto& A = *static_cast<ExplicitMatrix*>(h);
    EquilibrationParams p;
    p.gamma = gamma;
    p.max_log_scale = max_log_scale;
    p.iterations = iterations;
    p.seed = seed;
    DiagnosticsConfig diag;
    if (diag_stride > 0) {
      diag.matrix = &A;
      diag.stride = diag_stride;
    }
    const ScalingResult res =
        sgd_equilibrate_targets(A, to_vec(r, A.rows()), to_vec(c, A.cols()), p, diag);
    from_vec(res.u, out->u);
    from_vec(res.v, out->v);
    from_vec(res.d, out->d);
    from_vec(res.e, out->e);
    out->alpha = res.alpha;
    out->beta = res.beta;
    out->box_feasible = res.box_feasible;
    out->iterate_bound_ok = res.iterate_bound_ok;
    out->apply_count = res.apply_count;
    out->adjoint_count = res.adjoint_count;
    out->hist_len = static_cast<int>(res.history.size());
    for (std::size_t k = 0; k < res.history.size(); ++k) {
      if (out->hist_iter) out->hist_iter[k] = res.history[k].iter;
      if (out->hist_objective) out->hist_objective[k] = res.history[k].objective.value_or(0.0);
      if (out->hist_rms) out->hist_rms[k] = res.history[k].rms.value_or(0.0);
    }
  });
}

static void copy_scaling(const ScalingResult& res, er_sgd_out* out) {
  from_vec(res.u, out->u);
  from_vec(res.v, out->v);
  from_vec(res.d, out->d);
  from_vec(res.e, out->e);
  out->alpha = res.alpha;
  out->beta = res.beta;
  out->box_feasible = res.box_feasible;
  out->iterate_bound_ok = res.iterate_bound_ok;
  out->apply_count = res.apply_count;
  out->adjoint_count = res.adjoint_count;
  out->hist_len = static_cast<int>(res.history.size());
  for (std::size_t k = 0; k < res.history.size(); ++k) {
    if (out->hist_iter) out->hist_iter[k] = res.history[k].iter;
    if (out->hist_objective) out->hist_objective[k] = res.history[k].objective.value_or(0.0);
    if (out->hist_rms) out->hist_rms[k] = res.history[k].rms.value_or(0.0);
  }
}

// sgd_equilibrate_symmetric (include/equil/variants.hpp:16-18)
int er_sgd_symmetric(void* h, double alpha, double beta, double gamma, double max_log_scale,
                     int iterations, uint64_t seed, int diag_stride, er_sgd_out* out) {
  return guarded([&] {
    const auto& A = *static_cast<ExplicitMatrix*>(h);
    EquilibrationParams p;
    p.alpha = alpha;
    p.beta = beta;
    p.gamma = gamma;
    p.max_log_scale = max_log_scale;
    p.iterations = iterations;
    p.seed = seed;
    DiagnosticsConfig diag;
    if (diag_stride > 0) {
      diag.matrix = &A;
      diag.stride = diag_stride;
    }
    copy_scaling(sgd_equilibrate_symmetric(A, p, diag), out);
  });
}

// sgd_equilibrate_block (include/equil/variants.hpp:47-50)
int er_sgd_block(void* h, const int64_t* rb, const int64_t* cb, int64_t R, int64_t C,
                 double gamma, double max_log_scale, int iterations, uint64_t seed,
                 int diag_stride, er_sgd_out* out) {
  return guarded([&] {
    const auto& A = *static_cast<ExplicitMatrix*>(h);
    EquilibrationParams p;
    p.gamma = gamma;
    p.max_log_scale = max_log_scale;
    p.iterations = iterations;
    p.seed = seed;
    BlockStructure bs;
    bs.row_block.assign(rb, rb + A.rows());
    bs.col_block.assign(cb, cb + A.cols());
    bs.row_blocks = R;
    bs.col_blocks = C;
    DiagnosticsConfig diag;
    if (diag_stride > 0) {
      diag.matrix = &A;
      diag.stride = diag_stride;
    }
    copy_scaling(sgd_equilibrate_block(A, bs, p, diag), out);
  });
}

// ---- ccp_lasso / ccp_lasso_preconditioned / spectral_norm / lasso_fista
struct er_ccp_out {
  double* x;          // n
  double* obj_hist;   // capacity max_iters + 1 (+ T)
  double* gap_hist;   // same capacity (may be unused)
  int hist_len, gap_len;
  double tau, sigma, theta;
  int iterations, equil_iterations, reached_tol;
  long long apply_count, adjoint_count;
};

static void copy_ccp(const CcpRun& r, er_ccp_out* out) {
  from_vec(r.x, out->x);
  out->hist_len = static_cast<int>(r.objective_history.size());
  std::memcpy(out->obj_hist, r.objective_history.data(),
              r.objective_history.size() * sizeof(double));
  out->gap_len = static_cast<int>(r.gap_history.size());
  if (out->gap_hist && !r.gap_history.empty())
    std::memcpy(out->gap_hist, r.gap_history.data(), r.gap_history.size() * sizeof(double));
  out->tau = r.tau;
  out->sigma = r.sigma;
  out->theta = r.theta;
  out->iterations = r.iterations;
  out->equil_iterations = r.equil_iterations;
  out->reached_tol = r.reached_tol;
  out->apply_count = r.apply_count;
  out->adjoint_count = r.adjoint_count;
}

static CcpOptions ccp_opts(int max_iters, double tau, double sigma, double theta, double p_star,
                           double gap_tol) {
  CcpOptions o;
  o.max_iters = max_iters;
  o.tau = tau;
  o.sigma = sigma;
  o.theta = theta;
  o.p_star = p_star;
  o.gap_tol = gap_tol;
  return o;
}

int er_ccp_lasso(void* h, const double* b, double lambda, int max_iters, double tau,
                 double sigma, double theta, double p_star, double gap_tol, er_ccp_out* out) {
  return guarded([&] {
    const auto& A = *static_cast<ExplicitMatrix*>(h);
    LassoProblem prob{&A, to_vec(b, A.rows()), lambda};
    copy_ccp(ccp_lasso(prob, ccp_opts(max_iters, tau, sigma, theta, p_star, gap_tol)), out);
  });
}

int er_ccp_lasso_preconditioned(void* h, const double* b, double lambda, double alpha,
                                double beta, double gamma, double max_log_scale,
                                int iterations, uint64_t seed, int max_iters, double tau,
                                double sigma, double theta, double p_star, double gap_tol,
                                er_ccp_out* out) {
  return guarded([&] {
    const auto& A = *static_cast<ExplicitMatrix*>(h);
    LassoProblem prob{&A, to_vec(b, A.rows()), lambda};
    EquilibrationParams p;
    p.alpha = alpha;
    p.beta = beta;
    p.gamma = gamma;
    p.max_log_scale = max_log_scale;
    p.iterations = iterations;
    p.seed = seed;
    copy_ccp(ccp_lasso_preconditioned(prob, p,
                                      ccp_opts(max_iters, tau, sigma, theta, p_star, gap_tol)),
             out);
  });
}

int er_spectral_norm(void* h, int max_iters, double rel_tol, uint64_t seed, double* out) {
  return guarded([&] {
    *out = spectral_norm(*static_cast<ExplicitMatrix*>(h), max_iters, rel_tol, seed);
  });
}

int er_lasso_objective(void* h, const double* b, double lambda, const double* x, double* out) {
  return guarded([&] {
    const auto& A = *static_cast<ExplicitMatrix*>(h);
    LassoProblem prob{&A, to_vec(b, A.rows()), lambda};
    *out = lasso_objective(prob, to_vec(x, A.cols()));
  });
}

int er_lasso_fista(void* h, const double* b, double lambda, double grad_map_tol, int max_iters,
                   double* x, double* p_star) {
  return guarded([&] {
    const auto& A = *static_cast<ExplicitMatrix*>(h);
    LassoProblem prob{&A, to_vec(b, A.rows()), lambda};
    const FistaResult r = lasso_fista(prob, grad_map_tol, max_iters);
    from_vec(r.x, x);
    *p_star = r.p_star;
  });
}

// ---- read_matrix_market_file / write_matrix_market_file (matrix_market.hpp)
int er_mm_read(const char* path, void** out, int64_t* m, int64_t* n, int* is_sparse) {
  return guarded([&] {
    auto* A = new ExplicitMatrix(read_matrix_market_file(path));
    *out = A;
    *m = A->rows();
    *n = A->cols();
    *is_sparse = A->is_sparse() ? 1 : 0;
  });
}

int er_mm_write(void* h, const char* path) {
  return guarded([&] { write_matrix_market_file(path, *static_cast<ExplicitMatrix*>(h)); });
}

// dense values (row-major) of any ExplicitMatrix
int er_matrix_to_dense(void* h, double* out) {
  return guarded([&] {
    const auto& A = *static_cast<ExplicitMatrix*>(h);
    const Mat d = A.to_dense();
    for (Index i = 0; i < A.rows(); ++i)
      for (Index j = 0; j < A.cols(); ++j) out[i * A.cols() + j] = d(i, j);
  });
}

// ---- equilibrate.hpp helpers: objective / gradient (plain and weighted),
// stochastic_gradient_estimate (rng advanced by `offset` draws)
static EquilibrationParams mkparams(double alpha, double beta, double gamma, double M) {
  EquilibrationParams p;
  p.alpha = alpha;
  p.beta = beta;
  p.gamma = gamma;
  p.max_log_scale = M;
  return p;
}

int er_objective(void* h, const double* u, const double* v, double alpha, double beta,
                 double gamma, double* out) {
  return guarded([&] {
    const auto& A = *static_cast<ExplicitMatrix*>(h);
    *out = objective(A, to_vec(u, A.rows()), to_vec(v, A.cols()),
                     mkparams(alpha, beta, gamma, 9.210340371976184));
  });
}

int er_gradient(void* h, const double* u, const double* v, double alpha, double beta,
                double gamma, double* gu, double* gv) {
  return guarded([&] {
    const auto& A = *static_cast<ExplicitMatrix*>(h);
    Vec a, b;
    gradient(A, to_vec(u, A.rows()), to_vec(v, A.cols()),
             mkparams(alpha, beta, gamma, 9.210340371976184), a, b);
    from_vec(a, gu);
    from_vec(b, gv);
  });
}

int er_sge(void* h, const double* u, const double* v, double alpha, double beta, double gamma,
           uint64_t seed, uint64_t stream, uint64_t offset, double* gu, double* gv) {
  return guarded([&] {
    const auto& A = *static_cast<ExplicitMatrix*>(h);
    SeededRng rng(seed, stream);
    for (uint64_t k = 0; k < offset; ++k) rng.next_u64();
    Vec a, b;
    stochastic_gradient_estimate(A, to_vec(u, A.rows()), to_vec(v, A.cols()),
                                 mkparams(alpha, beta, gamma, 9.210340371976184), rng, a, b);
    from_vec(a, gu);
    from_vec(b, gv);
  });
}

struct er_lsqr_out {
  double* x;
  double* residual_history;  // capacity given by caller
  int hist_len;
  int iterations, equil_iterations, reached_tol, breakdown;
  long long apply_count, adjoint_count;
};

static void copy_run(const LsqrRun& r, er_lsqr_out* out) {
  from_vec(r.x, out->x);
  out->hist_len = static_cast<int>(r.residual_history.size());
  std::memcpy(out->residual_history, r.residual_history.data(),
              r.residual_history.size() * sizeof(double));
  out->iterations = r.iterations;
  out->equil_iterations = r.equil_iterations;
  out->reached_tol = r.reached_tol;
  out->breakdown = r.breakdown;
  out->apply_count = r.apply_count;
  out->adjoint_count = r.adjoint_count;
}

int er_lsqr(void* h, const double* b, int max_iters, double tol,
            er_lsqr_out* out) {
  return guarded([&] {
    const auto& A = *static_cast<ExplicitMatrix*>(h);
    copy_run(lsqr(A, to_vec(b, A.rows()), max_iters, tol), out);
  });
}

int er_lsqr_preconditioned(void* h, const double* b, double alpha, double beta,
                           double gamma, double max_log_scale, int iterations,
                           uint64_t seed, int max_iters, double tol,
                           er_lsqr_out* out) {
  return guarded([&] {
    const auto& A = *static_cast<ExplicitMatrix*>(h);
    EquilibrationParams p;
    p.alpha = alpha;
    p.beta = beta;
    p.gamma = gamma;
    p.max_log_scale = max_log_scale;
    p.iterations = iterations;
    p.seed = seed;
    copy_run(lsqr_preconditioned(A, to_vec(b, A.rows()), p, max_iters, tol),
             out);
  });
}

double er_rms_error(void* h, const double* u, const double* v, double alpha,
                    double beta) {
  const auto& A = *static_cast<ExplicitMatrix*>(h);
  return rms_error(A, to_vec(u, A.rows()), to_vec(v, A.cols()), alpha, beta);
}

}  // extern "C"
