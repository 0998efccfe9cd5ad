// equil_b200.hpp -- header-only C++ adapter over the C ABI (equil_b200.h) that
// mirrors the reference's C++ API for the hot path (namespace equil,
// include/equil/{params,equilibrate,lsqr}.hpp): same names, same defaults, same
// exception types (std::invalid_argument / std::runtime_error,
// include/equil/common.hpp:16-22).  Vectors are std::vector<double>; a
// reference-side shim converting Eigen::VectorXd / ExplicitMatrix is shown in
// INTEGRATION.md.
#pragma once

#include <cstdint>
#include <limits>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "equil_b200.h"

namespace equil_b200 {

using Vec = std::vector<double>;

inline void throw_on(equil_status s) {
  if (s == EQUIL_OK) return;
  const std::string msg = equil_last_error();
  if (s == EQUIL_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// include/equil/params.hpp:14-23
struct EquilibrationParams {
  static constexpr double kAutoTarget = 0.0;
  double alpha = kAutoTarget;
  double beta = kAutoTarget;
  double gamma = 0.1;
  double max_log_scale = 9.210340371976184;
  int iterations = 1000;
  std::uint64_t seed = 0;
  equil_params c() const { return {alpha, beta, gamma, max_log_scale, iterations, seed}; }
};

// include/equil/ccp.hpp:24-48
struct CcpOptions {
  int max_iters = 1000;
  double tau = 0.0;
  double sigma = 0.0;
  double theta = 1.0;
  double p_star = std::numeric_limits<double>::quiet_NaN();
  double gap_tol = 0.0;
};
struct CcpRun {
  Vec x;
  std::vector<double> objective_history, gap_history;
  double tau = 0.0, sigma = 0.0, theta = 1.0;
  int iterations = 0, equil_iterations = 0;
  bool reached_tol = false;
  long long apply_count = 0, adjoint_count = 0;
};

// include/equil/variants.hpp:30-39
struct BlockStructure {
  std::vector<std::int64_t> row_block, col_block;
  std::int64_t row_blocks = 0, col_blocks = 0;
  static BlockStructure trivial(std::int64_t rows, std::int64_t cols) {
    BlockStructure s;
    for (std::int64_t i = 0; i < rows; ++i) s.row_block.push_back(i);
    for (std::int64_t j = 0; j < cols; ++j) s.col_block.push_back(j);
    s.row_blocks = rows;
    s.col_blocks = cols;
    return s;
  }
};

// include/equil/equilibrate.hpp:51-78
struct IterationRecord {
  int iter = 0;
  std::optional<double> objective, rms, cond;
};
struct DiagnosticsConfig {
  bool enabled = false;  // the reference passes the explicit matrix; here it is implicit
  int stride = 1;
};
struct ScalingResult {
  Vec u, v, d, e;
  double alpha = 0.0, beta = 0.0;
  std::vector<IterationRecord> history;
  bool box_feasible = true, iterate_bound_ok = true;
  long long apply_count = 0, adjoint_count = 0;
};
// include/equil/lsqr.hpp:10-23
struct LsqrRun {
  Vec x;
  std::vector<double> residual_history;
  int iterations = 0, equil_iterations = 0;
  bool reached_tol = false, breakdown = false;
  long long apply_count = 0, adjoint_count = 0;
};

// Device-resident operator (ExplicitMatrix on the GPU).
class DeviceMatrix {
 public:
  static DeviceMatrix sparse_csr(std::int64_t rows, std::int64_t cols,
                                 const std::vector<std::int64_t>& row_ptr,
                                 const std::vector<std::int32_t>& col,
                                 const std::vector<double>& val, int device = 0) {
    equil_device_cfg cfg{device, 0, 1, nullptr};
    equil_matrix* h = nullptr;
    throw_on(equil_matrix_create_csr(rows, cols, row_ptr.data(), col.data(), val.data(),
                                     &cfg, &h));
    return DeviceMatrix(h);
  }
  static DeviceMatrix dense_rowmajor(std::int64_t rows, std::int64_t cols,
                                     const std::vector<double>& a, int device = 0) {
    equil_device_cfg cfg{device, 0, 1, nullptr};
    equil_matrix* h = nullptr;
    throw_on(equil_matrix_create_dense(rows, cols, a.data(), &cfg, &h));
    return DeviceMatrix(h);
  }
  std::int64_t rows() const { return shape().first; }
  std::int64_t cols() const { return shape().second; }
  Vec apply(const Vec& x) const {
    Vec y(static_cast<size_t>(rows()));
    throw_on(equil_apply(h_.get(), x.data(), y.data(), 0));
    return y;
  }
  Vec apply_adjoint(const Vec& y) const {
    Vec x(static_cast<size_t>(cols()));
    throw_on(equil_apply(h_.get(), y.data(), x.data(), 1));
    return x;
  }
  // read_matrix_market_file / write_matrix_market_file
  // (include/equil/matrix_market.hpp:17-21)
  static DeviceMatrix read_matrix_market(const std::string& path, int device = 0) {
    equil_device_cfg cfg{device, 0, 1, nullptr};
    equil_matrix* h = nullptr;
    throw_on(equil_matrix_read_matrix_market(path.c_str(), &cfg, &h));
    return DeviceMatrix(h);
  }
  void write_matrix_market(const std::string& path) const {
    throw_on(equil_matrix_write_matrix_market(h_.get(), path.c_str()));
  }
  equil_matrix* handle() const { return h_.get(); }

 private:
  explicit DeviceMatrix(equil_matrix* h) : h_(h, &equil_matrix_destroy) {}
  std::pair<std::int64_t, std::int64_t> shape() const {
    std::int64_t m = 0, n = 0;
    throw_on(equil_matrix_shape(h_.get(), &m, &n, nullptr));
    return {m, n};
  }
  std::shared_ptr<equil_matrix> h_;
};

// sgd_equilibrate (include/equil/equilibrate.hpp:89-91) and the variants
// (include/equil/variants.hpp:16-50) share the result plumbing
enum class Variant { kPlain, kSymmetric, kBlock };
inline ScalingResult sgd_run(const DeviceMatrix& op, const EquilibrationParams& p,
                             const DiagnosticsConfig& diag, Variant kind,
                             const BlockStructure* bs) {
  ScalingResult r;
  r.u.resize(static_cast<size_t>(op.rows()));
  r.d.resize(r.u.size());
  r.v.resize(static_cast<size_t>(op.cols()));
  r.e.resize(r.v.size());
  const int cap = diag.enabled && diag.stride > 0 ? p.iterations / diag.stride + 1 : 0;
  std::vector<int> hi(static_cast<size_t>(cap > 0 ? cap : 1));
  std::vector<double> ho(hi.size()), hr(hi.size());
  equil_scaling_out o{};
  o.u = r.u.data();
  o.v = r.v.data();
  o.d = r.d.data();
  o.e = r.e.data();
  o.hist_iter = hi.data();
  o.hist_objective = ho.data();
  o.hist_rms = hr.data();
  o.hist_cap = cap;
  const equil_params cp = p.c();
  equil_diag_cfg dc{diag.enabled ? diag.stride : 0, 1, 1};
  const equil_diag_cfg* dcp = diag.enabled ? &dc : nullptr;
  if (kind == Variant::kSymmetric) {
    throw_on(equil_sgd_equilibrate_symmetric(op.handle(), &cp, dcp, &o));
  } else if (kind == Variant::kBlock) {
    if (static_cast<std::int64_t>(bs->row_block.size()) != op.rows() ||
        static_cast<std::int64_t>(bs->col_block.size()) != op.cols())
      throw std::invalid_argument("BlockStructure: assignment length mismatch");
    throw_on(equil_sgd_equilibrate_block(op.handle(), bs->row_block.data(),
                                         bs->col_block.data(), bs->row_blocks, bs->col_blocks,
                                         &cp, dcp, &o));
  } else {
    throw_on(equil_sgd_equilibrate(op.handle(), &cp, dcp, &o));
  }
  r.alpha = o.alpha;
  r.beta = o.beta;
  r.box_feasible = o.box_feasible != 0;
  r.iterate_bound_ok = o.iterate_bound_ok != 0;
  r.apply_count = o.apply_count;
  r.adjoint_count = o.adjoint_count;
  for (int k = 0; k < o.hist_len; ++k) r.history.push_back({hi[k], ho[k], hr[k], std::nullopt});
  return r;
}

inline ScalingResult sgd_equilibrate(const DeviceMatrix& op, const EquilibrationParams& p,
                                     const DiagnosticsConfig& diag = {}) {
  return sgd_run(op, p, diag, Variant::kPlain, nullptr);
}
inline ScalingResult sgd_equilibrate_symmetric(const DeviceMatrix& op,
                                               const EquilibrationParams& p,
                                               const DiagnosticsConfig& diag = {}) {
  return sgd_run(op, p, diag, Variant::kSymmetric, nullptr);
}
inline ScalingResult sgd_equilibrate_block(const DeviceMatrix& op, const BlockStructure& s,
                                           const EquilibrationParams& p,
                                           const DiagnosticsConfig& diag = {}) {
  return sgd_run(op, p, diag, Variant::kBlock, &s);
}

inline LsqrRun lsqr_impl(const DeviceMatrix& op, const Vec& b, const EquilibrationParams* p,
                         int max_iters, double tol) {
  if (static_cast<std::int64_t>(b.size()) != op.rows())
    throw std::invalid_argument(p ? "lsqr_preconditioned: rhs length mismatch"
                                  : "lsqr: rhs length mismatch");
  LsqrRun r;
  r.x.resize(static_cast<size_t>(op.cols()));
  r.residual_history.resize(static_cast<size_t>(
      (max_iters > 0 ? max_iters : 0) + (p && p->iterations > 0 ? p->iterations : 0) + 2));
  equil_lsqr_out o{};
  o.x = r.x.data();
  o.residual_history = r.residual_history.data();
  o.residual_cap = static_cast<int>(r.residual_history.size());
  if (p) {
    const equil_params cp = p->c();
    throw_on(equil_lsqr_preconditioned(op.handle(), b.data(), &cp, max_iters, tol, &o));
  } else {
    throw_on(equil_lsqr(op.handle(), b.data(), max_iters, tol, &o));
  }
  r.residual_history.resize(static_cast<size_t>(o.hist_len));
  r.iterations = o.iterations;
  r.equil_iterations = o.equil_iterations;
  r.reached_tol = o.reached_tol != 0;
  r.breakdown = o.breakdown != 0;
  r.apply_count = o.apply_count;
  r.adjoint_count = o.adjoint_count;
  return r;
}

// lsqr / lsqr_preconditioned (include/equil/lsqr.hpp:30-40)
inline LsqrRun lsqr(const DeviceMatrix& op, const Vec& b, int max_iters, double tol) {
  return lsqr_impl(op, b, nullptr, max_iters, tol);
}
inline LsqrRun lsqr_preconditioned(const DeviceMatrix& op, const Vec& b,
                                   const EquilibrationParams& p, int max_iters, double tol) {
  return lsqr_impl(op, b, &p, max_iters, tol);
}

// ccp_lasso / ccp_lasso_preconditioned (include/equil/ccp.hpp:57-67); the
// problem's operator, rhs and lambda are passed directly (LassoProblem fields)
inline CcpRun ccp_impl(const DeviceMatrix& op, const Vec& b, double lambda,
                       const EquilibrationParams* p, const CcpOptions& opt) {
  if (static_cast<std::int64_t>(b.size()) != op.rows())
    throw std::invalid_argument("lasso: rhs length mismatch");
  CcpRun r;
  const int cap = (opt.max_iters > 0 ? opt.max_iters : 0) + 1 +
                  (p && p->iterations > 0 ? p->iterations : 0);
  r.x.resize(static_cast<size_t>(op.cols()));
  r.objective_history.resize(static_cast<size_t>(cap));
  r.gap_history.resize(static_cast<size_t>(cap));
  const equil_ccp_options o{opt.max_iters, opt.tau, opt.sigma, opt.theta, opt.p_star,
                            opt.gap_tol};
  equil_ccp_out out{};
  out.x = r.x.data();
  out.objective_history = r.objective_history.data();
  out.gap_history = r.gap_history.data();
  out.hist_cap = cap;
  if (p) {
    const equil_params cp = p->c();
    throw_on(equil_ccp_lasso_preconditioned(op.handle(), b.data(), lambda, &cp, &o, &out));
  } else {
    throw_on(equil_ccp_lasso(op.handle(), b.data(), lambda, &o, &out));
  }
  r.objective_history.resize(static_cast<size_t>(out.hist_len));
  r.gap_history.resize(static_cast<size_t>(out.gap_len));
  r.tau = out.tau;
  r.sigma = out.sigma;
  r.theta = out.theta;
  r.iterations = out.iterations;
  r.equil_iterations = out.equil_iterations;
  r.reached_tol = out.reached_tol != 0;
  r.apply_count = out.apply_count;
  r.adjoint_count = out.adjoint_count;
  return r;
}
inline CcpRun ccp_lasso(const DeviceMatrix& op, const Vec& b, double lambda,
                        const CcpOptions& opt = {}) {
  return ccp_impl(op, b, lambda, nullptr, opt);
}
inline CcpRun ccp_lasso_preconditioned(const DeviceMatrix& op, const Vec& b, double lambda,
                                       const EquilibrationParams& p,
                                       const CcpOptions& opt = {}) {
  return ccp_impl(op, b, lambda, &p, opt);
}
// spectral_norm (include/equil/lsqr.hpp:44-48)
inline double spectral_norm(const DeviceMatrix& op, int max_iters = 100, double rel_tol = 1e-6,
                            std::uint64_t seed = 0) {
  double v = 0.0;
  throw_on(equil_spectral_norm(op.handle(), max_iters, rel_tol, seed, &v));
  return v;
}

}  // namespace equil_b200
