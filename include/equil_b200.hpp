// equil_b200.hpp -- header-only C++ adapter over the C ABI (equil_b200.h) that
// mirrors the reference's C++ API for the hot path (namespace equil,
// include/equil/{params,equilibrate,lsqr}.hpp): same names, same defaults, same
// exception types (std::invalid_argument / std::runtime_error,
// include/equil/common.hpp:16-22).  Vectors are std::vector<double>; a
// reference-side shim converting Eigen::VectorXd / ExplicitMatrix is shown in
// INTEGRATION.md.
#pragma once

#include <cstdint>
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

// sgd_equilibrate (include/equil/equilibrate.hpp:89-91)
inline ScalingResult sgd_equilibrate(const DeviceMatrix& op, const EquilibrationParams& p,
                                     const DiagnosticsConfig& diag = {}) {
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
  throw_on(equil_sgd_equilibrate(op.handle(), &cp, diag.enabled ? &dc : nullptr, &o));
  r.alpha = o.alpha;
  r.beta = o.beta;
  r.box_feasible = o.box_feasible != 0;
  r.iterate_bound_ok = o.iterate_bound_ok != 0;
  r.apply_count = o.apply_count;
  r.adjoint_count = o.adjoint_count;
  for (int k = 0; k < o.hist_len; ++k) r.history.push_back({hi[k], ho[k], hr[k], std::nullopt});
  return r;
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

}  // namespace equil_b200
