// b200_backend.hpp -- the reference-side binding a maintainer adds to
// /root/reference/proj (as src/b200_backend.cpp + this header): the reference's
// own hot-path entry points, with the reference's own types, dispatched to the
// B200 library through its C ABI (include/equil_b200.h).
//
//   equil::b200::sgd_equilibrate      <- equil::sgd_equilibrate
//                                        (include/equil/equilibrate.hpp:89-91)
//   equil::b200::lsqr                 <- equil::lsqr (include/equil/lsqr.hpp:30-31)
//   equil::b200::lsqr_preconditioned  <- equil::lsqr_preconditioned
//                                        (include/equil/lsqr.hpp:38-40)
//
// Same arguments, same results (bit for bit: tests run by integration/
// test_backend.cpp), same exception types and messages
// (include/equil/common.hpp:16-22).  sgd_equilibrate takes any LinearOperator:
// an ExplicitMatrix runs on its device copy (CSR(A) and CSR(A^T), or the dense
// array); a matrix-free operator runs through the device-operator ABI
// (equil_sgd_equilibrate_operator, equil_lsqr_operator) with its own host apply
// bridged in each call.
#pragma once

#include <memory>

#include "equil/equilibrate.hpp"
#include "equil/explicit_matrix.hpp"
#include "equil/lsqr.hpp"

struct equil_matrix;

namespace equil::b200 {

/// The device copy of one ExplicitMatrix (CSR(A) and CSR(A^T), or the dense
/// row-major array), uploaded once and reused by every call that takes it.
class Device {
 public:
  explicit Device(const ExplicitMatrix& A, int device = 0);
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  equil_matrix* handle() const { return h_.get(); }

 private:
  Index rows_ = 0, cols_ = 0;
  std::shared_ptr<equil_matrix> h_;
};

ScalingResult sgd_equilibrate(const Device& A, const EquilibrationParams& params,
                              const DiagnosticsConfig& diag = {});
LsqrRun lsqr(const Device& A, const Vec& b, int max_iters, double rel_residual_tol);
LsqrRun lsqr_preconditioned(const Device& A, const Vec& b,
                            const EquilibrationParams& equil_params, int max_iters,
                            double rel_residual_tol);

/// Drop-in overloads on the reference's operator type: upload, run, release.
ScalingResult sgd_equilibrate(const LinearOperator& op, const EquilibrationParams& params,
                              const DiagnosticsConfig& diag = {});
LsqrRun lsqr(const LinearOperator& op, const Vec& b, int max_iters, double rel_residual_tol);
LsqrRun lsqr_preconditioned(const LinearOperator& op, const Vec& b,
                            const EquilibrationParams& equil_params, int max_iters,
                            double rel_residual_tol);

}  // namespace equil::b200
