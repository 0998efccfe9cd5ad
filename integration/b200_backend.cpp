// b200_backend.cpp -- reference-side binding of the B200 hot path (see
// b200_backend.hpp).  Compiled against the reference's headers
// (/root/reference/proj/include) and linked with libequil_b200.so; built by
// integration/Makefile.  Everything below is plumbing between the reference's
// types (ExplicitMatrix, EquilibrationParams, DiagnosticsConfig, ScalingResult,
// LsqrRun) and the C ABI: no arithmetic of the path runs here.
#include "b200_backend.hpp"

#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime_api.h>

#include "equil_b200.h"

namespace equil::b200 {
namespace {

void check(equil_status s) {
  if (s == EQUIL_OK) return;
  const std::string msg = equil_last_error();
  if (s == EQUIL_EINVAL) throw std::invalid_argument(msg);  // common.hpp:16-18
  throw std::runtime_error(msg);                            // common.hpp:20-22
}

equil_params to_c(const EquilibrationParams& p) {
  return {p.alpha, p.beta, p.gamma, p.max_log_scale, p.iterations, p.seed};
}

void cuda_ok(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("b200 backend: ") + cudaGetErrorString(e));
}

// A matrix-free LinearOperator whose apply is host code (the user's plugin):
// the device SGD loop calls it through the device-operator ABI, with the
// probe copied to the host and the result copied back.  The operator's own
// apply runs unchanged, so the result is the reference's bit for bit; the
// PCIe round trips bound its speed, and an operator with a device apply
// should implement equil_device_operator directly.
struct HostBridge {
  const LinearOperator* op;
  Vec in_m, in_n;
  std::exception_ptr error;
};
void bridge(void* ctx, const double* in, double* out, void* stream, bool adjoint) {
  auto* b = static_cast<HostBridge*>(ctx);
  if (b->error) return;
  try {
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    Vec& x = adjoint ? b->in_m : b->in_n;
    cuda_ok(cudaMemcpyAsync(x.data(), in, static_cast<size_t>(x.size()) * 8,
                            cudaMemcpyDeviceToHost, s));
    cuda_ok(cudaStreamSynchronize(s));
    const Vec y = adjoint ? b->op->apply_adjoint(x) : b->op->apply(x);
    cuda_ok(cudaMemcpyAsync(out, y.data(), static_cast<size_t>(y.size()) * 8,
                            cudaMemcpyHostToDevice, s));
    cuda_ok(cudaStreamSynchronize(s));
  } catch (...) {
    b->error = std::current_exception();
  }
}
void bridge_apply(void* ctx, const double* in, double* out, void* stream) {
  bridge(ctx, in, out, stream, false);
}
void bridge_adjoint(void* ctx, const double* in, double* out, void* stream) {
  bridge(ctx, in, out, stream, true);
}

Vec to_vec(const std::vector<double>& v) {
  Vec out(static_cast<Index>(v.size()));
  if (!v.empty()) std::memcpy(out.data(), v.data(), v.size() * sizeof(double));
  return out;
}

}  // namespace

// ExplicitMatrix's arrays are private: the CSR (sparse) or the row-major
// array (dense) is read through the public entry visitor, which walks rows in
// order and, within a row, the stored order (explicit_matrix.hpp:37-49).
Device::Device(const ExplicitMatrix& A, int device) : rows_(A.rows()), cols_(A.cols()) {
  equil_device_cfg cfg{device, 0, 1, nullptr};
  equil_matrix* h = nullptr;
  if (A.is_sparse()) {
    std::vector<int64_t> rp(static_cast<size_t>(rows_) + 1, 0);
    std::vector<int32_t> col;
    std::vector<double> val;
    col.reserve(static_cast<size_t>(A.stored_entries()));
    val.reserve(static_cast<size_t>(A.stored_entries()));
    A.for_each_entry([&](Index i, Index j, double v) {
      ++rp[static_cast<size_t>(i) + 1];
      col.push_back(static_cast<int32_t>(j));
      val.push_back(v);
    });
    for (Index i = 0; i < rows_; ++i) rp[i + 1] += rp[i];
    check(equil_matrix_create_csr(rows_, cols_, rp.data(), col.data(), val.data(), &cfg, &h));
  } else {
    std::vector<double> rowmajor(static_cast<size_t>(rows_) * static_cast<size_t>(cols_));
    A.for_each_entry([&](Index i, Index j, double v) {
      rowmajor[static_cast<size_t>(i) * static_cast<size_t>(cols_) + static_cast<size_t>(j)] = v;
    });
    check(equil_matrix_create_dense(rows_, cols_, rowmajor.data(), &cfg, &h));
  }
  h_ = std::shared_ptr<equil_matrix>(h, &equil_matrix_destroy);
}

// sgd_equilibrate (src/equilibrate.cpp:213-221 -> sgd_row_col :138-209):
// targets resolved and parameters validated first, then the diagnostics
// configuration, in the reference's order, so the same call throws the same
// message.  History rows: objective at every stride, RMS with uniform targets.
ScalingResult sgd_equilibrate(const Device& A, const EquilibrationParams& params,
                              const DiagnosticsConfig& diag) {
  const equil_params cp = to_c(params);
  double alpha = 0.0, beta = 0.0;
  check(equil_resolve_targets(&cp, A.rows(), A.cols(), &alpha, &beta));
  check(equil_validate_params(&cp));
  if (diag.matrix != nullptr) {
    if (diag.matrix->rows() != A.rows() || diag.matrix->cols() != A.cols())
      throw std::invalid_argument("sgd_row_col: diagnostics matrix shape mismatch");
    if (diag.stride <= 0) throw std::invalid_argument("sgd_row_col: stride must be positive");
    if (diag.cond_stride > 0)
      throw std::invalid_argument(
          "b200 backend: condition-number diagnostics (cond_stride > 0) are not on the GPU path");
  }
  const int T = params.iterations;
  const int cap = diag.matrix != nullptr ? T / diag.stride + 1 : 0;
  std::vector<double> u(static_cast<size_t>(A.rows())), d(u.size());
  std::vector<double> v(static_cast<size_t>(A.cols())), e(v.size());
  std::vector<int> hi(static_cast<size_t>(cap > 0 ? cap : 1));
  std::vector<double> ho(hi.size()), hr(hi.size());
  equil_scaling_out o{};
  o.u = u.data();
  o.v = v.data();
  o.d = d.data();
  o.e = e.data();
  o.hist_iter = hi.data();
  o.hist_objective = ho.data();
  o.hist_rms = hr.data();
  o.hist_cap = cap;
  const equil_diag_cfg dc{diag.matrix != nullptr ? diag.stride : 0, 1, 1};
  check(equil_sgd_equilibrate(A.handle(), &cp, diag.matrix != nullptr ? &dc : nullptr, &o));
  ScalingResult r;
  r.u = to_vec(u);
  r.v = to_vec(v);
  r.d = to_vec(d);
  r.e = to_vec(e);
  r.alpha = o.alpha;
  r.beta = o.beta;
  r.box_feasible = o.box_feasible != 0;
  r.iterate_bound_ok = o.iterate_bound_ok != 0;
  r.apply_count = o.apply_count;
  r.adjoint_count = o.adjoint_count;
  for (int k = 0; k < o.hist_len; ++k) {
    IterationRecord rec;
    rec.iter = hi[static_cast<size_t>(k)];
    rec.objective = ho[static_cast<size_t>(k)];
    if (o.alpha > 0.0 && o.beta > 0.0) rec.rms = hr[static_cast<size_t>(k)];
    r.history.push_back(rec);
  }
  return r;
}

namespace {
// lsqr (src/lsqr.cpp:85-103) and lsqr_preconditioned (:105-138)
LsqrRun lsqr_run(const Device& A, const Vec& b, const EquilibrationParams* p, int max_iters,
                 double tol) {
  if (b.size() != A.rows())  // the C ABI takes a raw pointer of rows() entries
    throw std::invalid_argument(p ? "lsqr_preconditioned: rhs length mismatch"
                                  : "lsqr: rhs length mismatch");
  std::vector<double> x(static_cast<size_t>(A.cols()));
  std::vector<double> hist(static_cast<size_t>((max_iters > 0 ? max_iters : 0) +
                                               (p && p->iterations > 0 ? p->iterations : 0) + 2));
  equil_lsqr_out o{};
  o.x = x.data();
  o.residual_history = hist.data();
  o.residual_cap = static_cast<int>(hist.size());
  if (p) {
    const equil_params cp = to_c(*p);
    check(equil_lsqr_preconditioned(A.handle(), b.data(), &cp, max_iters, tol, &o));
  } else {
    check(equil_lsqr(A.handle(), b.data(), max_iters, tol, &o));
  }
  LsqrRun r;
  r.x = to_vec(x);
  r.residual_history.assign(hist.begin(), hist.begin() + o.hist_len);
  r.iterations = o.iterations;
  r.equil_iterations = o.equil_iterations;
  r.reached_tol = o.reached_tol != 0;
  r.breakdown = o.breakdown != 0;
  r.apply_count = o.apply_count;
  r.adjoint_count = o.adjoint_count;
  return r;
}
}  // namespace

LsqrRun lsqr(const Device& A, const Vec& b, int max_iters, double rel_residual_tol) {
  return lsqr_run(A, b, nullptr, max_iters, rel_residual_tol);
}

LsqrRun lsqr_preconditioned(const Device& A, const Vec& b, const EquilibrationParams& p,
                            int max_iters, double rel_residual_tol) {
  return lsqr_run(A, b, &p, max_iters, rel_residual_tol);
}

ScalingResult sgd_equilibrate(const LinearOperator& op, const EquilibrationParams& params,
                              const DiagnosticsConfig& diag) {
  if (const auto* A = dynamic_cast<const ExplicitMatrix*>(&op))
    return sgd_equilibrate(Device(*A), params, diag);
  // matrix-free: the device loop around the operator's own apply
  // (equil_sgd_equilibrate_operator); diagnostics need the explicit matrix
  const equil_params cp = to_c(params);
  double alpha = 0.0, beta = 0.0;
  check(equil_resolve_targets(&cp, op.rows(), op.cols(), &alpha, &beta));
  check(equil_validate_params(&cp));
  if (diag.matrix != nullptr)
    throw std::invalid_argument(
        "b200 backend: diagnostics of a matrix-free operator need sgd_equilibrate on the "
        "explicit matrix");
  HostBridge hb{&op, Vec(op.rows()), Vec(op.cols()), nullptr};
  const equil_device_operator dop{op.rows(), op.cols(), &bridge_apply, &bridge_adjoint, &hb, 0};
  std::vector<double> u(static_cast<size_t>(op.rows())), d(u.size());
  std::vector<double> v(static_cast<size_t>(op.cols())), e(v.size());
  equil_scaling_out o{};
  o.u = u.data();
  o.v = v.data();
  o.d = d.data();
  o.e = e.data();
  const equil_status st = equil_sgd_equilibrate_operator(&dop, &cp, &o);
  if (hb.error) std::rethrow_exception(hb.error);  // the operator's own exception
  check(st);
  ScalingResult r;
  r.u = to_vec(u);
  r.v = to_vec(v);
  r.d = to_vec(d);
  r.e = to_vec(e);
  r.alpha = o.alpha;
  r.beta = o.beta;
  r.box_feasible = o.box_feasible != 0;
  r.iterate_bound_ok = o.iterate_bound_ok != 0;
  r.apply_count = o.apply_count;
  r.adjoint_count = o.adjoint_count;
  return r;
}

namespace {
// lsqr / lsqr_preconditioned of a matrix-free operator: the device loop
// (equil_lsqr_operator) around the operator's own host apply
LsqrRun lsqr_bridged(const LinearOperator& op, const Vec& b, const EquilibrationParams* p,
                     int max_iters, double tol) {
  if (b.size() != op.rows())
    throw std::invalid_argument(p ? "lsqr_preconditioned: rhs length mismatch"
                                  : "lsqr: rhs length mismatch");
  HostBridge hb{&op, Vec(op.rows()), Vec(op.cols()), nullptr};
  const equil_device_operator dop{op.rows(), op.cols(), &bridge_apply, &bridge_adjoint, &hb, 0};
  std::vector<double> x(static_cast<size_t>(op.cols()));
  std::vector<double> hist(static_cast<size_t>((max_iters > 0 ? max_iters : 0) +
                                               (p && p->iterations > 0 ? p->iterations : 0) + 2));
  equil_lsqr_out o{};
  o.x = x.data();
  o.residual_history = hist.data();
  o.residual_cap = static_cast<int>(hist.size());
  equil_params cp{};
  if (p) cp = to_c(*p);
  const equil_status st = equil_lsqr_operator(&dop, b.data(), p ? &cp : nullptr, max_iters, tol, &o);
  if (hb.error) std::rethrow_exception(hb.error);
  check(st);
  LsqrRun r;
  r.x = to_vec(x);
  r.residual_history.assign(hist.begin(), hist.begin() + o.hist_len);
  r.iterations = o.iterations;
  r.equil_iterations = o.equil_iterations;
  r.reached_tol = o.reached_tol != 0;
  r.breakdown = o.breakdown != 0;
  r.apply_count = o.apply_count;
  r.adjoint_count = o.adjoint_count;
  return r;
}
}  // namespace

LsqrRun lsqr(const LinearOperator& op, const Vec& b, int max_iters, double rel_residual_tol) {
  if (const auto* A = dynamic_cast<const ExplicitMatrix*>(&op))
    return lsqr(Device(*A), b, max_iters, rel_residual_tol);
  return lsqr_bridged(op, b, nullptr, max_iters, rel_residual_tol);
}

LsqrRun lsqr_preconditioned(const LinearOperator& op, const Vec& b,
                            const EquilibrationParams& p, int max_iters,
                            double rel_residual_tol) {
  if (const auto* A = dynamic_cast<const ExplicitMatrix*>(&op))
    return lsqr_preconditioned(Device(*A), b, p, max_iters, rel_residual_tol);
  return lsqr_bridged(op, b, &p, max_iters, rel_residual_tol);
}

}  // namespace equil::b200
