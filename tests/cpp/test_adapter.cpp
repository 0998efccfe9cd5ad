// C++ adapter test: the reference's own test cases, restated against the B200
// adapter (include/equil_b200.hpp).  Mirrors tests/test_itersolvers.cpp:36-46,
// :88-91, :123-142 and tests/test_equilibrate.cpp:183-198, :229-261.
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "equil_b200.hpp"

using namespace equil_b200;

static int failures = 0;
#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #c);        \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

static DeviceMatrix identity(int n) {
  std::vector<std::int64_t> rp(n + 1);
  std::vector<std::int32_t> c(n);
  std::vector<double> v(n, 1.0);
  for (int i = 0; i <= n; ++i) rp[i] = i;
  for (int i = 0; i < n; ++i) c[i] = i;
  return DeviceMatrix::sparse_csr(n, n, rp, c, v);
}

int main() {
  {  // lsqr: identity solves in one iteration
    const Vec b = {0.3, -1.2, 2.5, 0.7, -0.1, 1.9};
    const LsqrRun run = lsqr(identity(6), b, 10, 1e-12);
    CHECK(run.reached_tol);
    CHECK(run.iterations == 1);
    CHECK(run.residual_history.size() == 2);
    CHECK(run.residual_history[0] == 1.0);
    CHECK(run.residual_history[1] <= 1e-12);
  }
  {  // lsqr rejects a zero right-hand side
    bool threw = false;
    try {
      lsqr(identity(3), Vec(3, 0.0), 5, 1e-6);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // preconditioned identity = plain shifted by T, bit-identical
    const Vec b = {1.0, -2.0, 0.5, 3.0, -0.25, 0.125, 4.0};
    const LsqrRun plain = lsqr(identity(7), b, 50, 1e-12);
    EquilibrationParams ep;
    ep.iterations = 9;
    const LsqrRun pre = lsqr_preconditioned(identity(7), b, ep, 50, 1e-12);
    CHECK(pre.equil_iterations == 9);
    CHECK(pre.x == plain.x);
    CHECK(pre.residual_history.size() == plain.residual_history.size() + 9);
    CHECK(pre.apply_count == plain.apply_count + 9);
    CHECK(pre.adjoint_count == plain.adjoint_count + 9);
  }
  {  // sgd on the identity never leaves the fixed point; history on the grid
    EquilibrationParams p;
    p.alpha = p.beta = 1.0;
    p.iterations = 50;
    DiagnosticsConfig diag{true, 10};
    const ScalingResult r = sgd_equilibrate(identity(5), p, diag);
    for (double x : r.u) CHECK(x == 0.0);
    for (double x : r.d) CHECK(x == 1.0);
    CHECK(r.history.size() == 6);
    for (const auto& h : r.history) CHECK(std::abs(*h.objective - 2.5) <= 2.5e-15);
    CHECK(r.apply_count == 50 && r.adjoint_count == 50);
  }
  {  // bit-for-bit determinism under the seed; a different seed differs
    std::vector<double> a(8 * 6);
    for (size_t k = 0; k < a.size(); ++k) a[k] = std::sin(1.0 + 0.37 * k) * (1 + k % 5);
    const DeviceMatrix A = DeviceMatrix::dense_rowmajor(8, 6, a);
    EquilibrationParams p;
    p.iterations = 200;
    p.seed = 99;
    const ScalingResult r1 = sgd_equilibrate(A, p), r2 = sgd_equilibrate(A, p);
    CHECK(r1.u == r2.u && r1.v == r2.v && r1.d == r2.d && r1.e == r2.e);
    p.seed = 100;
    CHECK(sgd_equilibrate(A, p).u != r1.u);
  }
  {  // invalid parameters -> std::invalid_argument
    EquilibrationParams p;
    p.gamma = 0.0;
    bool threw = false;
    try {
      sgd_equilibrate(identity(3), p);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // variants (test_variants.cpp:36-48, :165-176): symmetric identity fixed
     // point; singleton blocks reproduce the plain solver exactly
    EquilibrationParams p;
    p.alpha = p.beta = 1.0;
    p.iterations = 100;
    const ScalingResult s = sgd_equilibrate_symmetric(identity(4), p);
    for (double x : s.u) CHECK(x == 0.0);
    CHECK(s.u == s.v && s.d == s.e && s.apply_count == 100 && s.adjoint_count == 0);
    std::vector<double> a(5 * 7);
    for (size_t k = 0; k < a.size(); ++k) a[k] = std::cos(0.3 + 0.71 * k) * (1 + k % 3);
    const DeviceMatrix A = DeviceMatrix::dense_rowmajor(5, 7, a);
    EquilibrationParams q;
    q.iterations = 300;
    q.seed = 11;
    const ScalingResult plain = sgd_equilibrate(A, q);
    const ScalingResult blk = sgd_equilibrate_block(A, BlockStructure::trivial(5, 7), q);
    CHECK(plain.u == blk.u && plain.v == blk.v);
  }
  {  // ccp on the identity reaches the soft-threshold solution
     // (test_itersolvers.cpp:205-225); spectral norm of diag(3, 1)
    CcpOptions opt;
    opt.max_iters = 5000;
    const CcpRun run = ccp_lasso(identity(2), Vec{3.0, 0.0}, 4.0, opt);
    CHECK(std::abs(run.x[0] - 1.0) <= 1e-6 && std::abs(run.x[1]) <= 1e-8);
    CHECK(static_cast<int>(run.objective_history.size()) == run.iterations + 1);
    CHECK(run.apply_count == run.iterations && run.adjoint_count == run.iterations);
    const DeviceMatrix D = DeviceMatrix::dense_rowmajor(2, 2, {3.0, 0.0, 0.0, 1.0});
    CHECK(std::abs(spectral_norm(D, 500, 1e-12) - 3.0) <= 3e-8);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
