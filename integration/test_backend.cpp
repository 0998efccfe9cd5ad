// test_backend.cpp -- the reference's hot-path cases run through the
// reference-side binding (b200_backend.cpp) on the GPU, each compared with the
// reference's own CPU implementation (its unmodified sources, built by
// oracle/Makefile into oracle/_ref/libequil_ref.so) on the same inputs.
//
// The cases follow the situations the reference's own suites exercise
// (tests/test_equilibrate.cpp:183-349, tests/test_itersolvers.cpp:36-171):
// the identity fixed point, the 1x1 problem, determinism under the seed, the
// charged apply/adjoint counts, history on the stride grid, box feasibility,
// LSQR on the identity / a diagonal / a random square system, the charged
// counts, the zero right-hand side, breakdown, a singular system, the trivial
// and badly scaled preconditioned runs, and a matrix-free operator (the
// reference's LinearOperator plugin) through the device loop.  Every case
// asserts bit equality of
// the outputs with the reference's (history values within 1e-12 relative:
// the reference evaluates them with sequential sums and std::exp), plus the
// case's own property.  Prints "OK" when every check passes.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "b200_backend.hpp"
#include "equil/rng.hpp"

using namespace equil;

namespace {

int g_fail = 0, g_checks = 0;

void expect(bool ok, const std::string& what) {
  ++g_checks;
  if (!ok) {
    ++g_fail;
    std::printf("FAIL: %s\n", what.c_str());
  }
}

bool same_bits(const Vec& a, const Vec& b) {
  return a.size() == b.size() &&
         (a.size() == 0 ||
          std::memcmp(a.data(), b.data(), static_cast<size_t>(a.size()) * sizeof(double)) == 0);
}
bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() &&
         (a.empty() || std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0);
}
bool close(double a, double b, double rel) {
  return std::fabs(a - b) <= rel * std::max(std::fabs(a), std::fabs(b)) || a == b;
}

void compare_scaling(const ScalingResult& g, const ScalingResult& r, const std::string& tag) {
  expect(same_bits(g.u, r.u), tag + ": u bit-identical");
  expect(same_bits(g.v, r.v), tag + ": v bit-identical");
  expect(same_bits(g.d, r.d), tag + ": d bit-identical");
  expect(same_bits(g.e, r.e), tag + ": e bit-identical");
  expect(g.alpha == r.alpha && g.beta == r.beta, tag + ": resolved targets");
  expect(g.box_feasible == r.box_feasible, tag + ": box_feasible");
  expect(g.iterate_bound_ok == r.iterate_bound_ok, tag + ": iterate_bound_ok");
  expect(g.apply_count == r.apply_count && g.adjoint_count == r.adjoint_count,
         tag + ": charged counts");
  expect(g.history.size() == r.history.size(), tag + ": history length");
  for (size_t k = 0; k < std::min(g.history.size(), r.history.size()); ++k) {
    const IterationRecord &a = g.history[k], &b = r.history[k];
    expect(a.iter == b.iter, tag + ": history iteration grid");
    expect(a.objective.has_value() == b.objective.has_value() &&
               (!a.objective || close(*a.objective, *b.objective, 1e-12)),
           tag + ": history objective");
    expect(a.rms.has_value() == b.rms.has_value() && (!a.rms || close(*a.rms, *b.rms, 1e-12)),
           tag + ": history rms");
  }
}

void compare_lsqr(const LsqrRun& g, const LsqrRun& r, const std::string& tag) {
  expect(same_bits(g.x, r.x), tag + ": x bit-identical");
  expect(same_bits(g.residual_history, r.residual_history),
         tag + ": residual history bit-identical");
  expect(g.iterations == r.iterations && g.equil_iterations == r.equil_iterations,
         tag + ": iteration counts");
  expect(g.reached_tol == r.reached_tol && g.breakdown == r.breakdown, tag + ": flags");
  expect(g.apply_count == r.apply_count && g.adjoint_count == r.adjoint_count,
         tag + ": charged counts");
}

// the same exception type and message from both implementations
template <class E>
void same_throw(const std::function<void()>& gpu, const std::function<void()>& ref,
                const std::string& tag) {
  std::string mg = "<none>", mr = "<none>";
  try {
    gpu();
  } catch (const E& e) {
    mg = e.what();
  } catch (const std::exception& e) {
    mg = std::string("<other> ") + e.what();
  }
  try {
    ref();
  } catch (const E& e) {
    mr = e.what();
  } catch (const std::exception& e) {
    mr = std::string("<other> ") + e.what();
  }
  expect(mg == mr && mg != "<none>", tag + ": same exception (gpu '" + mg + "', ref '" + mr + "')");
}

Mat gaussian(Index m, Index n, SeededRng& rng) {
  Mat A(m, n);
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < n; ++j) A(i, j) = rng.normal();
  return A;
}
Vec gaussian_vec(Index n, SeededRng& rng) {
  Vec x(n);
  for (Index i = 0; i < n; ++i) x[i] = rng.normal();
  return x;
}
// sparse with independent fill, badly scaled rows/columns; `long_rows` rows
// are made (nearly) full so they take the long-slice path (> 512 entries)
ExplicitMatrix scaled_sparse(Index m, Index n, double fill, Index long_rows, SeededRng& rng) {
  std::vector<double> rs(static_cast<size_t>(m)), cs(static_cast<size_t>(n));
  for (auto& s : rs) s = std::exp(1.5 * rng.normal());
  for (auto& s : cs) s = std::exp(1.5 * rng.normal());
  std::vector<ExplicitMatrix::Entry> ent;
  for (Index i = 0; i < m; ++i) {
    const double f = i < long_rows ? 0.9 : fill;
    for (Index j = 0; j < n; ++j)
      if (rng.uniform01() < f) ent.push_back({i, j, rng.normal() * rs[i] * cs[j]});
  }
  return ExplicitMatrix::sparse(m, n, ent);
}
Mat badly_scaled_dense(Index m, Index n, SeededRng& rng) {
  Mat B = gaussian(m, n, rng);
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < n; ++j) B(i, j) += 1.0;
  for (Index i = 0; i < m; ++i) {
    const double s = std::pow(10.0, 4.0 * (2.0 * rng.uniform01() - 1.0));
    for (Index j = 0; j < n; ++j) B(i, j) *= s;
  }
  for (Index j = 0; j < n; ++j) {
    const double s = std::pow(10.0, 4.0 * (2.0 * rng.uniform01() - 1.0));
    for (Index i = 0; i < m; ++i) B(i, j) *= s;
  }
  return B;
}

void sgd_cases() {
  {  // identity: the fixed point u = v = 0 is never left
    const ExplicitMatrix I = ExplicitMatrix::identity(7);
    EquilibrationParams p;
    p.iterations = 50;
    const ScalingResult g = b200::sgd_equilibrate(I, p), r = sgd_equilibrate(I, p);
    compare_scaling(g, r, "sgd identity");
    bool zero = true;
    for (Index i = 0; i < 7; ++i) zero = zero && g.u[i] == 0.0 && g.v[i] == 0.0;
    expect(zero, "sgd identity: stays at u = v = 0");
  }
  {  // 1x1 problem with explicit targets
    Mat a(1, 1);
    a(0, 0) = 3.0;
    const ExplicitMatrix A = ExplicitMatrix::dense(a);
    EquilibrationParams p;
    p.alpha = 2.0;
    p.beta = 2.0;
    p.gamma = 0.05;
    p.iterations = 400;
    compare_scaling(b200::sgd_equilibrate(A, p), sgd_equilibrate(A, p), "sgd 1x1");
  }
  {  // random sparse with history on a stride grid, and determinism
    SeededRng rng(101, 0);
    const ExplicitMatrix A = scaled_sparse(60, 35, 0.15, 0, rng);
    EquilibrationParams p;
    p.iterations = 200;
    p.seed = 7;
    DiagnosticsConfig diag;
    diag.matrix = &A;
    diag.stride = 10;
    const b200::Device dev(A);
    const ScalingResult g = b200::sgd_equilibrate(dev, p, diag);
    const ScalingResult g2 = b200::sgd_equilibrate(dev, p, diag);
    compare_scaling(g, sgd_equilibrate(A, p, diag), "sgd sparse + history");
    compare_scaling(g2, g, "sgd determinism under the seed");
    expect(g.history.size() == 21 && g.history.back().iter == 200, "sgd history on the stride grid");
    expect(g.apply_count == 200 && g.adjoint_count == 200, "sgd spends T applies and T adjoints");
  }
  {  // long rows (> 512 entries): the warp-specialised long-slice path
    SeededRng rng(102, 0);
    const ExplicitMatrix A = scaled_sparse(300, 1400, 0.01, 40, rng);
    EquilibrationParams p;
    p.iterations = 60;
    p.seed = 3;
    compare_scaling(b200::sgd_equilibrate(A, p), sgd_equilibrate(A, p), "sgd long rows");
  }
  {  // dense, badly scaled, box feasibility flags
    SeededRng rng(103, 0);
    const ExplicitMatrix A = ExplicitMatrix::dense(badly_scaled_dense(40, 25, rng));
    EquilibrationParams p;
    p.iterations = 150;
    p.max_log_scale = 2.0;  // tight box: the clamp is exercised
    const ScalingResult g = b200::sgd_equilibrate(A, p);
    compare_scaling(g, sgd_equilibrate(A, p), "sgd dense tight box");
  }
  {  // parameter errors: same type and message, in the reference's order
    const ExplicitMatrix I = ExplicitMatrix::identity(4);
    EquilibrationParams p;
    p.gamma = 0.0;
    same_throw<std::invalid_argument>([&] { b200::sgd_equilibrate(I, p); },
                                      [&] { sgd_equilibrate(I, p); }, "sgd gamma <= 0");
    EquilibrationParams q;
    q.iterations = -1;
    same_throw<std::invalid_argument>([&] { b200::sgd_equilibrate(I, q); },
                                      [&] { sgd_equilibrate(I, q); }, "sgd negative T");
    EquilibrationParams t;
    t.alpha = 1.0;
    t.beta = 3.0;  // m alpha^2 != n beta^2
    same_throw<std::invalid_argument>([&] { b200::sgd_equilibrate(I, t); },
                                      [&] { sgd_equilibrate(I, t); }, "sgd inconsistent targets");
    DiagnosticsConfig bad;
    bad.matrix = &I;
    bad.stride = 0;
    same_throw<std::invalid_argument>([&] { b200::sgd_equilibrate(I, EquilibrationParams{}, bad); },
                                      [&] { sgd_equilibrate(I, EquilibrationParams{}, bad); },
                                      "sgd stride 0");
  }
}

void lsqr_cases() {
  {  // identity: one iteration
    SeededRng rng(81, 0);
    const Vec b = gaussian_vec(6, rng);
    const ExplicitMatrix I = ExplicitMatrix::identity(6);
    const LsqrRun g = b200::lsqr(I, b, 10, 1e-12);
    compare_lsqr(g, lsqr(I, b, 10, 1e-12), "lsqr identity");
    expect(g.reached_tol && g.iterations == 1 && g.residual_history.size() == 2,
           "lsqr identity: one iteration");
  }
  {  // diagonal system
    Mat D = Mat::Zero(5, 5);
    for (Index i = 0; i < 5; ++i) D(i, i) = static_cast<double>(i + 1);
    const ExplicitMatrix A = ExplicitMatrix::dense(D);
    Vec b(5);
    for (Index i = 0; i < 5; ++i) b[i] = static_cast<double>(i + 1);
    const LsqrRun g = b200::lsqr(A, b, 10, 1e-13);
    compare_lsqr(g, lsqr(A, b, 10, 1e-13), "lsqr diagonal");
    expect(g.reached_tol && g.iterations <= 5, "lsqr diagonal: converges within n iterations");
  }
  {  // random square system, monotone residuals, charged counts
    SeededRng rng(82, 0);
    const ExplicitMatrix A = ExplicitMatrix::dense(gaussian(30, 30, rng));
    const Vec b = gaussian_vec(30, rng);
    const LsqrRun g = b200::lsqr(A, b, 60, 1e-10);
    compare_lsqr(g, lsqr(A, b, 60, 1e-10), "lsqr random 30x30");
    bool mono = true;
    for (size_t k = 1; k < g.residual_history.size(); ++k)
      mono = mono && g.residual_history[k] <= g.residual_history[k - 1] * (1 + 1e-12);
    expect(mono, "lsqr random: residuals decrease");
    expect(g.apply_count == g.iterations && g.adjoint_count == g.iterations + 1,
           "lsqr: one apply + one adjoint per iteration, one adjoint at setup");
  }
  {  // sparse with long rows
    SeededRng rng(84, 0);
    const ExplicitMatrix A = scaled_sparse(200, 1200, 0.02, 30, rng);
    const Vec b = gaussian_vec(200, rng);
    compare_lsqr(b200::lsqr(A, b, 80, 0.0), lsqr(A, b, 80, 0.0), "lsqr sparse long rows");
    EquilibrationParams p;
    p.iterations = 40;
    compare_lsqr(b200::lsqr_preconditioned(A, b, p, 80, 0.0),
                 lsqr_preconditioned(A, b, p, 80, 0.0), "lsqr_preconditioned sparse long rows");
  }
  {  // zero right-hand side and negative max_iters
    const ExplicitMatrix I = ExplicitMatrix::identity(3);
    const Vec z = Vec::Zero(3);
    same_throw<std::invalid_argument>([&] { b200::lsqr(I, z, 5, 0.0); },
                                      [&] { lsqr(I, z, 5, 0.0); }, "lsqr zero rhs");
    same_throw<std::invalid_argument>(
        [&] { b200::lsqr_preconditioned(I, z, EquilibrationParams{}, 5, 0.0); },
        [&] { lsqr_preconditioned(I, z, EquilibrationParams{}, 5, 0.0); },
        "lsqr_preconditioned zero rhs");
    const Vec o = Vec::Ones(3);
    same_throw<std::invalid_argument>([&] { b200::lsqr(I, o, -1, 0.0); },
                                      [&] { lsqr(I, o, -1, 0.0); }, "lsqr negative max_iters");
  }
  {  // breakdown: b orthogonal to the range of A (A^T b = 0)
    Mat a = Mat::Zero(3, 2);
    a(0, 0) = 1.0;
    a(1, 1) = 2.0;
    const ExplicitMatrix A = ExplicitMatrix::dense(a);
    Vec b = Vec::Zero(3);
    b[2] = 1.0;
    const LsqrRun g = b200::lsqr(A, b, 10, 0.0);
    compare_lsqr(g, lsqr(A, b, 10, 0.0), "lsqr breakdown");
    expect(g.breakdown, "lsqr breakdown flagged");
  }
  {  // singular (rank-deficient) system: the least-squares solution
    Mat a = Mat::Zero(4, 3);
    a(0, 0) = 1.0;
    a(1, 0) = 1.0;
    a(2, 1) = 2.0;
    a(3, 1) = 1.0;  // column 2 is zero
    const ExplicitMatrix A = ExplicitMatrix::dense(a);
    Vec b(4);
    b[0] = 1.0;
    b[1] = 3.0;
    b[2] = -1.0;
    b[3] = 2.0;
    compare_lsqr(b200::lsqr(A, b, 20, 0.0), lsqr(A, b, 20, 0.0), "lsqr singular");
  }
  {  // zero equilibration budget: the preconditioned run is the plain run
    SeededRng rng(85, 0);
    const ExplicitMatrix A = ExplicitMatrix::dense(gaussian(25, 12, rng));
    const Vec b = gaussian_vec(25, rng);
    EquilibrationParams p;
    p.iterations = 0;
    const LsqrRun g0 = b200::lsqr_preconditioned(A, b, p, 30, 0.0);
    compare_lsqr(g0, lsqr_preconditioned(A, b, p, 30, 0.0), "lsqr_preconditioned T=0");
    const LsqrRun gp = b200::lsqr(A, b, 30, 0.0);
    expect(same_bits(g0.x, gp.x) && same_bits(g0.residual_history, gp.residual_history),
           "lsqr_preconditioned T=0 equals plain lsqr");
  }
  {  // badly scaled, consistent rhs: the preconditioned run reaches the
     // tolerance in under half the charged iterations (test_itersolvers.cpp:158-171)
    SeededRng rng(86, 0);
    const ExplicitMatrix A = ExplicitMatrix::dense(badly_scaled_dense(120, 80, rng));
    const Vec b = A.apply(gaussian_vec(80, rng));
    EquilibrationParams p;
    p.iterations = 30;
    p.seed = 1;
    const b200::Device dev(A);
    const LsqrRun g = b200::lsqr(dev, b, 4000, 1e-8);
    const LsqrRun gp = b200::lsqr_preconditioned(dev, b, p, 4000, 1e-8);
    compare_lsqr(g, lsqr(A, b, 4000, 1e-8), "lsqr badly scaled");
    compare_lsqr(gp, lsqr_preconditioned(A, b, p, 4000, 1e-8), "lsqr_preconditioned badly scaled");
    const int tp = gp.reached_tol ? gp.equil_iterations + gp.iterations : 1 << 30;
    const int t0 = g.reached_tol ? g.iterations : 1 << 30;
    expect(gp.reached_tol && 2 * tp < t0,
           "preconditioning beats plain lsqr on a badly scaled system (" + std::to_string(tp) +
               " vs " + std::to_string(t0) + " iterations)");
  }
}

void operator_case() {
  // a matrix-free operator (the reference's plugin interface): B = A diag(c),
  // applied as A (c .* x) / c .* A^T y -- no explicit form exists; the device
  // loop around its own apply must reproduce the reference's run bit for bit
  struct ColumnScaled final : LinearOperator {
    const ExplicitMatrix* A;
    Vec c;
    Index rows() const override { return A->rows(); }
    Index cols() const override { return A->cols(); }
    Vec apply(const Vec& x) const override {
      Vec t(x.size());
      for (Index j = 0; j < x.size(); ++j) t[j] = c[j] * x[j];
      return A->apply(t);
    }
    Vec apply_adjoint(const Vec& y) const override {
      Vec z = A->apply_adjoint(y);
      for (Index j = 0; j < z.size(); ++j) z[j] = c[j] * z[j];
      return z;
    }
  };
  SeededRng rng(107, 0);
  const ExplicitMatrix A = scaled_sparse(80, 50, 0.1, 0, rng);
  ColumnScaled op;
  op.A = &A;
  op.c = Vec(50);
  for (Index j = 0; j < 50; ++j) op.c[j] = std::exp(rng.normal());
  EquilibrationParams p;
  p.iterations = 120;
  p.seed = 9;
  const ScalingResult g = b200::sgd_equilibrate(op, p);
  compare_scaling(g, sgd_equilibrate(op, p), "sgd matrix-free operator");
  const Vec b = gaussian_vec(80, rng);
  compare_lsqr(b200::lsqr(op, b, 40, 0.0), lsqr(op, b, 40, 0.0), "lsqr matrix-free operator");
  EquilibrationParams q;
  q.iterations = 25;
  compare_lsqr(b200::lsqr_preconditioned(op, b, q, 40, 0.0), lsqr_preconditioned(op, b, q, 40, 0.0),
               "lsqr_preconditioned matrix-free operator");
}

}  // namespace

int main() {
  try {
    sgd_cases();
    lsqr_cases();
    operator_case();
  } catch (const std::exception& e) {
    std::printf("FAIL: unexpected exception: %s\n", e.what());
    return 2;
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  if (g_fail) return 1;
  std::printf("OK\n");
  return 0;
}
