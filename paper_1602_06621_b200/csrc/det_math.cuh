// det_math.cuh -- the numerics contract, compiled for host and device.
//
// The reference delegates exactly three operations to Eigen (SURVEY.md §0
// fact 6): .array().exp() (src/equilibrate.cpp:162-163,203-204), the
// reductions behind .norm()/.dot() (src/lsqr.cpp:23,26,40,50,97,131) and the
// dense GEMV (src/explicit_matrix.cpp:69,84).  Eigen is absent, so those three
// are DEFINED here; every other operation on the
// path is the reference's own scalar arithmetic.  The oracle restates the same
// definitions independently (oracle/equil_oracle.c) and the tests compare the
// two.  All arithmetic is explicitly round-to-nearest with no contraction
// (__dmul_rn/__dadd_rn on device; the host side is compiled with
// -ffp-contract=off).
#pragma once

#include <cstdint>
#include <cstring>
#include <cmath>

#if defined(__CUDACC__)
#define EQ_HD __host__ __device__ __forceinline__
#else
#define EQ_HD inline
#endif

namespace eqb {

// -- exact round-to-nearest primitives ------------------------------------
EQ_HD double rn_mul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
EQ_HD double rn_add(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
EQ_HD double rn_sub(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
EQ_HD double rn_div(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __ddiv_rn(a, b);
#else
  return a / b;
#endif
}
EQ_HD double bits_to_double(uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double(static_cast<long long>(b));
#else
  double d;
  std::memcpy(&d, &b, 8);
  return d;
#endif
}

// -- det_exp ----------------------------------------------------------------
// exp(x) by Cody-Waite reduction with ln2 = C1 + C2 and the Cephes rational
// form exp(r) = 1 + 2 r P(r^2) / (Q(r^2) - r P(r^2)); 2^k applied in two
// exact halves.  Every step is one correctly rounded IEEE operation, so host
// and device agree bit for bit.
EQ_HD double det_exp(double x) {
  if (x != x) return x;
  if (x > 709.78) x = 709.78;
  if (x < -708.39) x = -708.39;
  const double fx = floor(rn_add(rn_mul(1.4426950408889634073599, x), 0.5));
  double r = rn_sub(x, rn_mul(fx, 6.93145751953125E-1));
  r = rn_sub(r, rn_mul(fx, 1.42860682030941723212E-6));
  const double rr = rn_mul(r, r);
  double px = 1.26177193074810590878E-4;
  px = rn_add(rn_mul(px, rr), 3.02994407707441961300E-2);
  px = rn_add(rn_mul(px, rr), 9.99999999999999999910E-1);
  px = rn_mul(px, r);
  double qx = 3.00198505138664455042E-6;
  qx = rn_add(rn_mul(qx, rr), 2.52448340349684104192E-3);
  qx = rn_add(rn_mul(qx, rr), 2.27265548208155028766E-1);
  qx = rn_add(rn_mul(qx, rr), 2.00000000000000000009E0);
  double y = rn_div(px, rn_sub(qx, px));
  y = rn_add(rn_mul(2.0, y), 1.0);
  const int k = static_cast<int>(fx);
  const int k1 = k / 2;
  const int k2 = k - k1;
  const double s1 = bits_to_double(static_cast<uint64_t>(k1 + 1023) << 52);
  const double s2 = bits_to_double(static_cast<uint64_t>(k2 + 1023) << 52);
  return rn_mul(rn_mul(y, s1), s2);
}

// -- canonical reduction tree ------------------------------------------------
// level 1: chunks of kChunk consecutive terms; lane l of kLanes1 sums terms
//          l, l+kLanes1, ... sequentially from +0.0; lanes fold pairwise
//          s[l] += s[l+h] for h = kLanes1/2 .. 1.
// level 2: the chunk results, folded the same way over kLanes2 lanes.
// Partials that start at +0.0 are never -0.0, so lanes without terms (or
// padded +0.0 terms) leave every fold step unchanged.
constexpr int kChunk = 2048;
constexpr int kLanes1 = 256;
constexpr int kLanes2 = 1024;

// -- per-iteration SGD scalars (src/equilibrate.cpp:106-107) ----------------
struct SgdStep {
  double step;  // 2.0 / (gamma * (t + 1))
  double aw;    // 2.0 / (t + 2.0)
  double aw1;   // 1.0 - aw
  double pad;
};

// Per-block constants of run_projected_sgd (:113-126).
struct SgdBlockConst {
  double lin;     // alpha^2 or beta^2
  double gamma;
  double M;       // max_log_scale
  double thresh;  // cap + 1e-9 * max(1, |cap|), cap = lin / gamma
};

// One coordinate update of run_projected_sgd (:113-128); returns new x, sets
// flag bits (1 = iterate bound violated, 2 = box violated).
EQ_HD double sgd_coord(double est, double x, const SgdBlockConst& c,
                       const SgdStep& s, double& avg, unsigned& flags) {
  const double g = rn_add(rn_sub(est, c.lin), rn_mul(c.gamma, x));
  double xi = rn_sub(x, rn_mul(s.step, g));
  const double negM = -c.M;
  xi = (xi < negM) ? negM : xi;  // std::max(xi, -M)
  xi = (c.M < xi) ? c.M : xi;    // std::min(xi, M)
  if (xi > c.thresh) flags |= 1u;
  if (fabs(xi) > c.M) flags |= 2u;
  avg = rn_add(rn_mul(s.aw, xi), rn_mul(s.aw1, avg));
  return xi;
}

// The same update with a per-coordinate linear term lin_i (nonuniform targets,
// src/variants.cpp:105-118 -> sgd_row_col); the iterate-bound threshold is
// formed per coordinate exactly as run_projected_sgd does (:122-125).
EQ_HD double sgd_coord_lin(double est, double x, double lin, const SgdBlockConst& c,
                           const SgdStep& s, double& avg, unsigned& flags) {
  const double g = rn_add(rn_sub(est, lin), rn_mul(c.gamma, x));
  double xi = rn_sub(x, rn_mul(s.step, g));
  const double negM = -c.M;
  xi = (xi < negM) ? negM : xi;
  xi = (c.M < xi) ? c.M : xi;
  const double cap = rn_div(lin, c.gamma);
  const double acap = fabs(cap);
  if (xi > rn_add(cap, rn_mul(1e-9, (1.0 < acap) ? acap : 1.0))) flags |= 1u;
  if (fabs(xi) > c.M) flags |= 2u;
  avg = rn_add(rn_mul(s.aw, xi), rn_mul(s.aw1, avg));
  return xi;
}

}  // namespace eqb
