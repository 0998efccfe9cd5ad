/*
 * equil_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see equil_oracle.h).  Plain C11, compiled with
 * -O2 -ffp-contract=off and no -march flags so every double operation is one
 * IEEE-754 round-to-nearest operation, exactly like the reference built with
 * its default flags (CMakeLists.txt:3-8: no -march, no -ffast-math).
 *
 * Reference paths are relative to /root/reference/proj/.
 */
#include "equil_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[512];
const char* eo_last_error(void) { return g_err; }
static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return 1;
}

/* ========================================================================== */
/* RNG: splitmix64-mixed std::mt19937_64 (src/rng.cpp:9-64)                   */
/* ========================================================================== */

#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x000000007FFFFFFFULL

static uint64_t splitmix64(uint64_t* state) { /* src/rng.cpp:9-15 */
  *state += 0x9E3779B97F4A7C15ULL;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* std::mersenne_twister_engine<uint64_t,64,312,156,31,...>::seed(v):
 * x0 = v, x_i = f * (x_{i-1} xor (x_{i-1} >> 62)) + i, f = 6364136223846793005 */
void eo_mt64_seed(eo_rng* r, uint64_t v) {
  r->mt[0] = v;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) +
               (uint64_t)i;
  r->mti = MT_N;
  r->has_spare = 0;
  r->spare = 0.0;
}

uint64_t eo_mixed_seed(uint64_t seed, uint64_t stream) { /* rng.cpp:19-27 */
  uint64_t state = seed;
  uint64_t mixed = splitmix64(&state);
  state ^= stream * 0xD1B54A32D192ED03ULL + 0x2545F4914F6CDD1DULL;
  mixed ^= splitmix64(&state);
  return mixed;
}

void eo_rng_init(eo_rng* r, uint64_t seed, uint64_t stream) {
  eo_mt64_seed(r, eo_mixed_seed(seed, stream));
}

static void mt_twist(eo_rng* r) {
  for (int i = 0; i < MT_N; ++i) {
    uint64_t x = (r->mt[i] & MT_UM) | (r->mt[(i + 1) % MT_N] & MT_LM);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= MT_A;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
  }
  r->mti = 0;
}

static uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

uint64_t eo_rng_next_u64(eo_rng* r) { /* rng.cpp:29 */
  if (r->mti >= MT_N) mt_twist(r);
  return mt_temper(r->mt[r->mti++]);
}

double eo_rng_uniform01(eo_rng* r) { /* rng.cpp:31-34 */
  return ((double)(eo_rng_next_u64(r) >> 11) + 0.5) * 0x1.0p-53;
}

double eo_rng_sign(eo_rng* r) { /* rng.cpp:36 */
  return (eo_rng_next_u64(r) >> 63) ? 1.0 : -1.0;
}

double eo_rng_normal(eo_rng* r) { /* rng.cpp:38-49 (glibc log/sin/cos) */
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u1 = eo_rng_uniform01(r);
  double u2 = eo_rng_uniform01(r);
  double rr = sqrt(-2.0 * log(u1));
  double theta = 6.283185307179586476925286766559 * u2;
  r->spare = rr * sin(theta);
  r->has_spare = 1;
  return rr * cos(theta);
}

uint64_t eo_rng_uniform_index(eo_rng* r, uint64_t n) { /* rng.cpp:51-57 */
  return eo_rng_next_u64(r) % n;
}

void eo_rng_state(uint64_t seed, uint64_t stream, uint64_t* out312) {
  eo_rng r;
  eo_rng_init(&r, seed, stream);
  memcpy(out312, r.mt, sizeof r.mt);
}

void eo_raw_outputs(uint64_t seed, uint64_t stream, uint64_t start,
                    uint64_t count, uint64_t* out) {
  eo_rng r;
  eo_rng_init(&r, seed, stream);
  for (uint64_t k = 0; k < start; ++k) (void)eo_rng_next_u64(&r);
  for (uint64_t k = 0; k < count; ++k) out[k] = eo_rng_next_u64(&r);
}

void eo_sign_bits(uint64_t seed, uint64_t stream, uint64_t start,
                  uint64_t count, uint32_t* bits_out) {
  eo_rng r;
  eo_rng_init(&r, seed, stream);
  for (uint64_t k = 0; k < start; ++k) (void)eo_rng_next_u64(&r);
  memset(bits_out, 0, ((count + 31) / 32) * sizeof(uint32_t));
  for (uint64_t k = 0; k < count; ++k)
    if (eo_rng_next_u64(&r) >> 63) bits_out[k >> 5] |= 1u << (k & 31);
}

/* ========================================================================== */
/* Numerics contract (shim-defined; restated independently in the product's   */
/* csrc/det_math.cuh and checked against this file by tests).                 */
/* ========================================================================== */

/* det_exp: Cody-Waite reduction by ln2 split in two parts, then the Cephes
 * (S. Moshier) rational approximation exp(r) = 1 + 2 r P(r^2)/(Q(r^2) - r P(r^2)),
 * the same scheme Eigen's packet exp uses on SSE2 (no FMA: every multiply and
 * add is separately rounded).  Scaling by 2^k is done in two exact halves.  */
double eo_det_exp(double x) {
  if (x != x) return x;
  if (x > 709.78) x = 709.78;
  if (x < -708.39) x = -708.39;
  double fx = floor(1.4426950408889634073599 * x + 0.5);
  double r = x - fx * 6.93145751953125E-1;
  r = r - fx * 1.42860682030941723212E-6;
  double rr = r * r;
  double px = 1.26177193074810590878E-4;
  px = px * rr + 3.02994407707441961300E-2;
  px = px * rr + 9.99999999999999999910E-1;
  px = px * r;
  double qx = 3.00198505138664455042E-6;
  qx = qx * rr + 2.52448340349684104192E-3;
  qx = qx * rr + 2.27265548208155028766E-1;
  qx = qx * rr + 2.00000000000000000009E0;
  double y = px / (qx - px);
  y = 2.0 * y + 1.0;
  int k = (int)fx;
  int k1 = k / 2;
  int k2 = k - k1;
  uint64_t b1 = (uint64_t)(k1 + 1023) << 52, b2 = (uint64_t)(k2 + 1023) << 52;
  double s1, s2;
  memcpy(&s1, &b1, 8);
  memcpy(&s2, &b2, 8);
  return (y * s1) * s2;
}

/* Canonical reduction tree (replaces Eigen's redux order, which is internal to
 * Eigen and not reproducible here):
 *   level 1: chunks of 2048 consecutive terms; in a chunk, lane l (0..255)
 *            sums terms l, l+256, ... sequentially from +0.0, then the 256
 *            lane sums fold pairwise s[l] += s[l+h], h = 128, 64, ..., 1;
 *   level 2: chunk results folded the same way with 1024 lanes.
 * A term is one rounded product where the reduction is a dot/sum of squares. */
#define EO_CHUNK 2048
#define EO_L1 256
#define EO_L2 1024

typedef double (*eo_term_fn)(const double*, const double*, int64_t);
static double t_sum(const double* a, const double* b, int64_t k) {
  (void)b;
  return a[k];
}
static double t_sq(const double* a, const double* b, int64_t k) {
  (void)b;
  return a[k] * a[k];
}
static double t_dot(const double* a, const double* b, int64_t k) {
  return a[k] * b[k];
}

static double fold(double* s, int lanes) {
  for (int h = lanes / 2; h >= 1; h >>= 1)
    for (int l = 0; l < h; ++l) s[l] = s[l] + s[l + h];
  return s[0];
}

static double canon(const double* a, const double* b, int64_t len,
                    eo_term_fn term) {
  if (len <= 0) return 0.0;
  int64_t nc = (len + EO_CHUNK - 1) / EO_CHUNK;
  double* part = (double*)malloc((size_t)nc * sizeof(double));
  double s1[EO_L1];
  for (int64_t c = 0; c < nc; ++c) {
    int64_t base = c * EO_CHUNK;
    int64_t clen = len - base < EO_CHUNK ? len - base : EO_CHUNK;
    for (int l = 0; l < EO_L1; ++l) {
      double acc = 0.0;
      for (int64_t k = l; k < clen; k += EO_L1) acc = acc + term(a, b, base + k);
      s1[l] = acc;
    }
    part[c] = fold(s1, EO_L1);
  }
  double* s2 = (double*)malloc(EO_L2 * sizeof(double));
  for (int l = 0; l < EO_L2; ++l) {
    double acc = 0.0;
    for (int64_t k = l; k < nc; k += EO_L2) acc = acc + part[k];
    s2[l] = acc;
  }
  double r = fold(s2, EO_L2);
  free(s2);
  free(part);
  return r;
}

double eo_canon_sum(const double* p, int64_t len) {
  return canon(p, NULL, len, t_sum);
}
double eo_canon_sumsq(const double* p, int64_t len) {
  return canon(p, NULL, len, t_sq);
}
double eo_canon_dot(const double* a, const double* b, int64_t len) {
  return canon(a, b, len, t_dot);
}

/* ========================================================================== */
/* Matrix store (src/explicit_matrix.cpp)                                     */
/* ========================================================================== */

/* transposed() (:117-125) emits {j, i, v} in CSR order (i ascending) and
 * sparse() (:19-57) sorts by (j, i): i.e. a stable counting sort by column. */
void eo_csr_transpose(int64_t m, int64_t n, const int64_t* row_ptr,
                      const int32_t* col, const double* val, int64_t* t_row_ptr,
                      int32_t* t_col, double* t_val) {
  int64_t nnz = row_ptr[m];
  memset(t_row_ptr, 0, (size_t)(n + 1) * sizeof(int64_t));
  for (int64_t k = 0; k < nnz; ++k) t_row_ptr[col[k] + 1]++;
  for (int64_t j = 0; j < n; ++j) t_row_ptr[j + 1] += t_row_ptr[j];
  int64_t* pos = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  memcpy(pos, t_row_ptr, (size_t)(n + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < m; ++i)
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      int64_t p = pos[col[k]]++;
      t_col[p] = (int32_t)i;
      t_val[p] = val[k];
    }
  free(pos);
}

void eo_csr_apply(int64_t m, const int64_t* row_ptr, const int32_t* col,
                  const double* val, const double* x, double* y) {
  for (int64_t i = 0; i < m; ++i) { /* :70-78 */
    double acc = 0.0;
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k)
      acc += val[k] * x[col[k]];
    y[i] = acc;
  }
}

void eo_csr_apply_adjoint(int64_t m, int64_t n, const int64_t* row_ptr,
                          const int32_t* col, const double* val,
                          const double* y, double* x) {
  for (int64_t j = 0; j < n; ++j) x[j] = 0.0; /* :85-92 */
  for (int64_t i = 0; i < m; ++i) {
    double yi = y[i];
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k)
      x[col[k]] += val[k] * yi;
  }
}

void eo_dense_apply(int64_t m, int64_t n, const double* A, const double* x,
                    double* y) {
  for (int64_t i = 0; i < m; ++i) y[i] = eo_canon_dot(A + i * n, x, n);
}

void eo_dense_apply_adjoint(int64_t m, int64_t n, const double* A,
                            const double* y, double* x) {
  double* colv = (double*)malloc((size_t)m * sizeof(double));
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t i = 0; i < m; ++i) colv[i] = A[i * n + j];
    x[j] = eo_canon_dot(colv, y, m);
  }
  free(colv);
}

static void mat_apply(const eo_matrix* A, const double* x, double* y) {
  if (A->dense)
    eo_dense_apply(A->m, A->n, A->dense, x, y);
  else
    eo_csr_apply(A->m, A->row_ptr, A->col, A->val, x, y);
}
static void mat_adjoint(const eo_matrix* A, const double* y, double* x) {
  if (A->dense)
    eo_dense_apply_adjoint(A->m, A->n, A->dense, y, x);
  else
    eo_csr_apply_adjoint(A->m, A->n, A->row_ptr, A->col, A->val, y, x);
}

/* ========================================================================== */
/* Params (src/params.cpp:7-44)                                               */
/* ========================================================================== */

int eo_resolve_targets(const eo_params* p, int64_t rows, int64_t cols,
                       double* alpha_out, double* beta_out) {
  if (!(rows > 0 && cols > 0))
    return fail("resolve_targets: dimensions must be positive");
  if (!(p->alpha >= 0.0 && p->beta >= 0.0))
    return fail("resolve_targets: targets must be positive (or 0 for auto)");
  const double m = (double)rows, n = (double)cols;
  double alpha = p->alpha, beta = p->beta;
  if (alpha == 0.0 && beta == 0.0) {
    alpha = pow(n / m, 0.25);
    beta = pow(m / n, 0.25);
  } else if (beta == 0.0) {
    beta = alpha * sqrt(m / n);
  } else if (alpha == 0.0) {
    alpha = beta * sqrt(n / m);
  } else {
    const double lhs = m * alpha * alpha;
    const double rhs = n * beta * beta;
    const double mx = lhs < rhs ? rhs : lhs;
    if (!(fabs(lhs - rhs) <= 1e-8 * mx))
      return fail("resolve_targets: m*alpha^2 == n*beta^2 violated");
  }
  *alpha_out = alpha;
  *beta_out = beta;
  return 0;
}

int eo_validate_params(const eo_params* p) {
  if (!(p->gamma > 0.0)) return fail("params: gamma must be positive");
  if (!(p->max_log_scale > 0.0))
    return fail("params: max_log_scale must be positive");
  if (!(p->iterations >= 0))
    return fail("params: iterations must be nonnegative");
  if (!(isfinite(p->gamma) && isfinite(p->max_log_scale)))
    return fail("params: gamma and max_log_scale must be finite");
  return 0;
}

/* ========================================================================== */
/* Diagnostics (src/equilibrate.cpp:10-22, src/metrics.cpp:24-56)            */
/* ========================================================================== */

#define FOR_EACH_ENTRY(A, BODY)                                             \
  do {                                                                      \
    if ((A)->dense) {                                                       \
      for (int64_t i_ = 0; i_ < (A)->m; ++i_)                               \
        for (int64_t j_ = 0; j_ < (A)->n; ++j_) {                           \
          const int64_t ei = i_, ej = j_;                                   \
          const double ea = (A)->dense[i_ * (A)->n + j_];                   \
          BODY;                                                             \
        }                                                                   \
    } else {                                                                \
      for (int64_t i_ = 0; i_ < (A)->m; ++i_)                               \
        for (int64_t k_ = (A)->row_ptr[i_]; k_ < (A)->row_ptr[i_ + 1]; ++k_) { \
          const int64_t ei = i_, ej = (A)->col[k_];                         \
          const double ea = (A)->val[k_];                                   \
          BODY;                                                             \
        }                                                                   \
    }                                                                       \
  } while (0)

/* objective_weighted with vector linear terms (src/equilibrate.cpp:10-22) */
static double objective_lin(const eo_matrix* A, const double* u, const double* v,
                            const double* lu, const double* lv, double gamma) {
  double quad = 0.0;
  FOR_EACH_ENTRY(A, {
    if (ea != 0.0) quad += ea * ea * exp(2.0 * (u[ei] + v[ej]));
  });
  double du = eo_canon_dot(lu, u, A->m);
  double dv = eo_canon_dot(lv, v, A->n);
  double su = eo_canon_sumsq(u, A->m), sv = eo_canon_sumsq(v, A->n);
  return 0.5 * quad - du - dv + 0.5 * gamma * (su + sv);
}

double eo_objective(const eo_matrix* A, const double* u, const double* v,
                    double alpha2, double beta2, double gamma) {
  /* lin_u.dot(u) with lin_u = alpha^2 * 1 */
  double* lu = (double*)malloc((size_t)A->m * sizeof(double));
  double* lv = (double*)malloc((size_t)A->n * sizeof(double));
  for (int64_t i = 0; i < A->m; ++i) lu[i] = alpha2;
  for (int64_t j = 0; j < A->n; ++j) lv[j] = beta2;
  const double r = objective_lin(A, u, v, lu, lv, gamma);
  free(lu);
  free(lv);
  return r;
}

double eo_rms_error(const eo_matrix* A, const double* u, const double* v,
                    double alpha, double beta) {
  const int64_t m = A->m, n = A->n;
  double* eu = (double*)malloc((size_t)m * sizeof(double));
  double* ev = (double*)malloc((size_t)n * sizeof(double));
  double* rs = (double*)calloc((size_t)m, sizeof(double));
  double* cs = (double*)calloc((size_t)n, sizeof(double));
  for (int64_t i = 0; i < m; ++i) eu[i] = eo_det_exp(2.0 * u[i]);
  for (int64_t j = 0; j < n; ++j) ev[j] = eo_det_exp(2.0 * v[j]);
  FOR_EACH_ENTRY(A, {
    const double t = ea * ea * eu[ei] * ev[ej];
    rs[ei] += t;
    cs[ej] += t;
  });
  double acc = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    const double dd = sqrt(rs[i]) - alpha;
    acc += dd * dd;
  }
  for (int64_t j = 0; j < n; ++j) {
    const double dd = sqrt(cs[j]) - beta;
    acc += dd * dd;
  }
  free(eu);
  free(ev);
  free(rs);
  free(cs);
  return sqrt(acc / (double)(m + n));
}

/* ========================================================================== */
/* SGD engine (src/equilibrate.cpp:79-221)                                    */
/* ========================================================================== */

/* One block update, run_projected_sgd :109-129. */
static void sgd_block(int64_t dim, double* x, double* avg, const double* est,
                      const double* lins, double gamma, double M, double step,
                      double aw, int* bound_ok, int* box_ok) {
  for (int64_t i = 0; i < dim; ++i) {
    const double lin = lins[i];
    const double g = est[i] - lin + gamma * x[i];
    double xi = x[i] - step * g;
    double lo = (xi < -M) ? -M : xi; /* std::max(xi, -M) */
    xi = (M < lo) ? M : lo;          /* std::min(., M)    */
    x[i] = xi;
    const double cap = lin / gamma;
    const double ac = fabs(cap);
    const double mx = (1.0 < ac) ? ac : 1.0;
    if (xi > cap + 1e-9 * mx) *bound_ok = 0;
    if (fabs(xi) > M) *box_ok = 0;
  }
  const double w1 = 1.0 - aw;
  for (int64_t i = 0; i < dim; ++i) avg[i] = aw * x[i] + w1 * avg[i];
}

/* internal::sgd_row_col (src/equilibrate.cpp:138-210) with per-coordinate
 * linear terms; alpha, beta > 0 enable the RMS diagnostic. */
static int sgd_row_col(const eo_matrix* A, const eo_params* p, const double* lin_u,
                       const double* lin_v, double alpha, double beta, int diag_stride,
                       eo_scaling* out);

int eo_sgd_equilibrate(const eo_matrix* A, const eo_params* p, int diag_stride,
                       eo_scaling* out) {
  double alpha, beta;
  if (eo_resolve_targets(p, A->m, A->n, &alpha, &beta)) return 1; /* :216 */
  double* lu = (double*)malloc((size_t)A->m * sizeof(double));
  double* lv = (double*)malloc((size_t)A->n * sizeof(double));
  for (int64_t i = 0; i < A->m; ++i) lu[i] = alpha * alpha; /* :218-220 */
  for (int64_t j = 0; j < A->n; ++j) lv[j] = beta * beta;
  const int rc = sgd_row_col(A, p, lu, lv, alpha, beta, diag_stride, out);
  free(lu);
  free(lv);
  return rc;
}

/* sgd_equilibrate_targets (src/variants.cpp:105-118) */
int eo_sgd_equilibrate_targets(const eo_matrix* A, const double* r, const double* c,
                               const eo_params* p, int diag_stride, eo_scaling* out) {
  for (int64_t i = 0; i < A->m; ++i)
    if (!(r[i] > 0.0)) return fail("sgd_equilibrate_targets: targets must be positive");
  for (int64_t j = 0; j < A->n; ++j)
    if (!(c[j] > 0.0)) return fail("sgd_equilibrate_targets: targets must be positive");
  const double sr = eo_canon_sum(r, A->m), sc = eo_canon_sum(c, A->n);
  const double mx = sr < sc ? sc : sr;
  if (!(fabs(sr - sc) <= 1e-8 * mx))
    return fail("sgd_equilibrate_targets: sum(r) == sum(c) violated");
  return sgd_row_col(A, p, r, c, 0.0, 0.0, diag_stride, out);
}

static int sgd_row_col(const eo_matrix* A, const eo_params* p, const double* lin_u,
                       const double* lin_v, double alpha, double beta, int diag_stride,
                       eo_scaling* out) {
  if (eo_validate_params(p)) return 1; /* :142 */
  if (diag_stride < 0) return fail("sgd_row_col: stride must be positive");
  const int64_t m = A->m, n = A->n;
  const double gamma = p->gamma, M = p->max_log_scale;
  const int T = p->iterations;

  double* u = (double*)calloc((size_t)m, sizeof(double));
  double* v = (double*)calloc((size_t)n, sizeof(double));
  double* ub = (double*)calloc((size_t)m, sizeof(double));
  double* vb = (double*)calloc((size_t)n, sizeof(double));
  double* d = (double*)malloc((size_t)m * sizeof(double));
  double* e = (double*)malloc((size_t)n * sizeof(double));
  double* xs = (double*)malloc((size_t)n * sizeof(double));
  double* xw = (double*)malloc((size_t)m * sizeof(double));
  double* yu = (double*)malloc((size_t)m * sizeof(double));
  double* zv = (double*)malloc((size_t)n * sizeof(double));
  eo_rng rng;
  eo_rng_init(&rng, p->seed, 17); /* streams::kSgdProbes, :154 */
  int bound_ok = 1, box_ok = 1;
  out->hist_len = 0;

#define RECORD(t)                                                         \
  do {                                                                    \
    if (diag_stride > 0 && ((t) == 0 || (t) % diag_stride == 0)) {        \
      int h = out->hist_len++;                                            \
      if (out->hist_iter) out->hist_iter[h] = (t);                        \
      if (out->hist_objective)                                            \
        out->hist_objective[h] = objective_lin(A, ub, vb, lin_u, lin_v, gamma); \
      if (out->hist_rms)                                                  \
        out->hist_rms[h] = (alpha > 0.0 && beta > 0.0)                    \
                               ? eo_rms_error(A, ub, vb, alpha, beta) : 0.0; \
    }                                                                     \
  } while (0)

  RECORD(0);
  for (int t = 1; t <= T; ++t) {
    /* estimator, :160-167 */
    for (int64_t i = 0; i < m; ++i) d[i] = eo_det_exp(u[i]);
    for (int64_t j = 0; j < n; ++j) e[j] = eo_det_exp(v[j]);
    for (int64_t j = 0; j < n; ++j) xs[j] = e[j] * eo_rng_sign(&rng);
    mat_apply(A, xs, yu);
    for (int64_t i = 0; i < m; ++i) {
      const double y = d[i] * yu[i];
      yu[i] = y * y;
    }
    for (int64_t i = 0; i < m; ++i) xw[i] = d[i] * eo_rng_sign(&rng);
    mat_adjoint(A, xw, zv);
    for (int64_t j = 0; j < n; ++j) {
      const double z = e[j] * zv[j];
      zv[j] = z * z;
    }
    /* update, :106-129 */
    const double step = 2.0 / (gamma * (double)(t + 1));
    const double aw = 2.0 / ((double)t + 2.0);
    sgd_block(m, u, ub, yu, lin_u, gamma, M, step, aw, &bound_ok, &box_ok);
    sgd_block(n, v, vb, zv, lin_v, gamma, M, step, aw, &bound_ok, &box_ok);
    if (out->traj_u) memcpy(out->traj_u + (size_t)(t - 1) * m, u, m * 8);
    if (out->traj_v) memcpy(out->traj_v + (size_t)(t - 1) * n, v, n * 8);
    RECORD(t);
  }
#undef RECORD
  memcpy(out->u, ub, (size_t)m * 8); /* :201-204 */
  memcpy(out->v, vb, (size_t)n * 8);
  for (int64_t i = 0; i < m; ++i) out->d[i] = eo_det_exp(ub[i]);
  for (int64_t j = 0; j < n; ++j) out->e[j] = eo_det_exp(vb[j]);
  out->alpha = alpha;
  out->beta = beta;
  out->box_feasible = box_ok;
  out->iterate_bound_ok = bound_ok;
  out->apply_count = T;
  out->adjoint_count = T;
  free(u); free(v); free(ub); free(vb); free(d); free(e);
  free(xs); free(xw); free(yu); free(zv);
  return 0;
}

/* sgd_equilibrate_symmetric (src/variants.cpp:35-103).  check_symmetry
 * (:14-33): three probes of normals drawn on stream 18 (kSymmetryCheck),
 * <Ax, y> vs <x, Ay> with Eigen dot/norm -> canonical reductions. */
int eo_sgd_equilibrate_symmetric(const eo_matrix* A, const eo_params* p, int diag_stride,
                                 eo_scaling* out) {
  if (eo_validate_params(p)) return 1; /* :38 */
  if (A->m != A->n) return fail("sgd_equilibrate_symmetric: operator must be square");
  const int64_t n = A->n;
  {
    double* x = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
    double* y = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
    double* ax = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
    double* ay = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
    eo_rng r;
    eo_rng_init(&r, p->seed, 18);
    int ok = 1;
    for (int probe = 0; probe < 3 && ok; ++probe) {
      for (int64_t i = 0; i < n; ++i) x[i] = eo_rng_normal(&r);
      for (int64_t i = 0; i < n; ++i) y[i] = eo_rng_normal(&r);
      mat_apply(A, x, ax);
      mat_apply(A, y, ay);
      const double lhs = eo_canon_dot(ax, y, n);
      const double rhs = eo_canon_dot(x, ay, n);
      const double scale = sqrt(eo_canon_sumsq(ax, n)) * sqrt(eo_canon_sumsq(y, n)) +
                           sqrt(eo_canon_sumsq(x, n)) * sqrt(eo_canon_sumsq(ay, n)) + 1e-30;
      if (!(fabs(lhs - rhs) <= 1e-10 * scale)) ok = 0;
    }
    free(x); free(y); free(ax); free(ay);
    if (!ok) return fail("sgd_equilibrate_symmetric: operator failed symmetry check");
  }
  double alpha, beta;
  if (eo_resolve_targets(p, n, n, &alpha, &beta)) return 1; /* :41 */
  {
    const double mx = alpha < beta ? beta : alpha;
    if (!(fabs(alpha - beta) <= 1e-12 * mx))
      return fail("sgd_equilibrate_symmetric: targets must coincide");
  }
  if (diag_stride < 0) return fail("sgd_equilibrate_symmetric: stride must be positive");
  const double gamma = p->gamma, M = p->max_log_scale;
  const int T = p->iterations;
  double* u = (double*)calloc((size_t)(n ? n : 1), sizeof(double));
  double* ub = (double*)calloc((size_t)(n ? n : 1), sizeof(double));
  double* d = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
  double* xs = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
  double* yu = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
  double* lin = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
  for (int64_t i = 0; i < n; ++i) lin[i] = alpha * alpha; /* :56 */
  eo_rng rng;
  eo_rng_init(&rng, p->seed, 17);
  int bound_ok = 1, box_ok = 1;
  out->hist_len = 0;
#define SYM_RECORD(t)                                                         \
  do {                                                                        \
    if (diag_stride > 0 && ((t) == 0 || (t) % diag_stride == 0)) {            \
      int h = out->hist_len++;                                                \
      if (out->hist_iter) out->hist_iter[h] = (t);                            \
      if (out->hist_objective) /* :75-78, each unordered pair once */          \
        out->hist_objective[h] = 0.5 * objective_lin(A, ub, ub, lin, lin, gamma); \
      if (out->hist_rms) out->hist_rms[h] = eo_rms_error(A, ub, ub, alpha, alpha); \
    }                                                                         \
  } while (0)
  SYM_RECORD(0);
  for (int t = 1; t <= T; ++t) {
    /* estimator :60-64: d = exp(u); est = (d .* A (d .* s))^2, n draws */
    for (int64_t i = 0; i < n; ++i) d[i] = eo_det_exp(u[i]);
    for (int64_t j = 0; j < n; ++j) xs[j] = d[j] * eo_rng_sign(&rng);
    mat_apply(A, xs, yu);
    for (int64_t i = 0; i < n; ++i) {
      const double yy = d[i] * yu[i];
      yu[i] = yy * yy;
    }
    const double step = 2.0 / (gamma * (double)(t + 1));
    const double aw = 2.0 / ((double)t + 2.0);
    sgd_block(n, u, ub, yu, lin, gamma, M, step, aw, &bound_ok, &box_ok);
    SYM_RECORD(t);
  }
#undef SYM_RECORD
  memcpy(out->u, ub, (size_t)n * 8); /* :93-96 */
  memcpy(out->v, ub, (size_t)n * 8);
  for (int64_t i = 0; i < n; ++i) out->d[i] = eo_det_exp(ub[i]);
  memcpy(out->e, out->d, (size_t)n * 8);
  out->alpha = alpha;
  out->beta = alpha;
  out->box_feasible = box_ok;
  out->iterate_bound_ok = bound_ok;
  out->apply_count = T;
  out->adjoint_count = 0;
  free(u); free(ub); free(d); free(xs); free(yu); free(lin);
  return 0;
}

/* sgd_equilibrate_block (src/variants.cpp:156-240) with BlockStructure::validate
 * (:131-154).  Block estimates sum the members' row (column) estimates in
 * ascending index order starting from 0.0 (:190-193). */
int eo_sgd_equilibrate_block(const eo_matrix* A, const int64_t* rb, const int64_t* cb,
                             int64_t R, int64_t C, const eo_params* p, int diag_stride,
                             eo_scaling* out) {
  if (eo_validate_params(p)) return 1;
  const int64_t m = A->m, n = A->n;
  if (!(R > 0 && C > 0)) return fail("BlockStructure: block counts must be positive");
  for (int64_t i = 0; i < m; ++i)
    if (rb[i] < 0 || rb[i] >= R) return fail("BlockStructure: row block index out of range");
  for (int64_t j = 0; j < n; ++j)
    if (cb[j] < 0 || cb[j] >= C) return fail("BlockStructure: col block index out of range");
  double* rc = (double*)calloc((size_t)R, sizeof(double));
  double* cc = (double*)calloc((size_t)C, sizeof(double));
  for (int64_t i = 0; i < m; ++i) rc[rb[i]] += 1.0;
  for (int64_t j = 0; j < n; ++j) cc[cb[j]] += 1.0;
  for (int64_t b = 0; b < R; ++b)
    if (rc[b] == 0.0) {
      free(rc); free(cc);
      return fail("BlockStructure: empty row block");
    }
  for (int64_t b = 0; b < C; ++b)
    if (cc[b] == 0.0) {
      free(rc); free(cc);
      return fail("BlockStructure: empty col block");
    }
  double alpha, beta;
  if (eo_resolve_targets(p, m, n, &alpha, &beta)) {
    free(rc); free(cc);
    return 1;
  }
  if (diag_stride < 0) {
    free(rc); free(cc);
    return fail("sgd_equilibrate_block: stride must be positive");
  }
  const double gamma = p->gamma, M = p->max_log_scale;
  const int T = p->iterations;
  double* lu = (double*)malloc((size_t)R * sizeof(double));
  double* lv = (double*)malloc((size_t)C * sizeof(double));
  for (int64_t b = 0; b < R; ++b) lu[b] = (alpha * alpha) * rc[b]; /* :172-173 */
  for (int64_t b = 0; b < C; ++b) lv[b] = (beta * beta) * cc[b];
  double* xu = (double*)calloc((size_t)R, sizeof(double));
  double* xub = (double*)calloc((size_t)R, sizeof(double));
  double* xv = (double*)calloc((size_t)C, sizeof(double));
  double* xvb = (double*)calloc((size_t)C, sizeof(double));
  double* eu = (double*)malloc((size_t)R * sizeof(double));
  double* ev = (double*)malloc((size_t)C * sizeof(double));
  double* d = (double*)malloc((size_t)(m ? m : 1) * sizeof(double));
  double* e = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
  double* xs = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
  double* xw = (double*)malloc((size_t)(m ? m : 1) * sizeof(double));
  double* yu = (double*)malloc((size_t)(m ? m : 1) * sizeof(double));
  double* zv = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
  double* uf = (double*)malloc((size_t)(m ? m : 1) * sizeof(double));
  double* vf = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
  double* l1 = (double*)malloc((size_t)(m ? m : 1) * sizeof(double));
  double* l2 = (double*)malloc((size_t)(n ? n : 1) * sizeof(double));
  for (int64_t i = 0; i < m; ++i) l1[i] = alpha * alpha;
  for (int64_t j = 0; j < n; ++j) l2[j] = beta * beta;
  eo_rng rng;
  eo_rng_init(&rng, p->seed, 17);
  int bound_ok = 1, box_ok = 1;
  out->hist_len = 0;
#define BLK_RECORD(t)                                                         \
  do {                                                                        \
    if (diag_stride > 0 && ((t) == 0 || (t) % diag_stride == 0)) {            \
      for (int64_t i = 0; i < m; ++i) uf[i] = xub[rb[i]];                     \
      for (int64_t j = 0; j < n; ++j) vf[j] = xvb[cb[j]];                     \
      int h = out->hist_len++;                                                \
      if (out->hist_iter) out->hist_iter[h] = (t);                            \
      if (out->hist_objective)                                                \
        out->hist_objective[h] = objective_lin(A, uf, vf, l1, l2, gamma);     \
      if (out->hist_rms) out->hist_rms[h] = eo_rms_error(A, uf, vf, alpha, beta); \
    }                                                                         \
  } while (0)
  BLK_RECORD(0);
  for (int t = 1; t <= T; ++t) {
    /* estimator :181-194 */
    for (int64_t i = 0; i < m; ++i) d[i] = eo_det_exp(xu[rb[i]]);
    for (int64_t j = 0; j < n; ++j) e[j] = eo_det_exp(xv[cb[j]]);
    for (int64_t j = 0; j < n; ++j) xs[j] = e[j] * eo_rng_sign(&rng);
    mat_apply(A, xs, yu);
    for (int64_t i = 0; i < m; ++i) {
      const double yy = d[i] * yu[i];
      yu[i] = yy * yy;
    }
    for (int64_t i = 0; i < m; ++i) xw[i] = d[i] * eo_rng_sign(&rng);
    mat_adjoint(A, xw, zv);
    for (int64_t j = 0; j < n; ++j) {
      const double z = e[j] * zv[j];
      zv[j] = z * z;
    }
    for (int64_t b = 0; b < R; ++b) eu[b] = 0.0;
    for (int64_t b = 0; b < C; ++b) ev[b] = 0.0;
    for (int64_t i = 0; i < m; ++i) eu[rb[i]] += yu[i];
    for (int64_t j = 0; j < n; ++j) ev[cb[j]] += zv[j];
    const double step = 2.0 / (gamma * (double)(t + 1));
    const double aw = 2.0 / ((double)t + 2.0);
    sgd_block(R, xu, xub, eu, lu, gamma, M, step, aw, &bound_ok, &box_ok);
    sgd_block(C, xv, xvb, ev, lv, gamma, M, step, aw, &bound_ok, &box_ok);
    BLK_RECORD(t);
  }
#undef BLK_RECORD
  for (int64_t i = 0; i < m; ++i) out->u[i] = xub[rb[i]]; /* :226-229 */
  for (int64_t j = 0; j < n; ++j) out->v[j] = xvb[cb[j]];
  for (int64_t i = 0; i < m; ++i) out->d[i] = eo_det_exp(out->u[i]);
  for (int64_t j = 0; j < n; ++j) out->e[j] = eo_det_exp(out->v[j]);
  out->alpha = alpha;
  out->beta = beta;
  out->box_feasible = box_ok;
  out->iterate_bound_ok = bound_ok;
  out->apply_count = T;
  out->adjoint_count = T;
  free(rc); free(cc); free(lu); free(lv); free(xu); free(xub); free(xv); free(xvb);
  free(eu); free(ev); free(d); free(e); free(xs); free(xw); free(yu); free(zv);
  free(uf); free(vf); free(l1); free(l2);
  return 0;
}

/* ========================================================================== */
/* LSQR (src/lsqr.cpp:17-138)                                                 */
/* ========================================================================== */

typedef struct {
  const eo_matrix* A;
  const double* d; /* NULL: unscaled */
  const double* e;
  double* tmp_n;
  double* tmp_m;
  long long applies, adjoints;
} lsqr_op;

static void B_apply(lsqr_op* B, const double* x, double* y) { /* linop.cpp:17-20 */
  B->applies++;
  if (!B->d) {
    mat_apply(B->A, x, y);
    return;
  }
  for (int64_t j = 0; j < B->A->n; ++j) B->tmp_n[j] = B->e[j] * x[j];
  mat_apply(B->A, B->tmp_n, y);
  for (int64_t i = 0; i < B->A->m; ++i) y[i] = B->d[i] * y[i];
}

static void B_adjoint(lsqr_op* B, const double* y, double* x) { /* :22-26 */
  B->adjoints++;
  if (!B->d) {
    mat_adjoint(B->A, y, x);
    return;
  }
  for (int64_t i = 0; i < B->A->m; ++i) B->tmp_m[i] = B->d[i] * y[i];
  mat_adjoint(B->A, B->tmp_m, x);
  for (int64_t j = 0; j < B->A->n; ++j) x[j] = B->e[j] * x[j];
}

/* relative residual |b - A(e.x)| / |b| on the uncharged operator */
static double rel_residual(const eo_matrix* A, const double* b, double bnorm,
                           const double* e, const double* x, double* tmp_n,
                           double* tmp_m) {
  const double* xo = x;
  if (e) {
    for (int64_t j = 0; j < A->n; ++j) tmp_n[j] = e[j] * x[j];
    xo = tmp_n;
  }
  mat_apply(A, xo, tmp_m);
  for (int64_t i = 0; i < A->m; ++i) tmp_m[i] = b[i] - tmp_m[i];
  return sqrt(eo_canon_sumsq(tmp_m, A->m)) / bnorm;
}

static void lsqr_core(lsqr_op* B, const double* c, int max_iters, double tol,
                      const double* b, double bnorm, eo_lsqr_run* run,
                      double* x) {
  const int64_t m = B->A->m, n = B->A->n;
  double* u = (double*)malloc((size_t)m * 8);
  double* un = (double*)malloc((size_t)m * 8);
  double* v = (double*)malloc((size_t)n * 8);
  double* vn = (double*)malloc((size_t)n * 8);
  double* w = (double*)malloc((size_t)n * 8);
  double* rt_n = (double*)malloc((size_t)n * 8);
  double* rt_m = (double*)malloc((size_t)m * 8);
  for (int64_t j = 0; j < n; ++j) x[j] = 0.0;

  double beta = sqrt(eo_canon_sumsq(c, m)); /* :23 */
  for (int64_t i = 0; i < m; ++i) u[i] = c[i] / beta;
  B_adjoint(B, u, v);
  double alpha = sqrt(eo_canon_sumsq(v, n));
  if (alpha == 0.0) {
    run->breakdown = 1;
    goto done;
  }
  for (int64_t j = 0; j < n; ++j) v[j] = v[j] / alpha;
  memcpy(w, v, (size_t)n * 8);
  double phibar = beta, rhobar = alpha;

  for (int t = 1; t <= max_iters; ++t) { /* :36-80 */
    int invariant = 0;
    B_apply(B, v, un);
    for (int64_t i = 0; i < m; ++i) un[i] = un[i] - alpha * u[i];
    beta = sqrt(eo_canon_sumsq(un, m));
    if (beta > 0.0) {
      for (int64_t i = 0; i < m; ++i) u[i] = un[i] / beta;
    } else {
      invariant = 1;
    }
    alpha = 0.0;
    if (!invariant) {
      B_adjoint(B, u, vn);
      for (int64_t j = 0; j < n; ++j) vn[j] = vn[j] - beta * v[j];
      alpha = sqrt(eo_canon_sumsq(vn, n));
      if (alpha > 0.0) {
        for (int64_t j = 0; j < n; ++j) v[j] = vn[j] / alpha;
      } else {
        invariant = 1;
      }
    }
    const double rho = hypot(rhobar, beta);
    const double cs = rhobar / rho;
    const double sn = beta / rho;
    const double theta = sn * alpha;
    rhobar = -cs * alpha;
    const double phi = cs * phibar;
    phibar = sn * phibar;
    const double c1 = phi / rho, c2 = theta / rho;
    for (int64_t j = 0; j < n; ++j) x[j] = x[j] + c1 * w[j];
    for (int64_t j = 0; j < n; ++j) w[j] = v[j] - c2 * w[j];
    run->iterations = t;
    const double rel = rel_residual(B->A, b, bnorm, B->e, x, rt_n, rt_m);
    run->residual_history[run->hist_len++] = rel;
    if (rel <= tol) {
      run->reached_tol = 1;
      break;
    }
    if (invariant) {
      run->breakdown = 1;
      break;
    }
  }
done:
  free(u); free(un); free(v); free(vn); free(w); free(rt_n); free(rt_m);
}

int eo_lsqr(const eo_matrix* A, const double* b, int max_iters, double tol,
            eo_lsqr_run* run) { /* :85-103 */
  const double bnorm = sqrt(eo_canon_sumsq(b, A->m));
  if (!(bnorm > 0.0)) return fail("lsqr: rhs must be nonzero");
  if (!(max_iters >= 0)) return fail("lsqr: max_iters must be nonnegative");
  lsqr_op B = {A, NULL, NULL, NULL, NULL, 0, 0};
  run->hist_len = 0;
  run->iterations = 0;
  run->equil_iterations = 0;
  run->reached_tol = 0;
  run->breakdown = 0;
  run->residual_history[run->hist_len++] = 1.0;
  lsqr_core(&B, b, max_iters, tol, b, bnorm, run, run->x);
  run->apply_count = B.applies;
  run->adjoint_count = B.adjoints;
  return 0;
}

int eo_lsqr_preconditioned(const eo_matrix* A, const double* b,
                           const eo_params* p, int max_iters, double tol,
                           eo_lsqr_run* run) { /* :105-138 */
  const int64_t m = A->m, n = A->n;
  const double bnorm = sqrt(eo_canon_sumsq(b, m));
  if (!(bnorm > 0.0)) return fail("lsqr_preconditioned: rhs must be nonzero");
  if (!(max_iters >= 0))
    return fail("lsqr_preconditioned: max_iters must be nonnegative");
  eo_scaling sc;
  memset(&sc, 0, sizeof sc);
  double* su = (double*)malloc((size_t)m * 8);
  double* sv = (double*)malloc((size_t)n * 8);
  double* d = (double*)malloc((size_t)m * 8);
  double* e = (double*)malloc((size_t)n * 8);
  sc.u = su; sc.v = sv; sc.d = d; sc.e = e;
  if (eo_sgd_equilibrate(A, p, 0, &sc)) {
    free(su); free(sv); free(d); free(e);
    return 1;
  }
  run->hist_len = 0;
  run->iterations = 0;
  run->reached_tol = 0;
  run->breakdown = 0;
  run->equil_iterations = p->iterations;
  for (int t = 0; t <= p->iterations; ++t)
    run->residual_history[run->hist_len++] = 1.0;
  double* c = (double*)malloc((size_t)m * 8);
  for (int64_t i = 0; i < m; ++i) c[i] = d[i] * b[i];
  double* xs = (double*)malloc((size_t)n * 8);
  double* tn = (double*)malloc((size_t)n * 8);
  double* tm = (double*)malloc((size_t)m * 8);
  lsqr_op B = {A, d, e, tn, tm, 0, 0};
  lsqr_core(&B, c, max_iters, tol, b, bnorm, run, xs);
  for (int64_t j = 0; j < n; ++j) run->x[j] = e[j] * xs[j];
  run->apply_count = B.applies + sc.apply_count;
  run->adjoint_count = B.adjoints + sc.adjoint_count;
  if (run->d) memcpy(run->d, d, (size_t)m * 8);
  if (run->e) memcpy(run->e, e, (size_t)n * 8);
  free(c); free(xs); free(tn); free(tm);
  free(su); free(sv); free(d); free(e);
  return 0;
}

/* ========================================================================== */
/* spectral_norm (src/lsqr.cpp:140-163) and ccp_lasso (src/ccp.cpp:28-160)     */
/* ========================================================================== */

/* power iteration on B = diag(d) A diag(e) (d == NULL: A), uncharged */
static int spectral_norm_op(const eo_matrix* A, const double* d, const double* e,
                            int max_iters, double rel_tol, uint64_t seed, double* out) {
  if (max_iters <= 0) return fail("spectral_norm: max_iters must be positive");
  const int64_t m = A->m, n = A->n;
  double* x = (double*)malloc((size_t)(n ? n : 1) * 8);
  double* y = (double*)malloc((size_t)(m ? m : 1) * 8);
  double* z = (double*)malloc((size_t)(n ? n : 1) * 8);
  double* tn = (double*)malloc((size_t)(n ? n : 1) * 8);
  double* tm = (double*)malloc((size_t)(m ? m : 1) * 8);
  lsqr_op B = {A, d, e, tn, tm, 0, 0};
  eo_rng r;
  eo_rng_init(&r, seed, 19); /* streams::kPowerIteration */
  for (int64_t j = 0; j < n; ++j) x[j] = eo_rng_normal(&r);
  const double xn = sqrt(eo_canon_sumsq(x, n));
  int rc = 0;
  double lambda = 0.0;
  if (!(xn > 0.0)) {
    rc = fail("spectral_norm: degenerate start");
  } else {
    for (int64_t j = 0; j < n; ++j) x[j] = x[j] / xn;
    for (int t = 0; t < max_iters; ++t) {
      B_apply(&B, x, y);
      const double next = eo_canon_sumsq(y, m); /* Rayleigh quotient of A^T A */
      if (next == 0.0) {
        lambda = 0.0;
        break;
      }
      const int settled = fabs(next - lambda) <= rel_tol * next;
      lambda = next;
      if (settled) break;
      B_adjoint(&B, y, z);
      const double zn = sqrt(eo_canon_sumsq(z, n));
      if (zn == 0.0) break;
      for (int64_t j = 0; j < n; ++j) x[j] = z[j] / zn;
    }
  }
  *out = sqrt(lambda);
  free(x); free(y); free(z); free(tn); free(tm);
  return rc;
}

int eo_spectral_norm(const eo_matrix* A, int max_iters, double rel_tol, uint64_t seed,
                     double* out) {
  return spectral_norm_op(A, NULL, NULL, max_iters, rel_tol, seed, out);
}

/* |A x - b|^2 / sqrt(lambda) + sqrt(lambda) |x|_1 (src/ccp.cpp:115-123) */
double eo_lasso_objective(const eo_matrix* A, const double* b, double lambda, const double* x) {
  const int64_t m = A->m, n = A->n;
  const double sl = sqrt(lambda);
  double* r = (double*)malloc((size_t)(m ? m : 1) * 8);
  double* ax = (double*)malloc((size_t)(n ? n : 1) * 8);
  mat_apply(A, x, r);
  for (int64_t i = 0; i < m; ++i) r[i] = r[i] - b[i];
  for (int64_t j = 0; j < n; ++j) ax[j] = fabs(x[j]);
  const double f = eo_canon_sumsq(r, m) / sl + sl * eo_canon_sum(ax, n);
  free(r);
  free(ax);
  return f;
}

static double soft_threshold(double q, double t) { /* src/ccp.cpp:19-23 */
  if (q > t) return q - t;
  if (q < -t) return q + t;
  return 0.0;
}

static int ccp_validate(const eo_matrix* A, const double* b, double lambda,
                        const eo_ccp_options* o, const char* who) { /* :11-17 */
  if (!(lambda > 0.0)) return fail("lasso: lambda must be positive");
  if (!(sqrt(eo_canon_sumsq(b, A->m)) > 0.0)) return fail("lasso: rhs must be nonzero");
  if (o->max_iters < 0) {
    static char msg[128];
    snprintf(msg, sizeof msg, "%s: max_iters must be nonnegative", who);
    return fail(msg);
  }
  return 0;
}

/* ccp_core (src/ccp.cpp:27-110); d == NULL: plain run (d = e = 1) */
static int ccp_core(const eo_matrix* A, const double* b, double lambda, const double* d,
                    const double* e, int equil_iters, long long applies0, long long adjoints0,
                    const eo_ccp_options* o, eo_ccp_run* out) {
  const int64_t m = A->m, n = A->n;
  const double sl = sqrt(lambda);
  double tau, sigma;
  if (o->tau > 0.0 && o->sigma > 0.0) {
    tau = o->tau;
    sigma = o->sigma;
  } else {
    double norm2;
    if (spectral_norm_op(A, d, e, 100, 1e-9, 0, &norm2)) return 1;
    if (!(norm2 > 0.0)) return fail("ccp_lasso: zero operator");
    tau = 0.9 / norm2;
    sigma = 0.9 / norm2;
  }
  out->tau = tau;
  out->sigma = sigma;
  out->theta = o->theta;
  out->equil_iterations = equil_iters;
  out->iterations = 0;
  out->reached_tol = 0;
  out->hist_len = 0;
  out->gap_len = 0;
  double* zero = (double*)calloc((size_t)(n ? n : 1), 8);
  const double f0 = eo_lasso_objective(A, b, lambda, zero);
  const int track = isfinite(o->p_star);
#define CCP_PUSH(f)                                                   \
  do {                                                                \
    out->obj_hist[out->hist_len++] = (f);                             \
    if (track) out->gap_hist[out->gap_len++] = ((f) - o->p_star) / f0; \
  } while (0)
  for (int t = 0; t <= equil_iters; ++t) CCP_PUSH(f0);
  if (track && o->gap_tol > 0.0 && out->gap_hist[out->gap_len - 1] <= o->gap_tol)
    out->reached_tol = 1;
  double* y = (double*)calloc((size_t)(m ? m : 1), 8);
  double* kz = (double*)malloc((size_t)(m ? m : 1) * 8);
  double* z = (double*)calloc((size_t)(n ? n : 1), 8);
  double* zt = (double*)calloc((size_t)(n ? n : 1), 8);
  double* zn = (double*)malloc((size_t)(n ? n : 1) * 8);
  double* g = (double*)malloc((size_t)(n ? n : 1) * 8);
  double* x = (double*)malloc((size_t)(n ? n : 1) * 8);
  double* tn = (double*)malloc((size_t)(n ? n : 1) * 8);
  double* tm = (double*)malloc((size_t)(m ? m : 1) * 8);
  lsqr_op K = {A, d, e, tn, tm, 0, 0};
  for (int t = 1; t <= o->max_iters && !out->reached_tol; ++t) {
    /* dual: y = (y + sigma K z~ - sigma d b) / (1 + 0.5 sigma d d sqrt(lambda)) */
    B_apply(&K, zt, kz);
    for (int64_t i = 0; i < m; ++i) {
      const double di = d ? d[i] : 1.0;
      const double yh = y[i] + sigma * kz[i];
      y[i] = (yh - sigma * di * b[i]) / (1.0 + 0.5 * sigma * di * di * sl);
    }
    /* primal: weighted shrinkage, extrapolation */
    B_adjoint(&K, y, g);
    for (int64_t j = 0; j < n; ++j) {
      const double ej = e ? e[j] : 1.0;
      zn[j] = soft_threshold(z[j] - tau * g[j], tau * sl * ej);
    }
    for (int64_t j = 0; j < n; ++j) {
      zt[j] = zn[j] + o->theta * (zn[j] - z[j]);
      z[j] = zn[j];
    }
    out->iterations = t;
    for (int64_t j = 0; j < n; ++j) x[j] = (e ? e[j] : 1.0) * z[j];
    const double f = eo_lasso_objective(A, b, lambda, x);
    CCP_PUSH(f);
    if (track && o->gap_tol > 0.0 && out->gap_hist[out->gap_len - 1] <= o->gap_tol)
      out->reached_tol = 1;
  }
#undef CCP_PUSH
  for (int64_t j = 0; j < n; ++j) out->x[j] = (e ? e[j] : 1.0) * z[j];
  out->apply_count = applies0 + K.applies;
  out->adjoint_count = adjoints0 + K.adjoints;
  free(zero); free(y); free(kz); free(z); free(zt); free(zn); free(g); free(x);
  free(tn); free(tm);
  return 0;
}

int eo_ccp_lasso(const eo_matrix* A, const double* b, double lambda, const eo_ccp_options* o,
                 eo_ccp_run* out) {
  if (ccp_validate(A, b, lambda, o, "ccp_lasso")) return 1;
  return ccp_core(A, b, lambda, NULL, NULL, 0, 0, 0, o, out);
}

int eo_ccp_lasso_preconditioned(const eo_matrix* A, const double* b, double lambda,
                                const eo_params* p, const eo_ccp_options* o, eo_ccp_run* out) {
  if (ccp_validate(A, b, lambda, o, "ccp_lasso_preconditioned")) return 1;
  const int64_t m = A->m, n = A->n;
  double* u = (double*)malloc((size_t)(m ? m : 1) * 8);
  double* v = (double*)malloc((size_t)(n ? n : 1) * 8);
  double* d = (double*)malloc((size_t)(m ? m : 1) * 8);
  double* e = (double*)malloc((size_t)(n ? n : 1) * 8);
  eo_scaling s;
  memset(&s, 0, sizeof s);
  s.u = u;
  s.v = v;
  s.d = d;
  s.e = e;
  int rc = eo_sgd_equilibrate(A, p, 0, &s); /* :139 */
  if (!rc) rc = ccp_core(A, b, lambda, d, e, p->iterations, s.apply_count, s.adjoint_count, o,
                         out);
  free(u); free(v); free(d); free(e);
  return rc;
}

/* stochastic_gradient_estimate (src/equilibrate.cpp:60-71) */
int eo_stochastic_gradient_estimate(const eo_matrix* A, const double* u, const double* v,
                                    const eo_params* p, uint64_t seed, uint64_t stream,
                                    uint64_t offset, double* g_u, double* g_v) {
  if (eo_validate_params(p)) return 1;
  double alpha, beta;
  if (eo_resolve_targets(p, A->m, A->n, &alpha, &beta)) return 1;
  const int64_t m = A->m, n = A->n;
  double* d = (double*)malloc((size_t)(m ? m : 1) * 8);
  double* e = (double*)malloc((size_t)(n ? n : 1) * 8);
  double* xs = (double*)malloc((size_t)(n ? n : 1) * 8);
  double* xw = (double*)malloc((size_t)(m ? m : 1) * 8);
  for (int64_t i = 0; i < m; ++i) d[i] = eo_det_exp(u[i]);
  for (int64_t j = 0; j < n; ++j) e[j] = eo_det_exp(v[j]);
  eo_rng r;
  eo_rng_init(&r, seed, stream);
  for (uint64_t k = 0; k < offset; ++k) (void)eo_rng_next_u64(&r);
  for (int64_t j = 0; j < n; ++j) xs[j] = e[j] * eo_rng_sign(&r);
  mat_apply(A, xs, g_u);
  for (int64_t i = 0; i < m; ++i) {
    const double y = d[i] * g_u[i];
    g_u[i] = y * y;
  }
  for (int64_t i = 0; i < m; ++i) xw[i] = d[i] * eo_rng_sign(&r);
  mat_adjoint(A, xw, g_v);
  for (int64_t j = 0; j < n; ++j) {
    const double z = e[j] * g_v[j];
    g_v[j] = z * z;
  }
  const double nla = -alpha * alpha, nlb = -beta * beta;
  for (int64_t i = 0; i < m; ++i) g_u[i] = g_u[i] + (nla + p->gamma * u[i]);
  for (int64_t j = 0; j < n; ++j) g_v[j] = g_v[j] + (nlb + p->gamma * v[j]);
  free(d); free(e); free(xs); free(xw);
  return 0;
}
