// variants.cu -- kernels of the engine variants sharing the SGD loop
// (src/variants.cpp): symmetric equilibration (:35-103) and block
// equilibration (:156-240), and of the second consumer of D, E: the
// Chambolle-Pock lasso (src/ccp.cpp:27-110).  The matrix passes themselves are
// the generic pass kernels; these kernels form the scalings and the gathered
// probes, sum row estimates over blocks, update the block iterates, and run
// the CCP dual / primal steps.
#include "internal.h"
#include "sgd_common.cuh"

namespace eqb {
namespace {

__global__ void expand_scale_kernel(const double* __restrict__ x, const int32_t* __restrict__ map,
                                    int64_t len, const uint32_t* __restrict__ signs,
                                    int64_t sign0, double* __restrict__ scale,
                                    double* __restrict__ signed_out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= len) return;
  const double d = det_exp(x[map ? map[i] : i]);  // .array().exp() of the expanded iterate
  scale[i] = d;
  signed_out[i] = sign_bit(signs, sign0 + i) ? d : -d;  // d .* rademacher
}

// One warp per block: lanes fetch 32 member estimates at a time, lane 0 adds
// them in ascending member order onto a running sum that starts at 0.0
// (Vec::Zero then +=, variants.cpp:190-193).
__global__ void block_sum_kernel(const double* __restrict__ est,
                                 const int32_t* __restrict__ members,
                                 const int64_t* __restrict__ off, int64_t nblocks,
                                 double* __restrict__ out) {
  const int64_t b = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (b >= nblocks) return;
  double acc = 0.0;
  for (int64_t k0 = off[b]; k0 < off[b + 1]; k0 += 32) {
    const int64_t k = k0 + lane;
    const double v = k < off[b + 1] ? est[members[k]] : 0.0;
    const int cnt = static_cast<int>(off[b + 1] - k0 < 32 ? off[b + 1] - k0 : 32);
    for (int q = 0; q < cnt; ++q) {
      const double t = __shfl_sync(0xffffffffu, v, q);
      acc = __dadd_rn(acc, t);
    }
  }
  if (lane == 0) out[b] = acc;
}

__global__ void sgd_update_kernel(double* __restrict__ x, double* __restrict__ avg,
                                  const double* __restrict__ est,
                                  const double* __restrict__ lin, SgdBlockConst c,
                                  SgdStep st, int64_t len, unsigned* flags) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  unsigned fl = 0;
  if (i < len) {
    double a = avg[i];
    x[i] = sgd_coord_lin(est[i], x[i], lin[i], c, st, a, fl);  // run_projected_sgd :109-129
    avg[i] = a;
  }
  fl = __reduce_or_sync(0xffffffffu, fl);
  if (fl && (threadIdx.x & 31) == 0) atomicOr(flags, fl);
}

__global__ void gather_map_kernel(const double* __restrict__ x, const int32_t* __restrict__ map,
                                  int64_t len, double* __restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < len) out[i] = x[map[i]];
}

// dual step (src/ccp.cpp:73-78): y = (y + sigma*(K z~)_i - (sigma*d_i)*b_i) /
// (1 + ((0.5*sigma*d_i)*d_i)*sqrt(lambda)); dy = d .* y feeds K^T
__global__ void ccp_dual_kernel(double* __restrict__ y, const double* __restrict__ kz,
                                const double* __restrict__ d, const double* __restrict__ b,
                                double sigma, double sqrt_lambda, int64_t m,
                                double* __restrict__ dy) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= m) return;
  const double di = d ? d[i] : 1.0;
  const double yh = __dadd_rn(y[i], __dmul_rn(sigma, kz[i]));
  const double num = __dsub_rn(yh, __dmul_rn(__dmul_rn(sigma, di), b[i]));
  const double den =
      __dadd_rn(1.0, __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(0.5, sigma), di), di), sqrt_lambda));
  const double yn = __ddiv_rn(num, den);
  y[i] = yn;
  dy[i] = d ? __dmul_rn(di, yn) : yn;
}

__device__ __forceinline__ double soft_threshold(double q, double t) {  // src/ccp.cpp:19-23
  if (q > t) return __dsub_rn(q, t);
  if (q < -t) return __dadd_rn(q, t);
  return 0.0;
}

// primal step (:81-88): z' = soft(z - tau*g, (tau*sqrt(lambda))*e_j),
// z~ = z' + theta*(z' - z); ez~ = e .* z~ feeds K, x = e .* z', |x| for |x|_1
__global__ void ccp_primal_kernel(double* __restrict__ z, double* __restrict__ ezt,
                                  const double* __restrict__ g, const double* __restrict__ e,
                                  double tau, double tau_sl, double theta, int64_t n,
                                  double* __restrict__ x, double* __restrict__ absx) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= n) return;
  const double ej = e ? e[j] : 1.0;
  const double zo = z[j];
  const double zn = soft_threshold(__dsub_rn(zo, __dmul_rn(tau, g[j])), __dmul_rn(tau_sl, ej));
  const double zt = __dadd_rn(zn, __dmul_rn(theta, __dsub_rn(zn, zo)));
  z[j] = zn;
  ezt[j] = e ? __dmul_rn(ej, zt) : zt;
  const double xj = e ? __dmul_rn(ej, zn) : zn;
  x[j] = xj;
  absx[j] = fabs(xj);
}

// lasso objective from its two reductions (:121-122): r2 / sqrt(l) + sqrt(l) * l1
__global__ void lasso_value_kernel(const double* r2, const double* l1, double sqrt_lambda,
                                   double* out) {
  *out = __dadd_rn(__ddiv_rn(*r2, sqrt_lambda), __dmul_rn(sqrt_lambda, *l1));
}

__global__ void abs_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ out) {
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j < n) out[j] = fabs(x[j]);
}

// stochastic_gradient_estimate (src/equilibrate.cpp:69-70): g = est + (neg_lin + gamma * x)
__global__ void sge_finish_kernel(double* __restrict__ g, const double* __restrict__ x,
                                  double neg_lin, double gamma, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) g[i] = __dadd_rn(g[i], __dadd_rn(neg_lin, __dmul_rn(gamma, x[i])));
}

// gradient_weighted (src/equilibrate.cpp:35-36): g = g + (gamma * x - lin_i)
__global__ void grad_finish_kernel(double* __restrict__ g, const double* __restrict__ x,
                                   const double* __restrict__ lin, double lin_c, double gamma,
                                   int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n)
    g[i] = __dadd_rn(g[i], __dsub_rn(__dmul_rn(gamma, x[i]), lin ? lin[i] : lin_c));
}

unsigned grid(int64_t n, int t = 256) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

cudaError_t launch_expand_scale(const double* x, const int32_t* map, int64_t len,
                                const uint32_t* signs, int64_t sign0, double* scale,
                                double* signed_out, cudaStream_t s) {
  if (len == 0) return cudaSuccess;
  expand_scale_kernel<<<grid(len), 256, 0, s>>>(x, map, len, signs, sign0, scale, signed_out);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_block_sum(const double* est, const int32_t* members, const int64_t* off,
                             int64_t nblocks, double* out, cudaStream_t s) {
  if (nblocks == 0) return cudaSuccess;
  block_sum_kernel<<<grid(nblocks * 32), 256, 0, s>>>(est, members, off, nblocks, out);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_sgd_update(double* x, double* avg, const double* est, const double* lin,
                              const SgdBlockConst& c, const SgdStep& st, int64_t len,
                              unsigned* flags, cudaStream_t s) {
  if (len == 0) return cudaSuccess;
  sgd_update_kernel<<<grid(len), 256, 0, s>>>(x, avg, est, lin, c, st, len, flags);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_gather_map(const double* x, const int32_t* map, int64_t len, double* out,
                              cudaStream_t s) {
  if (len == 0) return cudaSuccess;
  gather_map_kernel<<<grid(len), 256, 0, s>>>(x, map, len, out);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_ccp_dual(double* y, const double* kz, const double* d, const double* b,
                            double sigma, double sqrt_lambda, int64_t m, double* dy,
                            cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  ccp_dual_kernel<<<grid(m), 256, 0, s>>>(y, kz, d, b, sigma, sqrt_lambda, m, dy);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_ccp_primal(double* z, double* ezt, const double* g, const double* e,
                              double tau, double tau_sl, double theta, int64_t n, double* x,
                              double* absx, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  ccp_primal_kernel<<<grid(n), 256, 0, s>>>(z, ezt, g, e, tau, tau_sl, theta, n, x, absx);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_lasso_value(const double* r2, const double* l1, double sqrt_lambda,
                               double* out, cudaStream_t s) {
  lasso_value_kernel<<<1, 1, 0, s>>>(r2, l1, sqrt_lambda, out);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_sge_finish(double* g, const double* x, double neg_lin, double gamma,
                              int64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  sge_finish_kernel<<<grid(n), 256, 0, s>>>(g, x, neg_lin, gamma, n);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_grad_finish(double* g, const double* x, const double* lin, double lin_c,
                               double gamma, int64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  grad_finish_kernel<<<grid(n), 256, 0, s>>>(g, x, lin, lin_c, gamma, n);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_abs(const double* x, int64_t n, double* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  abs_kernel<<<grid(n), 256, 0, s>>>(x, n, out);
  count_launch(s);
  return cudaGetLastError();
}

}  // namespace eqb
