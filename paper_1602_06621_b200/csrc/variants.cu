// variants.cu -- kernels of the engine variants sharing the SGD loop
// (src/variants.cpp): symmetric equilibration (:35-103) and block
// equilibration (:156-240).  The matrix passes themselves are the generic
// pass kernels (kPassEst epilogue); these kernels form the scalings and the
// gathered probes, sum row estimates over blocks and update the block iterates.
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

}  // namespace eqb
