// dense.cu -- K5: the dense GEMV pair in the canonical order (row-major A).
//
// The reference's dense apply/adjoint is Eigen GEMV on column-major storage
// (src/explicit_matrix.cpp:69,84); its summation order is Eigen-internal and
// not reproducible here, so the order is DEFINED by the canonical tree of
// det_math.cuh and restated in the oracle (eo_dense_apply / _adjoint):
//   y_i = canon_j (A_ij * x_j)       z_j = canon_i (A_ij * w_i)
// Both kernels keep the canonical fold in registers:
//   rows: one warp per row; lane l holds canonical lanes l + 32q (q < 8) of a
//         2048-column chunk, folds 256 -> 32 in registers and 32 -> 1 with
//         shuffles; chunk partials fold with shuffles (n <= 32 * 2048).
//   cols: CTA = (16 columns, 2048-row chunk), 512 threads; thread (g, j) holds
//         canonical lanes g + 32q (q < 8) -> 8 independent 8-term chains,
//         folds 256 -> 32 in registers and 32 -> 1 through shared memory.
#include "internal.h"

namespace eqb {

namespace {

__device__ __forceinline__ bool dsign_bit(const uint32_t* bits, int64_t b) {
  return (__ldg(bits + (b >> 5)) >> (b & 31)) & 1u;
}

constexpr unsigned kFull = 0xffffffffu;

// canonical dot of one row with x; result valid in lane 0
__device__ double dense_row_dot_warp(const double* __restrict__ Arow,
                                     const double* __restrict__ x, int64_t n, int lane) {
  const int nc = static_cast<int>((n + kChunk - 1) / kChunk);
  double mine = 0.0;  // chunk partial c is kept by lane c
  for (int c = 0; c < nc; ++c) {
    const int64_t base = static_cast<int64_t>(c) * kChunk;
    const int clen = static_cast<int>(n - base < kChunk ? n - base : kChunk);
    double s[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) s[q] = 0.0;
    if (clen == kChunk) {  // full chunk: unguarded loads, 16 in flight per lane
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        double av[16], xv[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int idx = lane + 32 * (u & 7) + 256 * (k + (u >> 3));
          av[u] = __ldg(Arow + base + idx);
          xv[u] = __ldg(x + base + idx);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) s[u & 7] = __dadd_rn(s[u & 7], __dmul_rn(av[u], xv[u]));
      }
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int idx = lane + 32 * q + 256 * k;  // canonical lane L = lane + 32q
          if (idx < clen)
            s[q] = __dadd_rn(s[q], __dmul_rn(__ldg(Arow + base + idx), __ldg(x + base + idx)));
        }
      }
    }
    // fold h = 128, 64, 32 in registers, then 16 .. 1 across lanes
#pragma unroll
    for (int q = 0; q < 4; ++q) s[q] = __dadd_rn(s[q], s[q + 4]);
    s[0] = __dadd_rn(s[0], s[2]);
    s[1] = __dadd_rn(s[1], s[3]);
    double v = __dadd_rn(s[0], s[1]);
#pragma unroll
    for (int h = 16; h >= 1; h >>= 1) v = __dadd_rn(v, __shfl_down_sync(kFull, v, h));
    const double p = __shfl_sync(kFull, v, 0);
    if (lane == c) mine = p;
  }
  if (nc == 1) return mine;  // lane 0
  // level 2: lanes >= nc hold +0.0, so the 1024-lane fold equals the fold over
  // the next power of two >= nc
  int p2 = 1;
  while (p2 < nc) p2 <<= 1;
  double v = mine;
  for (int h = p2 / 2; h >= 1; h >>= 1) v = __dadd_rn(v, __shfl_down_sync(kFull, v, h));
  return v;
}

constexpr int kRowsPerCta = 8;

__global__ void __launch_bounds__(256)
dense_sgd_rows_kernel(const DenseIterArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kRowsPerCta + (threadIdx.x >> 5);
  if (i >= a.m) return;
  const double acc = dense_row_dot_warp(a.A + i * a.n, a.xs_cur, a.n, lane);
  if (lane == 0) {  // u epilogue (src/equilibrate.cpp:113-128)
    unsigned fl = 0;
    const double d = fabs(a.xw_cur[i]);
    const double y = __dmul_rn(d, acc);
    const double est = __dmul_rn(y, y);
    double avg = a.ub[i];
    const double xn = a.lin_u ? sgd_coord_lin(est, a.u[i], a.lin_u[i], a.cu, a.st, avg, fl)
                              : sgd_coord(est, a.u[i], a.cu, a.st, avg, fl);
    a.u[i] = xn;
    a.ub[i] = avg;
    if (a.has_next) {
      const double dn = det_exp(xn);
      a.xw_next[i] = dsign_bit(a.signs, a.sign_next_w + i) ? dn : -dn;
    }
    if (fl) atomicOr(a.flags, fl);
  }
}

// level 2 over chunk partials for column j (nc <= 64, see create_dense)
__device__ double dense_col_level2(const double* colpart, int64_t nc, int64_t n, int64_t j) {
  if (nc == 1) return colpart[j];
  double s[64];
  int lanes = 1;
  while (lanes < nc) lanes <<= 1;
  for (int q = 0; q < lanes; ++q) s[q] = q < nc ? __dadd_rn(0.0, __ldcg(colpart + q * n + j)) : 0.0;
  for (int h = lanes / 2; h >= 1; h >>= 1)
    for (int q = 0; q < h; ++q) s[q] = __dadd_rn(s[q], s[q + h]);
  return s[0];
}

// partial column sums of one (16-column strip, 2048-row chunk): colpart[c*n + j].
// Thread (g, jj): column j0 + jj, canonical lanes L = g + 32q (q < 8), g < 32.
template <class Epi>
__global__ void __launch_bounds__(512, 2)
dense_cols_kernel(const double* __restrict__ A, int64_t m, int64_t n,
                  const double* __restrict__ w, double* __restrict__ colpart,
                  unsigned* __restrict__ colcnt, const Epi epi) {
  __shared__ double sc[32][16];
  const int jj = threadIdx.x & 15, g = threadIdx.x >> 4;  // g: 0..31
  const int64_t j = static_cast<int64_t>(blockIdx.x) * 16 + jj;
  const int64_t c = blockIdx.y;
  const int64_t base = c * kChunk;
  const int clen = static_cast<int>(m - base < kChunk ? m - base : kChunk);
  double s[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) s[q] = 0.0;
  if (j < n && clen == kChunk) {  // full chunk: unguarded, 16 loads in flight
    const double* Ac = A + (base + g) * n + j;
    const double* wc = w + base + g;
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      double av[16], wv[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int off = 32 * (u & 7) + 256 * (k + (u >> 3));
        av[u] = __ldg(Ac + static_cast<int64_t>(off) * n);
        wv[u] = __ldg(wc + off);
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) s[u & 7] = __dadd_rn(s[u & 7], __dmul_rn(av[u], wv[u]));
    }
  } else if (j < n) {
#pragma unroll 1
    for (int k = 0; k < 8; ++k) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int r = g + 32 * q + 256 * k;
        if (r < clen)
          s[q] = __dadd_rn(s[q], __dmul_rn(__ldg(A + (base + r) * n + j), __ldg(w + base + r)));
      }
    }
  }
  // h = 128, 64, 32 in registers (L + h = g + 32(q + h/32))
#pragma unroll
  for (int q = 0; q < 4; ++q) s[q] = __dadd_rn(s[q], s[q + 4]);
  s[0] = __dadd_rn(s[0], s[2]);
  s[1] = __dadd_rn(s[1], s[3]);
  sc[g][jj] = __dadd_rn(s[0], s[1]);
  __syncthreads();
  // h = 16 .. 1 across thread groups
  for (int h = 16; h >= 1; h >>= 1) {
    if (g < h) sc[g][jj] = __dadd_rn(sc[g][jj], sc[g + h][jj]);
    __syncthreads();
  }
  const int nc = static_cast<int>(gridDim.y);
  if (nc == 1) {  // one chunk: the partial is the column sum
    if (g == 0 && j < n) epi(j, sc[0][jj]);
    return;
  }
  if (g == 0 && j < n) colpart[c * n + j] = sc[0][jj];
  // the strip's last chunk CTA folds level 2 and runs the epilogue (one launch
  // instead of a partial kernel plus a final kernel)
  __shared__ unsigned ticket;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(colcnt + blockIdx.x, 1u);
  __syncthreads();
  if (ticket != static_cast<unsigned>(nc - 1)) return;
  __threadfence();
  if (g == 0 && j < n) epi(j, dense_col_level2(colpart, nc, n, j));
  if (threadIdx.x == 0) colcnt[blockIdx.x] = 0;  // ready for the next launch
}

// v epilogue of the dense SGD iteration (src/equilibrate.cpp:113-128) for column j
struct ColsSgdEpi {
  DenseIterArgs a;
  __device__ void operator()(int64_t j, double acc) const {
    unsigned fl = 0;
    const double e = fabs(a.xs_cur[j]);
    const double z = __dmul_rn(e, acc);
    const double est = __dmul_rn(z, z);
    double avg = a.vb[j];
    const double xn = a.lin_v ? sgd_coord_lin(est, a.v[j], a.lin_v[j], a.cv, a.st, avg, fl)
                              : sgd_coord(est, a.v[j], a.cv, a.st, avg, fl);
    a.v[j] = xn;
    a.vb[j] = avg;
    if (a.has_next) {
      const double dn = det_exp(xn);
      a.xs_next[j] = dsign_bit(a.signs, a.sign_next_s + j) ? dn : -dn;
    }
    if (fl) atomicOr(a.flags, fl);
  }
};

__device__ __forceinline__ void dense_pass_epi(const DensePassArgs& a, int64_t r, double acc) {
  switch (a.mode) {
    case kPassPlain: a.out[r] = acc; break;
    case kPassLsqrU:
    case kPassLsqrV: {  // B.apply(v) - alpha*u  (src/lsqr.cpp:39, :49)
      const double bv = a.scale ? __dmul_rn(a.scale[r], acc) : acc;
      a.out[r] = __dsub_rn(bv, __dmul_rn(*a.coef, a.prev[r]));
      break;
    }
    case kPassResid: a.out[r] = __dsub_rn(a.prev[r], acc); break;
    case kPassScaled: a.out[r] = a.scale ? __dmul_rn(a.scale[r], acc) : acc; break;
    case kPassEst: {  // estimate_row_norms_sq (src/estimator.cpp:5-9)
      const double y = __dmul_rn(a.scale[r], acc);
      a.out[r] = __dmul_rn(y, y);
      break;
    }
  }
}

__global__ void __launch_bounds__(256) dense_pass_rows_kernel(const DensePassArgs a) {
  if (a.skip && *a.skip) return;
  const int lane = threadIdx.x & 31;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kRowsPerCta + (threadIdx.x >> 5);
  if (i >= a.m) return;
  const double acc = dense_row_dot_warp(a.A + i * a.n, a.xg, a.n, lane);
  if (lane == 0) dense_pass_epi(a, i, acc);
}

struct ColsPassEpi {
  DensePassArgs a;
  __device__ void operator()(int64_t j, double acc) const {
    if (a.skip && *a.skip) return;  // the counters still run, so they reset
    dense_pass_epi(a, j, acc);
  }
};

template <class Epi>
cudaError_t dense_cols(const double* A, int64_t m, int64_t n, const double* w, double* colpart,
                       unsigned* colcnt, const Epi& epi, cudaStream_t s) {
  const dim3 grid(static_cast<unsigned>((n + 15) / 16),
                  static_cast<unsigned>((m + kChunk - 1) / kChunk));
  dense_cols_kernel<Epi><<<grid, 512, 0, s>>>(A, m, n, w, colpart, colcnt, epi);
  count_launch(s);
  return cudaGetLastError();
}

}  // namespace

// rows (u block) and columns (v block) read A independently: with a side
// stream s2 they run concurrently (fork on ev_fork, join on ev_join)
cudaError_t launch_dense_sgd_iter(const DenseIterArgs& a, cudaStream_t s, cudaStream_t s2,
                                  cudaEvent_t ev_fork, cudaEvent_t ev_join) {
  if (a.n > static_cast<int64_t>(kChunk) * 32) return cudaErrorInvalidValue;
  cudaError_t e = cudaSuccess;
  cudaStream_t rs = s;
  if (s2) {
    if ((e = cudaEventRecord(ev_fork, s)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(s2, ev_fork, 0)) != cudaSuccess) return e;
    rs = s2;
  }
  dense_sgd_rows_kernel<<<static_cast<unsigned>((a.m + kRowsPerCta - 1) / kRowsPerCta), 256, 0,
                          rs>>>(a);
  count_launch(rs);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  e = dense_cols(a.A, a.m, a.n, a.xw_cur, a.colpart, a.colcnt, ColsSgdEpi{a}, s);
  if (e != cudaSuccess) return e;
  if (s2) {
    if ((e = cudaEventRecord(ev_join, s2)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(s, ev_join, 0)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_dense_pass(const DensePassArgs& a, cudaStream_t s) {
  if (!a.adjoint) {
    if (a.n > static_cast<int64_t>(kChunk) * 32) return cudaErrorInvalidValue;
    dense_pass_rows_kernel<<<static_cast<unsigned>((a.m + kRowsPerCta - 1) / kRowsPerCta), 256,
                             0, s>>>(a);
    count_launch(s);
    return cudaGetLastError();
  }
  return dense_cols(a.A, a.m, a.n, a.xg, a.colpart, a.colcnt, ColsPassEpi{a}, s);
}

}  // namespace eqb
