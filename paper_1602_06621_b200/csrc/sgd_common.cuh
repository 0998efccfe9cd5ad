// sgd_common.cuh -- device helpers shared by the SGD traversals (kernels.cu:
// staged warp tiles / long rows, sell.cu: interleaved slices): streamed loads, the
// sequential row sum and the fused u/v epilogue.
#pragma once

#include "internal.h"

namespace eqb {

// read-only load that does not allocate in L1 (streamed CSR arrays).
// EQ_STREAM_EF: the stream is also marked evict-first in L2, so a column block
// of the gathered vector (EQUIL_BLOCK_MB) is not pushed out by it.
#ifndef EQ_STREAM_EF
#define EQ_STREAM_EF 1
#endif
#if EQ_STREAM_EF
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double ld_na(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
      : "=d"(v) : "l"(p), "l"(l2_evict_first()));
  return v;
}
__device__ __forceinline__ int32_t ld_na(const int32_t* p) {
  int32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
      : "=r"(v) : "l"(p), "l"(l2_evict_first()));
  return v;
}
#else
__device__ __forceinline__ double ld_na(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int32_t ld_na(const int32_t* p) {
  int32_t v;
  asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
#endif

// element `mat` of a two-element kernel-parameter array, selected without a
// dynamic index (which would copy the whole parameter struct to local memory,
// whose stores then compete with the gathers for L1TEX and L2)
template <class T>
__device__ __forceinline__ T pick(const T (&arr)[2], int mat) {
  return mat ? arr[1] : arr[0];
}

__device__ __forceinline__ bool sign_bit(const uint32_t* bits, int64_t b) {
  return (__ldg(bits + (b >> 5)) >> (b & 31)) & 1u;
}

// Sequential CSR-order sum of sp[b, e) onto acc (explicit_matrix.cpp:73-75).
// The adds form one dependent chain; the shared-memory loads feeding it are
// software-pipelined 8 products ahead (16-byte LDS) so the chain runs at add
// latency instead of load latency.
__device__ __forceinline__ double chain_sum(double acc, const double* sp, int b,
                                            int e) {
  int k = b;
  if ((k & 1) && k < e) acc = __dadd_rn(acc, sp[k++]);
  const double2* s2 = reinterpret_cast<const double2*>(sp);  // sp is 16B aligned
  int k2 = k >> 1;
  const int e2 = e >> 1;
  if (k2 + 4 <= e2) {
    double2 c0 = s2[k2], c1 = s2[k2 + 1], c2 = s2[k2 + 2], c3 = s2[k2 + 3];
    for (k2 += 4; k2 + 4 <= e2; k2 += 4) {
      const double2 n0 = s2[k2], n1 = s2[k2 + 1], n2 = s2[k2 + 2], n3 = s2[k2 + 3];
      acc = __dadd_rn(acc, c0.x); acc = __dadd_rn(acc, c0.y);
      acc = __dadd_rn(acc, c1.x); acc = __dadd_rn(acc, c1.y);
      acc = __dadd_rn(acc, c2.x); acc = __dadd_rn(acc, c2.y);
      acc = __dadd_rn(acc, c3.x); acc = __dadd_rn(acc, c3.y);
      c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    acc = __dadd_rn(acc, c0.x); acc = __dadd_rn(acc, c0.y);
    acc = __dadd_rn(acc, c1.x); acc = __dadd_rn(acc, c1.y);
    acc = __dadd_rn(acc, c2.x); acc = __dadd_rn(acc, c2.y);
    acc = __dadd_rn(acc, c3.x); acc = __dadd_rn(acc, c3.y);
  }
  for (; k2 < e2; ++k2) {
    const double2 c = s2[k2];
    acc = __dadd_rn(acc, c.x);
    acc = __dadd_rn(acc, c.y);
  }
  if ((e & 1) && e - 1 >= k) acc = __dadd_rn(acc, sp[e - 1]);
  return acc;
}

__device__ __forceinline__ void sgd_epilogue(const SgdIterArgs& a, int mat,
                                             int64_t r, double acc,
                                             unsigned& fl) {
  const int64_t pi = pick(a.slot, mat) ? static_cast<int64_t>(pick(a.slot, mat)[r]) : pick(a.poff, mat) + r;
  // |d_i w_i| = d_i exactly (w = +-1): this iteration's d (mat 0) or e (mat 1)
  const double scl = fabs(mat ? a.xs_cur[pi] : a.xw_cur[pi]);
  const double y = __dmul_rn(scl, acc);          // linop.cpp:19 / :25
  const double est = __dmul_rn(y, y);            // estimator.cpp:8
  double* const xp = pick(a.x, mat);
  double* const ap = pick(a.avg, mat);
  const double* const lp = pick(a.lin, mat);
  double avg = ap[r];
  const SgdBlockConst cb = pick(a.c, mat);
  const double xn = lp ? sgd_coord_lin(est, xp[r], lp[r], cb, a.st, avg, fl)
                       : sgd_coord(est, xp[r], cb, a.st, avg, fl);
  xp[r] = xn;
  ap[r] = avg;
  if (a.has_next) {  // next iteration's e.*s (from v) / d.*w (from u)
    const double dn = det_exp(xn);
    const bool pos = sign_bit(a.signs, pick(a.sign_next, mat) + r);
    double* dst = (mat ? a.xs_next : a.xw_next) + pi;
    const double val = pos ? dn : -dn;
    *dst = val;
    for (int g = 0; g < a.npeer; ++g) dst[a.peer_delta[g]] = val;  // peers' copies
  }
}
// epilogues of the generic passes (LSQR, variants, apply)
__device__ __forceinline__ void pass_epilogue(const PassArgs& a, int64_t r,
                                              double acc) {
  switch (a.mode) {
    case kPassPlain:
      a.out[r] = acc;
      break;
    case kPassLsqrU:
    case kPassLsqrV: {  // B.apply(v) - alpha*u  (lsqr.cpp:39, :49)
      const double bv = a.scale ? __dmul_rn(a.scale[r], acc) : acc;
      a.out[r] = __dsub_rn(bv, __dmul_rn(*a.coef, a.prev[r]));
      break;
    }
    case kPassResid:  // b - A x  (lsqr.cpp:97, :131)
      a.out[r] = __dsub_rn(a.prev[r], acc);
      break;
    case kPassScaled:
      a.out[r] = a.scale ? __dmul_rn(a.scale[r], acc) : acc;
      break;
    case kPassEst: {  // estimate_row_norms_sq: y = s_i * acc, y * y (estimator.cpp:5-9)
      const double y = __dmul_rn(a.scale[r], acc);
      a.out[r] = __dmul_rn(y, y);
      break;
    }
  }
}

__device__ __forceinline__ uint32_t ld_na(const uint32_t* p) {
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ uint16_t ld_na(const uint16_t* p) {
  unsigned short v;
  asm("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}

}  // namespace eqb
