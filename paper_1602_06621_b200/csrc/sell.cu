// sell.cu -- the SGD iteration over interleaved row slices (K3/K4, default).
//
// Layout (internal.h SellSlice): the rows of a slice (<= 32, length-sorted by
// plan_tiles) are stored interleaved, entry k of lane l at off + 32 k + l, so
// the warp that owns the slice reads entry k of all its rows with one 128-byte
// column load and one 256-byte value load.  Each lane owns one row: it forms
// the products val * x[slot] (one rounded multiply each) and extends its row's
// sum in CSR order with rounded adds, exactly explicit_matrix.cpp:73-75 for
// CSR(A) and, on CSR(A^T) whose rows hold ascending original rows,
// explicit_matrix.cpp:86-91.  There is no shared-memory staging, no barrier and
// no cross-lane step: the only limit is how many column / value loads and
// gathers each SM keeps in flight.
//
// Slices of both matrices are ordered longest first (a greedy
// longest-processing-time order: the 10^4-entry rows of a Zipf matrix start at
// once instead of trailing the launch).  Rows longer than kTileNnz go to the
// warp-specialised sell_long_kernel, the rest to sell_warp_kernel; the two run
// concurrently.  (On one GPU the SGD passes run A's long rows on the column
// sweep of sweep.cu instead, when the matrix allows it; sell_long_kernel then
// serves the generic passes.)  By default (SgdSplitOp) both only store each row's sum and
// sgd_update_rows_kernel then applies the SGD update (sgd_epilogue,
// sgd_common.cuh) to every row; SgdOp fuses the epilogue instead, SgdBlockOp
// carries sums between column-block rounds, PassOp<NV> runs the generic passes
// (LSQR, variants) with one or two gathered vectors.
#include <atomic>
#include <cstdlib>
#include <type_traits>

#include "sgd_common.cuh"

namespace eqb {
namespace {

// One warp per work item = (slice, block of 32 entries per row): the rows'
// entries are read row by row (coalesced along the row, columns mapped to
// slots), transposed through shared memory and written interleaved (coalesced
// along the lanes).  Lanes past a row's end write zero padding.
__global__ void __launch_bounds__(64)
build_sell_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                  const int32_t* __restrict__ map, const double* __restrict__ val,
                  const int64_t* __restrict__ kbp, const int32_t* __restrict__ midx, int nms,
                  const SellSlice* __restrict__ slices, const int32_t* __restrict__ row,
                  const int32_t* __restrict__ len, const int32_t* __restrict__ kst,
                  int32_t* __restrict__ oc, double* __restrict__ ov, int quad_min) {
  __shared__ int32_t tc[2][32][33];
  __shared__ double tv[2][32][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t item = blockIdx.x * 2LL + warp;
  if (item >= kbp[nms]) return;
  int lo = 0, hi = nms;  // last slice with kbp[j] <= item
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (kbp[mid] <= item) lo = mid; else hi = mid;
  }
  const int w = midx[lo];
  const int k0 = static_cast<int>(item - kbp[lo]) * 32;
  const SellSlice sd = slices[w];
  const int mylen = len[32 * w + lane];
  const int64_t mystart =
      lane < sd.cnt ? rp[row[32 * w + lane]] + (kst ? kst[32 * w + lane] : 0) : 0;
  // eight rows per batch: their loads (and then their slot lookups) are issued
  // together instead of one dependent round trip per row
  const int k = k0 + lane;
  for (int r0 = 0; r0 < sd.cnt; r0 += 8) {
    int32_t c[8];
    double v[8];
    bool ok[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t st = __shfl_sync(0xffffffffu, mystart, r0 + j);
      const int ln = __shfl_sync(0xffffffffu, mylen, r0 + j);
      ok[j] = r0 + j < sd.cnt && k < ln;
      if (ok[j]) {
        if (oc) c[j] = ci[st + k];
        if (ov) v[j] = val[st + k];
      }
    }
    if (map && oc) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (ok[j]) c[j] = map[c[j]];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (ok[j]) {
        if (oc) tc[warp][lane][r0 + j] = c[j];
        if (ov) tv[warp][lane][r0 + j] = v[j];
      }
  }
  __syncwarp();
  const bool quad = sd.maxlen >= quad_min;
  const int kend = min(32, static_cast<int>(quad ? sell_quad_len(sd.maxlen) : sd.maxlen) - k0);
  for (int kk = 0; kk < kend; ++kk) {
    const int k = k0 + kk;
    const int64_t dst = sd.off + (quad ? static_cast<int64_t>(k >> 2) * 128 + 4 * lane + (k & 3)
                                       : static_cast<int64_t>(k) * 32 + lane);
    const bool ok = lane < sd.cnt && k < mylen;
    if (oc) oc[dst] = ok ? tc[warp][kk][lane] : 0;
    if (ov) ov[dst] = ok ? tv[warp][kk][lane] : 0.0;
  }
}

// Column blocks (gathered vectors larger than L2): for every slice lane, the
// range of its row's entries in each block of `width` columns (columns
// ascend within a row) -- kst / bln[b * 32 nslices + q] -- and per block the
// slice's longest range, maxb[b * nslices + w].  Blocks past a matrix's count
// are empty.
__global__ void sell_block_lanes_kernel(const SellSlice* __restrict__ slices, int nslices,
                                        const int32_t* __restrict__ row,
                                        const int32_t* __restrict__ len,
                                        const int64_t* __restrict__ rpa,
                                        const int32_t* __restrict__ cia,
                                        const int64_t* __restrict__ rpt,
                                        const int32_t* __restrict__ cit, int nba, int nbt,
                                        int64_t wa, int64_t wt, int nbmax,
                                        int32_t* __restrict__ kst, int32_t* __restrict__ bln,
                                        int32_t* __restrict__ maxb) {
  const int64_t gt = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t w = gt >> 5;
  if (w >= nslices) return;
  const int lane = static_cast<int>(gt & 31);
  const int64_t q = 32 * w + lane;
  const int64_t nq = 32LL * nslices;
  const SellSlice sd = slices[w];
  const int mat = sd.mat;
  const int nb = mat ? nbt : nba;
  const int64_t width = mat ? wt : wa;
  const int L = lane < sd.cnt ? len[q] : 0;
  const int32_t* c = L > 0 ? (mat ? cit + rpt[row[q]] : cia + rpa[row[q]]) : nullptr;
  int k0 = 0;
  for (int b = 0; b < nbmax; ++b) {
    int k1 = k0;
    if (b < nb) {
      if (b == nb - 1) {
        k1 = L;
      } else {  // first entry with column >= (b + 1) * width
        const int64_t key = (b + 1) * width;
        int lo = k0, hi = L;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (c[mid] < key) lo = mid + 1; else hi = mid;
        }
        k1 = lo;
      }
    }
    kst[b * nq + q] = k0;
    bln[b * nq + q] = k1 - k0;
    const unsigned mx = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(k1 - k0));
    if (lane == 0) maxb[static_cast<int64_t>(b) * nslices + w] = static_cast<int32_t>(mx);
    k0 = k1;
  }
}

// the split epilogue: rows [0, m_loc) of A then [0, n_loc) of A^T, in order
__global__ void __launch_bounds__(256) sgd_update_rows_kernel(const SgdIterArgs a, int64_t m_loc,
                                                              int64_t n_loc) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  unsigned fl = 0;
  if (k < m_loc + n_loc) {
    const int mat = k >= m_loc ? 1 : 0;
    const int64_t r = mat ? k - m_loc : k;
    sgd_epilogue(a, mat, r, pick(a.carry, mat)[r], fl);
  }
  if (a.npeer) __threadfence_system();
  fl = __reduce_or_sync(0xffffffffu, fl);
  if (fl && (threadIdx.x & 31) == 0) atomicOr(a.flags, fl);
}

__global__ void sell_rows_kernel(const SellSlice* __restrict__ slices,
                                 const int32_t* __restrict__ r0, int nslices,
                                 const int32_t* __restrict__ rla, const int32_t* __restrict__ rlt,
                                 const int64_t* __restrict__ rpa, const int64_t* __restrict__ rpt,
                                 int32_t* __restrict__ row, int32_t* __restrict__ len) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q >= 32LL * nslices) return;
  const int64_t w = q >> 5;
  const int lane = static_cast<int>(q & 31);
  const SellSlice sd = slices[w];
  int32_t r = 0, l = 0;
  if (lane < sd.cnt) {
    r = (sd.mat ? rlt : rla)[r0[w] + lane];
    const int64_t* rp = sd.mat ? rpt : rpa;
    l = static_cast<int32_t>(rp[r + 1] - rp[r]);
  }
  row[q] = r;
  len[q] = l;
}

// streamed interleaved entries (read once per iteration)
#ifndef EQ_STREAM_HINT
#define EQ_STREAM_HINT 0  // 1: L2::128B, 2: L2::256B prefetch-size hint on the stream loads
#endif
__device__ __forceinline__ double ld_st(const double* p) {
#if EQ_STREAM_HINT == 1
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::128B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
#elif EQ_STREAM_HINT == 2
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::256B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
#else
  return ld_na(p);
#endif
}
__device__ __forceinline__ int32_t ld_st(const int32_t* p) {
#if EQ_STREAM_HINT == 1
  int32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::128B.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
#elif EQ_STREAM_HINT == 2
  int32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::256B.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
#else
  return ld_na(p);
#endif
}

// 128-bit / 64-bit streamed loads of the quad layout (same qualifiers as ld_na:
// no L1 allocation, L2 evict-first)
__device__ __forceinline__ int4 ld_st4(const int32_t* p) {
  int4 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(l2_evict_first()));
  return v;
}
__device__ __forceinline__ int2 ld_st2(const int32_t* p) {
  int2 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;"
      : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(l2_evict_first()));
  return v;
}
// 256-bit load (sm_100: LDG.E.NA.ENL2.256): a lane's whole quad of values in one
// access, so a warp's value load is 1 KB contiguous (two 128-bit loads would
// each touch every sector half-used, and without L1 allocation fetch it twice)
__device__ __forceinline__ void ld_st4(const double* p, double* v) {
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p), "l"(l2_evict_first()));
}
__device__ __forceinline__ double2 ld_st2(const double* p) {
  double2 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
      : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(l2_evict_first()));
  return v;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

// What a traversal does with its row sums.  NV gathered vectors per entry (2:
// LSQR's fused residual + next B v pass, one value / column stream, two
// sequential sums per row).
struct SgdOp {  // the fused u / v update of one SGD iteration
  static constexpr int NV = 1;
  static constexpr bool PAIR = false;
  SgdIterArgs a;
  __device__ bool skip() const { return false; }
  __device__ const double* x(int mat) const { return mat ? a.xw_cur : a.xs_cur; }
  __device__ const double* x2(int) const { return nullptr; }
  __device__ double start(int, int64_t) const { return 0.0; }
  __device__ void finish(int mat, int32_t r, double acc, double, unsigned& fl, int64_t) const {
    sgd_epilogue(a, mat, r, acc, fl);
  }
  __device__ void end(unsigned fl) const {
    // peer stores performed system-wide before the kernel completes (the
    // barrier that follows orders every peer's next reads after them)
    if (a.npeer) __threadfence_system();
    if (fl) atomicOr(a.flags, fl);
  }
};
// split epilogue: the traversal only stores each row's sum (carry[mat][row]);
// sgd_update_rows_kernel applies the update afterwards with full occupancy, so
// the epilogue's dependent loads no longer hold the traversal's warps
struct SgdSplitOp : SgdOp {
  __device__ void finish(int mat, int32_t r, double acc, double, unsigned&, int64_t) const {
    pick(a.carry, mat)[r] = acc;
  }
  __device__ void end(unsigned) const {}
};
// column-block rounds: the running sum of lane q waits in carry[0][q]
struct SgdBlockOp : SgdOp {
  __device__ double start(int mat, int64_t q) const {
    return a.round > 0 && a.round < pick(a.nblk, mat) ? a.carry[0][q] : 0.0;
  }
  __device__ void finish(int mat, int32_t r, double acc, double, unsigned& fl, int64_t q) const {
    if (a.round < pick(a.nblk, mat) - 1) {
      a.carry[0][q] = acc;
      return;
    }
    sgd_epilogue(a, mat, r, acc, fl);
  }
};
template <int NV_>
struct PassOp {  // generic passes (pass_epilogue); one matrix per launch
  static constexpr int NV = NV_;
  static constexpr bool PAIR = false;
  PassArgs p, q;
  __device__ bool skip() const { return p.skip && *p.skip; }
  __device__ const double* x(int) const { return p.xg; }
  __device__ const double* x2(int) const { return q.xg; }
  __device__ double start(int, int64_t) const { return 0.0; }
  __device__ void finish(int, int32_t r, double acc, double acc2, unsigned&, int64_t) const {
    pass_epilogue(p, r, acc);
    if constexpr (NV == 2) pass_epilogue(q, r, acc2);
  }
  __device__ void end(unsigned) const {}
};
// LSQR's fused residual + next B v pass with its two gathered vectors stored
// interleaved (p.xg[2 c] = (e.x)_c, p.xg[2 c + 1] = (e.v)_c): one 16-byte
// gather (one L2 sector) per entry instead of two 8-byte gathers from two arrays
struct PassPairOp : PassOp<2> {
  static constexpr bool PAIR = true;
};

// the gathered value(s) of slot c: one vector, two vectors, or one interleaved pair
template <class Op>
__device__ __forceinline__ void gather_x(const double* __restrict__ x, const double* __restrict__ x2,
                                         int32_t c, double& g, double& g2) {
  if constexpr (Op::PAIR) {
    const double2 p = __ldg(reinterpret_cast<const double2*>(x) + c);
    g = p.x;
    g2 = p.y;
  } else {
    g = __ldg(x + c);
    if constexpr (Op::NV == 2) g2 = __ldg(x2 + c);
  }
}

__device__ __forceinline__ int slice_at(const SellArgs& sa, int i) {
  return sa.order ? __ldg(sa.order + i) : i;
}

// The traversal of one warp slice, for its layout: Q = 1 (entry k of lane l
// at 32 k + l: one 32-bit column and one 64-bit value load per entry) or
// Q = kQuad (the lane's entries 4 at a time: one 128-bit column load and two
// 128-bit value loads per quad).
template <class Op, int B, bool PIPE, int Q>
__device__ __forceinline__ void warp_slice(const Op& op, const SellArgs& sa, const SellSlice& sd,
                                           int mat, int q, int len, int lane) {
  static_assert(Q == 1 || B % kQuad == 0, "quad batches: whole quads");
  constexpr int NV = Op::NV;
  const int32_t* __restrict__ cp = pick(sa.ci, mat) + sd.off + (Q == 1 ? lane : 4 * lane);
  const double* __restrict__ vp = pick(sa.va, mat) + sd.off + (Q == 1 ? lane : 4 * lane);
  const double* __restrict__ x = op.x(mat);
  const double* __restrict__ x2 = op.x2(mat);
  double acc = op.start(mat, q), acc2 = 0.0;
  // entries k .. k + B - 1 of the lane's row (full: all within the row)
  auto load = [&](int k, int32_t* c, double* v, bool full) {
    if constexpr (Q == 1) {
#pragma unroll
      for (int b = 0; b < B; ++b)
        if (full || k + b < len) c[b] = ld_st(cp + 32 * (k + b));
#pragma unroll
      for (int b = 0; b < B; ++b)
        if (full || k + b < len) v[b] = ld_st(vp + 32 * (k + b));
    } else {
#pragma unroll
      for (int t = 0; t < B / kQuad; ++t) {
        const int kk = k + kQuad * t;  // a multiple of 4: whole quads
        if (full || kk < len) {
          const int64_t o = static_cast<int64_t>(kk >> 2) * 128;
          const int4 c4 = ld_st4(cp + o);
          c[4 * t] = c4.x, c[4 * t + 1] = c4.y, c[4 * t + 2] = c4.z, c[4 * t + 3] = c4.w;
          ld_st4(vp + o, v + 4 * t);
        }
      }
    }
  };
  auto consume = [&](const int32_t* c, const double* v, int k0, bool full) {
    double g[B], g2[B];
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (full || k0 + b < len) {
        EQ_CHECK(c[b] >= 0 && c[b] < pick(sa.xlen, mat));
        gather_x<Op>(x, x2, c[b], g[b], g2[b]);
      }
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (full || k0 + b < len) {
        acc = __dadd_rn(acc, __dmul_rn(v[b], g[b]));
        if constexpr (NV == 2) acc2 = __dadd_rn(acc2, __dmul_rn(v[b], g2[b]));
      }
  };
  int k = 0;
  if constexpr (!PIPE) {
    for (; k + B <= len; k += B) {
      int32_t c[B];
      double v[B];
      load(k, c, v, true);
      consume(c, v, k, true);
    }
  } else {
    if (k + B <= len) {
      int32_t c[B];
      double v[B];
      load(0, c, v, true);
      for (;;) {
        const int kn = k + B;
        const bool more = kn + B <= len;
        int32_t cn[B];
        double vn[B];
        if (more) load(kn, cn, vn, true);
        consume(c, v, k, true);
        k = kn;
        if (!more) break;
#pragma unroll
        for (int b = 0; b < B; ++b) {
          c[b] = cn[b];
          v[b] = vn[b];
        }
      }
    }
  }
  if (k < len) {  // tail: fewer than B entries left
    int32_t c[B];
    double v[B];
    load(k, c, v, false);
    consume(c, v, k, false);
  }
  unsigned fl = 0;
  if (lane < sd.cnt) op.finish(mat, __ldg(sa.row + q), acc, acc2, fl, q);
  op.end(fl);
}

// One warp per slice (rows <= kTileNnz).  B entries per lane per batch: B
// column loads and B value loads, then the gathers, then the dependent adds.
// PIPE: the next batch's column / value loads are issued before this batch's
// gathers (one batch of CSR stream in flight behind the gathers).  Slices with
// maxlen >= sa.quad_min are in the quad layout (uniform branch per warp).
template <class Op, int B, bool PIPE, int MINB>
__global__ void __launch_bounds__(128, MINB) sell_warp_kernel(const Op op, const SellArgs sa) {
  if (op.skip()) return;
  const int lane = threadIdx.x & 31;
  const int i = sa.first + blockIdx.x * 4 + (threadIdx.x >> 5);
  if (i >= sa.nslices) return;
  const int w = slice_at(sa, i);
  const SellSlice sd = sa.slices[w];
  const int mat = sd.mat;
  const int q = 32 * w + lane;
  const int len = __ldg(sa.len + q);
  if (sd.maxlen >= sa.quad_min) warp_slice<Op, B, PIPE, kQuad>(op, sa, sd, mat, q, len, lane);
  else warp_slice<Op, B, PIPE, 1>(op, sa, sd, mat, q, len, lane);
}

// Long slices (rows longer than kTileNnz): one CTA per slice, warp-specialised.
// A lane-per-row chain that waits on its own loads would make the slice's
// longest row (10^4 entries on c3) the critical path of the whole launch, so
// S stager warps run ahead: stager s takes rounds s, s + S, ... (B entries of
// every row per round: coalesced interleaved loads, gathers, rounded products)
// into a ring of S + 1 shared-memory stages, and warp 0's lanes extend their
// rows' sequential sums from the ring (conflict-free: lane l reads column l).
// Stages hand over on mbarriers (full: 32 stager lanes arrive; empty: 32 chain
// lanes arrive).  PIPE: a stager issues its next round's loads before this
// round's gathers.  Products are formed in any order; the adds are the
// reference's CSR-order chain.
template <class Op, int B, int S, bool PIPE, int MINB, int Q>
__global__ void __launch_bounds__(32 * (S + 1), MINB)
sell_long_kernel(const Op op, const SellArgs sa) {
  static_assert(Q == 1 || (Q == kQuad && (B == 2 || B == 4)), "quad rounds: 2 or 4 entries");
  constexpr int NV = Op::NV;
  constexpr int R = S + 1;
  __shared__ __align__(16) double buf[NV][R][B * 32];
  __shared__ __align__(8) unsigned long long full[R], empty[R];
#ifdef EQ_CHECKED
  __shared__ int tag[R];  // round whose products a stage holds (ring protocol check)
#endif
  if (op.skip()) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = sa.first + blockIdx.x;
  if (threadIdx.x < R) {
    mbar_init(&full[threadIdx.x], 32);
    mbar_init(&empty[threadIdx.x], 32);
  }
  __syncthreads();
  if (i >= sa.nslices) return;
  const int w = slice_at(sa, i);
  const SellSlice sd = sa.slices[w];
  const int mat = sd.mat;
  const int q = 32 * w + lane;
  const int len = __ldg(sa.len + q);
  const int rounds = (sd.maxlen + B - 1) / B;
  if (warp > 0) {
    const int32_t* __restrict__ cp = pick(sa.ci, mat) + sd.off + lane;
    const double* __restrict__ vp = pick(sa.va, mat) + sd.off + lane;
    const double* __restrict__ x = op.x(mat);
    const double* __restrict__ x2 = op.x2(mat);
    int r = warp - 1;
    int32_t c[B];
    double v[B];
    auto load = [&](int rr, int32_t* cc, double* vv) {
      const int k0 = rr * B;
      if constexpr (Q == kQuad) {  // the lane's B entries are adjacent: vector loads
        if (k0 < len) {
          const int64_t o = static_cast<int64_t>(k0 >> 2) * 128 + 3 * lane + (k0 & 3);
          if constexpr (B == 4) {
            const int4 c4 = ld_st4(cp + o);
            cc[0] = c4.x, cc[1] = c4.y, cc[2] = c4.z, cc[3] = c4.w;
            ld_st4(vp + o, vv);
          } else {
            const int2 c2 = ld_st2(cp + o);
            cc[0] = c2.x, cc[1] = c2.y;
            const double2 v0 = ld_st2(vp + o);
            vv[0] = v0.x, vv[1] = v0.y;
          }
        }
      } else {
#pragma unroll
        for (int b = 0; b < B; ++b)
          if (k0 + b < len) cc[b] = ld_st(cp + 32 * (k0 + b));
#pragma unroll
        for (int b = 0; b < B; ++b)
          if (k0 + b < len) vv[b] = ld_st(vp + 32 * (k0 + b));
      }
    };
    if (PIPE && r < rounds) load(r, c, v);
    for (; r < rounds; r += S) {
      const int k0 = r * B;
      int32_t cn[B];
      double vn[B];
      if constexpr (PIPE) {
        if (r + S < rounds) load(r + S, cn, vn);
      } else {
        load(r, c, v);
      }
      double g[B], g2[B];
#pragma unroll
      for (int b = 0; b < B; ++b)
        if (k0 + b < len) {
          EQ_CHECK(c[b] >= 0 && c[b] < pick(sa.xlen, mat));
          gather_x<Op>(x, x2, c[b], g[b], g2[b]);
        }
      const int bi = r % R;
      if (r >= R) mbar_wait(&empty[bi], ((r / R) - 1) & 1);
#ifdef EQ_CHECKED
      if (lane == 0) tag[bi] = r;
#endif
#pragma unroll
      for (int b = 0; b < B; ++b)
        if (k0 + b < len) {
          buf[0][bi][32 * b + lane] = __dmul_rn(v[b], g[b]);
          if constexpr (NV == 2) buf[NV - 1][bi][32 * b + lane] = __dmul_rn(v[b], g2[b]);
        }
      mbar_arrive(&full[bi]);
      if constexpr (PIPE) {
#pragma unroll
        for (int b = 0; b < B; ++b) {
          c[b] = cn[b];
          v[b] = vn[b];
        }
      }
    }
    return;
  }
  double acc = op.start(mat, q), acc2 = 0.0;
  for (int r = 0; r < rounds; ++r) {
    const int bi = r % R;
    mbar_wait(&full[bi], (r / R) & 1);
#ifdef EQ_CHECKED
    EQ_CHECK(tag[bi] == r);  // the stage holds this round's products
#endif
    const int k0 = r * B;
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (k0 + b < len) {
        acc = __dadd_rn(acc, buf[0][bi][32 * b + lane]);
        if constexpr (NV == 2) acc2 = __dadd_rn(acc2, buf[NV - 1][bi][32 * b + lane]);
      }
    mbar_arrive(&empty[bi]);
  }
  unsigned fl = 0;
  if (lane < sd.cnt) op.finish(mat, __ldg(sa.row + q), acc, acc2, fl, q);
  op.end(fl);
}

// Preferred shared-memory carveout (percent of the maximum), once per kernel
// instantiation.  The SGD long slices need 16.6 KB per CTA: 22% (~50 KB, three
// CTAs) leaves the rest of each SM's 256 KB to L1, where xw's hot slots live
// (c3: 1.158 -> 1.117-1.128 ms; 8% starves the long kernel, 30-50% shrinks L1).
// EQUIL_CARVE_LONG / EQUIL_CARVE_WARP override (-1: the driver's choice).
template <class K>
void carveout(K kernel, const char* env, int dflt) {
  // once per (instantiation, device): the attribute is per device context
  static std::atomic<unsigned long long> done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  const unsigned long long bit = 1ULL << (dev & 63);
  if (done.fetch_or(bit) & bit) return;
  int pct = dflt;
  if (const char* e = getenv(env)) pct = atoi(e);
  if (pct >= 0) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaGetLastError();
  }
}
template <class Op>
constexpr bool is_sgd() { return std::is_same<Op, SgdOp>::value || std::is_same<Op, SgdSplitOp>::value; }
// (LSQR passes too: 1.815 -> 1.803 ms).  The dual LSQR pass with 4-entry rounds
// (quad layout) keeps 2 CTAs per SM only with 36% (its ring is 32 KB): c4
// 1.331 -> 1.277 ms per LSQR iteration.
template <class Op, int B>
constexpr int carve_long() { return Op::NV == 2 && B == 4 ? 36 : 22; }
template <class Op>
constexpr int carve_warp() { return is_sgd<Op>() ? 0 : -1; }

template <class Op, int B, int S, bool PIPE, int MINB, int Q>
void launch_long_q(const Op& op, const SellArgs& sa, cudaStream_t s) {
  carveout(sell_long_kernel<Op, B, S, PIPE, MINB, Q>, "EQUIL_CARVE_LONG", carve_long<Op, B>());
  sell_long_kernel<Op, B, S, PIPE, MINB, Q>
      <<<static_cast<unsigned>(sa.nslices - sa.first), 32 * (S + 1), 0, s>>>(op, sa);
}
// the slices' layout picks the instantiation (quad: 128-bit stream loads)
template <class Op, int B, int S, bool PIPE, int MINB>
void launch_long(const Op& op, const SellArgs& sa, cudaStream_t s) {
  if (sa.quad_min <= kTileNnz + 1) launch_long_q<Op, B, S, PIPE, MINB, kQuad>(op, sa, s);
  else launch_long_q<Op, B, S, PIPE, MINB, 1>(op, sa, s);
}

template <class Op, int B, bool PIPE, int MINB>
void launch_warp(const Op& op, const SellArgs& sa, cudaStream_t s) {
  const unsigned g = static_cast<unsigned>((sa.nslices - sa.first + 3) / 4);
  carveout(sell_warp_kernel<Op, B, PIPE, MINB>, "EQUIL_CARVE_WARP", carve_warp<Op>());
  sell_warp_kernel<Op, B, PIPE, MINB><<<g, 128, 0, s>>>(op, sa);
}

}  // namespace

cudaError_t build_sell(const int64_t* rp, const int32_t* ci, const int32_t* map, const double* val,
                       const int64_t* kbp, int64_t items, const int32_t* midx, int nmat_slices,
                       const SellSlice* slices, const int32_t* row, const int32_t* len,
                       const int32_t* kst, int32_t* out_ci, double* out_va, cudaStream_t s,
                       int quad_min) {
  if (nmat_slices == 0 || items == 0) return cudaSuccess;
  build_sell_kernel<<<static_cast<unsigned>((items + 1) / 2), 64, 0, s>>>(
      rp, ci, map, val, kbp, midx, nmat_slices, slices, row, len, kst, out_ci, out_va, quad_min);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_sell_rows(const SellSlice* slices, const int32_t* r0, int nslices,
                             const int32_t* rowlist_a, const int32_t* rowlist_t,
                             const int64_t* rp_a, const int64_t* rp_t, int32_t* row,
                             int32_t* len, cudaStream_t s) {
  if (nslices == 0) return cudaSuccess;
  const int64_t n = 32LL * nslices;
  sell_rows_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
      slices, r0, nslices, rowlist_a, rowlist_t, rp_a, rp_t, row, len);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_sell_block_lanes(const SellSlice* slices, int nslices, const int32_t* row,
                                    const int32_t* len, const int64_t* rpa, const int32_t* cia,
                                    const int64_t* rpt, const int32_t* cit, int nba, int nbt,
                                    int64_t wa, int64_t wt, int nbmax, int32_t* kst, int32_t* bln,
                                    int32_t* maxb, cudaStream_t s) {
  if (nslices == 0) return cudaSuccess;
  const int64_t n = 32LL * nslices;
  sell_block_lanes_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
      slices, nslices, row, len, rpa, cia, rpt, cit, nba, nbt, wa, wt, nbmax, kst, bln, maxb);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_sgd_sell_long(const SgdIterArgs& a, const SellArgs& sa, int variant,
                                 cudaStream_t s) {
  if (sa.nslices <= sa.first) return cudaSuccess;
  if (a.nblk[0] > 1 || a.nblk[1] > 1) {
    launch_long_q<SgdBlockOp, 4, 15, true, 1, 1>(SgdBlockOp{{a}}, sa, s);
    count_launch(s);
    return cudaGetLastError();
  }
  const SgdOp op{a};
  switch (variant) {  // EQUIL_SELL_LVARIANT (A/B knob); 0 = measured best on c3
    case 2: launch_long<SgdOp, 4, 7, true, 3>(op, sa, s); break;
    case 3: launch_long<SgdOp, 2, 15, true, 2>(op, sa, s); break;
    default: launch_long<SgdOp, 4, 15, true, 1>(op, sa, s); break;
  }
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_sgd_update_rows(const SgdIterArgs& a, int64_t m_loc, int64_t n_loc,
                                   cudaStream_t s) {
  const int64_t n = m_loc + n_loc;
  if (n == 0) return cudaSuccess;
  sgd_update_rows_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(a, m_loc, n_loc);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_sgd_sell_split(const SgdIterArgs& a, const SellArgs& sa, bool lng,
                                  int variant, cudaStream_t s) {
  if (sa.nslices <= sa.first) return cudaSuccess;
  const SgdSplitOp op{{a}};
  if (lng) {
    switch (variant) {  // EQUIL_SELL_LVARIANT
      case 1: launch_long<SgdSplitOp, 4, 15, true, 2>(op, sa, s); break;
      case 2: launch_long<SgdSplitOp, 2, 15, true, 2>(op, sa, s); break;
      case 3: launch_long<SgdSplitOp, 4, 7, true, 4>(op, sa, s); break;
      default: launch_long<SgdSplitOp, 4, 15, true, 1>(op, sa, s); break;
    }
  } else {
    switch (variant) {  // EQUIL_SELL_VARIANT: <batch, pipelined, CTAs per SM> (DESIGN §3 has the sweep)
      case 1: launch_warp<SgdSplitOp, 8, true, 8>(op, sa, s); break;
      case 2: launch_warp<SgdSplitOp, 4, true, 10>(op, sa, s); break;
      case 3: launch_warp<SgdSplitOp, 8, true, 6>(op, sa, s); break;
      // quad layout (256-bit value loads): 56 registers, 9 CTAs per SM (c3:
      // 0.997-1.010 vs 1.067-1.083 ms at <8, true, 6>)
      default: launch_warp<SgdSplitOp, 8, true, 9>(op, sa, s); break;
    }
  }
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_sgd_sell(const SgdIterArgs& a, const SellArgs& sa, int variant,
                            cudaStream_t s) {
  if (sa.nslices <= sa.first) return cudaSuccess;
  if (a.nblk[0] > 1 || a.nblk[1] > 1) {
    launch_warp<SgdBlockOp, 8, true, 6>(SgdBlockOp{{a}}, sa, s);
    count_launch(s);
    return cudaGetLastError();
  }
  const SgdOp op{a};
  switch (variant) {  // EQUIL_SELL_VARIANT (A/B knob); 0 = measured best on c3
    case 1: launch_warp<SgdOp, 4, false, 12>(op, sa, s); break;
    case 2: launch_warp<SgdOp, 8, false, 8>(op, sa, s); break;
    case 3: launch_warp<SgdOp, 16, false, 6>(op, sa, s); break;
    case 4: launch_warp<SgdOp, 8, true, 8>(op, sa, s); break;
    default: launch_warp<SgdOp, 8, true, 6>(op, sa, s); break;
  }
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_sell_pass(const PassArgs& a, const PassArgs* b, const SellArgs& sa, bool lng,
                             bool pair, cudaStream_t s) {
  if (sa.nslices <= sa.first) return cudaSuccess;
  static const int pv = getenv("EQUIL_PASS_VARIANT") ? atoi(getenv("EQUIL_PASS_VARIANT")) : 0;
  if (b && pair) {
    PassPairOp op;
    op.p = a;
    op.q = *b;
    if (lng) {
      switch (pv) {  // EQUIL_PASS_VARIANT
        case 1: launch_long<PassPairOp, 4, 15, true, 1>(op, sa, s); break;
        case 2: launch_long<PassPairOp, 4, 7, true, 2>(op, sa, s); break;
        default:  // quad layout: a round is one whole quad (B = 4), else B = 2
          if (sa.quad_min <= kTileNnz + 1) launch_long<PassPairOp, 4, 15, true, 1>(op, sa, s);
          else launch_long<PassPairOp, 2, 15, true, 1>(op, sa, s);
          break;
      }
    } else {
      switch (pv) {
        case 4: launch_warp<PassPairOp, 8, true, 6>(op, sa, s); break;
        case 5: launch_warp<PassPairOp, 4, true, 10>(op, sa, s); break;
        case 6: launch_warp<PassPairOp, 4, true, 6>(op, sa, s); break;
        case 7: launch_warp<PassPairOp, 8, true, 8>(op, sa, s); break;
        // 8 CTAs per SM on the quad layout (c4: 1.208-1.211 vs 1.227-1.228 ms at 6)
        default: launch_warp<PassPairOp, 4, true, 8>(op, sa, s); break;
      }
    }
  } else if (b) {
    const PassOp<2> op{a, *b};
    if (lng) {
      switch (pv) {  // EQUIL_PASS_VARIANT; 0 = measured best on c4 (1.82 vs 1.86 ms)
        case 1: launch_long<PassOp<2>, 4, 15, true, 1>(op, sa, s); break;
        case 2: launch_long<PassOp<2>, 4, 7, true, 2>(op, sa, s); break;
        default:
          if (sa.quad_min <= kTileNnz + 1) launch_long<PassOp<2>, 4, 15, true, 1>(op, sa, s);
          else launch_long<PassOp<2>, 2, 15, true, 1>(op, sa, s);
          break;
      }
    } else {
      switch (pv) {
        case 4: launch_warp<PassOp<2>, 8, true, 6>(op, sa, s); break;
        default: launch_warp<PassOp<2>, 4, true, 6>(op, sa, s); break;
      }
    }
  } else {
    const PassOp<1> op{a, a};
    if (lng) {
      launch_long<PassOp<1>, 4, 15, true, 1>(op, sa, s);
    } else {
      switch (pv) {
        case 5: launch_warp<PassOp<1>, 8, true, 9>(op, sa, s); break;
        case 6: launch_warp<PassOp<1>, 8, true, 6>(op, sa, s); break;
        case 7: launch_warp<PassOp<1>, 4, true, 10>(op, sa, s); break;
        default: launch_warp<PassOp<1>, 8, true, 8>(op, sa, s); break;
      }
    }
  }
  count_launch(s);
  return cudaGetLastError();
}

}  // namespace eqb
