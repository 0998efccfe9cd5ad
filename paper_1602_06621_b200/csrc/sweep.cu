// sweep.cu -- column-synchronous sweep of A's long rows (one SGD pass of the
// rows longer than kTileNnz; explicit_matrix.cpp:73-75 order).
//
// Why: every entry of a long row gathers x[col] from an 8 MB vector, a cold
// 32-byte sector each -- one L1 miss request per entry, and an SM's L1 sends
// about one request per clock ("SM <-> L2 port model").  Here the
// long rows are dealt to one persistent CTA per SM (~360 rows on c3) and every
// CTA sweeps the gathered vector in panels of W columns: panel p (W doubles)
// and the CTA's entries with columns in it arrive in shared memory by bulk
// asynchronous copies (whole lines, no LSU requests), and each row's run of
// entries in the panel extends the row's sequential sum from shared memory.
// Columns ascend within a row, so runs in ascending panel order are exactly
// the row's CSR order: the sum is the reference's, bit for bit.
//
// Layout (built once per matrix by the kernels below): for CTA c and panel p a
// contiguous blob
//   uint32 nepad, 3 x uint32 0, uint32 gbase[NG]   (NG = Rmax / 32 groups)
//   uint16 perm[Rmax]     sorted position t -> the CTA's local row
//   uint16 runl[Rmax]     its run length in this panel (sorted descending)
//   uint16 cols[nepad]    column - p W
//   double vals[nepad]
// Rows are sorted by run length per panel and cut into groups of 32; group g
// is stored 32-way interleaved (entry k of lane l at gbase[g] + 32 k + l) and
// padded to its longest run, so consumer thread t = 32 g + l reads coalesced,
// conflict-free shared memory and the padding is a few percent.  The running
// sums wait in shared memory between panels (the permutation changes).
#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "sgd_common.cuh"

namespace eqb {
namespace {

__device__ __forceinline__ uint32_t s32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(bar)) : "memory");
}
__device__ __forceinline__ void bar_expect(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(s32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// global -> shared bulk copy (16-byte aligned, size a multiple of 16), completion on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          s32(dst)),
      "l"(src), "r"(bytes), "r"(s32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_stream(void* dst, const void* src, unsigned bytes,
                                                unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(s32(dst)),
      "l"(src), "r"(bytes), "r"(s32(bar)), "l"(l2_evict_first())
      : "memory");
}

// ---- the pass ---------------------------------------------------------------
// Block: 32 producer threads (lane 0 issues the copies) + Rmax consumer threads.
// Dynamic shared memory: NSTAGE x (panel W doubles | blob), then sums[Rmax],
// then the barriers.
template <int MAXT>
__global__ void __launch_bounds__(MAXT, 1)
sweep_kernel(const double* __restrict__ x, double* __restrict__ rowsum, const SweepArgs sw) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  const int c = blockIdx.x;
  const int R = sw.rmax, P = sw.npanels, NST = sw.stages;
  const int NG = R / 32;
  const size_t stage_bytes = static_cast<size_t>(sw.width) * 8 + sw.blob_max;
  double* sums = reinterpret_cast<double*>(smem + stage_bytes * NST);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sums + R);
  unsigned long long* empty = full + NST;
  // the CTA's blob offsets (the producer must not wait on a global load per panel)
  int64_t* soff = reinterpret_cast<int64_t*>(empty + NST);
  for (int k = tid; k <= P; k += blockDim.x)
    soff[k] = sw.blob_off[static_cast<int64_t>(c) * P + k];

  if (tid == 0) {
    for (int k = 0; k < NST; ++k) {
      bar_init(&full[k], 1);
      bar_init(&empty[k], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid < 32) {
    if (tid == 0) {
      int st = 0;
      unsigned ph = 1;  // parity of the completion that frees the stage: 0 for its first reuse
      for (int p = 0; p < P; ++p) {
        if (p >= NST) bar_wait(&empty[st], ph);
        unsigned char* base = smem + stage_bytes * st;
        const int64_t c0 = static_cast<int64_t>(p) * sw.width;
        // (an odd tail is rounded up: the gathered vectors are followed by
        // slack words, and the extra slot is never indexed)
        const unsigned pbytes =
            static_cast<unsigned>((min(static_cast<int64_t>(sw.width), sw.ncols - c0) + 1) / 2 * 16);
        const int64_t b0 = soff[p], b1 = soff[p + 1];
        const unsigned bbytes = static_cast<unsigned>(b1 - b0);
        bar_expect(&full[st], pbytes + bbytes);
        bulk_g2s(base, x + c0, pbytes, &full[st]);
        bulk_g2s_stream(base + static_cast<size_t>(sw.width) * 8, sw.blobs + b0, bbytes, &full[st]);
        if (++st == NST) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
    return;
  }
  const int t = tid - 32;  // sorted position (consumer), t < R
  const int g = t >> 5, lane = t & 31;
  sums[t] = 0.0;
  asm volatile("bar.sync 1, %0;" ::"r"(R) : "memory");
  int st = 0;
  unsigned ph = 0;
  for (int p = 0; p < P; ++p) {
    bar_wait(&full[st], ph);
    const unsigned char* base = smem + stage_bytes * st;
    const double* panel = reinterpret_cast<const double*>(base);
    const unsigned char* blob = base + static_cast<size_t>(sw.width) * 8;
    const uint32_t* hdr = reinterpret_cast<const uint32_t*>(blob);
    const uint32_t nepad = hdr[0];
    const uint16_t* perm = reinterpret_cast<const uint16_t*>(blob + 16 + 4 * NG);
    const uint16_t* runl = perm + R;
    const uint16_t* cols = runl + R;
    const double* vals = reinterpret_cast<const double*>(cols + nepad);
    const int run = runl[t];
    const int lr = perm[t];
    const uint32_t e0 = hdr[4 + g] + lane;
    if (run > 0) {
      double acc = sums[lr];
      int k = 0;
      for (; k + 4 <= run; k += 4) {
        const uint32_t e = e0 + 32u * k;
        const unsigned c0 = cols[e], c1 = cols[e + 32], c2 = cols[e + 64], c3 = cols[e + 96];
        const double v0 = vals[e], v1 = vals[e + 32], v2 = vals[e + 64], v3 = vals[e + 96];
        EQ_CHECK(c0 < sw.width && c1 < sw.width && c2 < sw.width && c3 < sw.width);
        const double x0 = panel[c0], x1 = panel[c1], x2 = panel[c2], x3 = panel[c3];
        acc = __dadd_rn(acc, __dmul_rn(v0, x0));
        acc = __dadd_rn(acc, __dmul_rn(v1, x1));
        acc = __dadd_rn(acc, __dmul_rn(v2, x2));
        acc = __dadd_rn(acc, __dmul_rn(v3, x3));
      }
      for (; k < run; ++k) {
        const uint32_t e = e0 + 32u * k;
        EQ_CHECK(cols[e] < sw.width);
        acc = __dadd_rn(acc, __dmul_rn(vals[e], panel[cols[e]]));
      }
      sums[lr] = acc;
    }
    // the next panel's permutation may hand a row to another thread, and the
    // stage may be refilled: all consumers are done with panel p first
    asm volatile("bar.sync 1, %0;" ::"r"(R) : "memory");
    if (t == 0) bar_arrive(&empty[st]);
    if (++st == NST) {
      st = 0;
      ph ^= 1u;
    }
  }
  const int32_t row = sw.crow[static_cast<int64_t>(c) * R + t];
  if (row >= 0) rowsum[row] = sums[t];
}

// ---- layout construction ------------------------------------------------------
// per (cta, panel, local row): the first entry of the row with column >= p W,
// relative to the row start (columns ascend within a row); the run of the row
// in panel p is the difference to panel p + 1 (the row length after the last)
__global__ void sweep_runs_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                  const int32_t* __restrict__ crow, int ncta, int R, int P, int W,
                                  int32_t* __restrict__ rstart, int32_t* __restrict__ rowlen) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<int64_t>(ncta) * P * R) return;
  const int lr = static_cast<int>(idx % R);
  const int64_t cp = idx / R;
  const int p = static_cast<int>(cp % P), c = static_cast<int>(cp / P);
  const int32_t row = crow[static_cast<int64_t>(c) * R + lr];
  if (row < 0) {
    rstart[idx] = 0;
    if (p == 0) rowlen[static_cast<int64_t>(c) * R + lr] = 0;
    return;
  }
  const int64_t k0 = rp[row], k1 = rp[row + 1];
  const int64_t key = static_cast<int64_t>(p) * W;
  int64_t lo = k0, hi = k1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (ci[mid] < key) lo = mid + 1; else hi = mid;
  }
  rstart[idx] = static_cast<int32_t>(lo - k0);
  if (p == 0) rowlen[static_cast<int64_t>(c) * R + lr] = static_cast<int32_t>(k1 - k0);
}

// one CTA per (cta, panel): rows by decreasing run length (stable), the group
// bases and the padded entry count
__global__ void sweep_sort_kernel(const int32_t* __restrict__ rstart,
                                  const int32_t* __restrict__ rowlen, int R, int P,
                                  uint16_t* __restrict__ perm, uint16_t* __restrict__ srun,
                                  uint32_t* __restrict__ gbase, uint32_t* __restrict__ nepad) {
  extern __shared__ uint16_t sh[];  // runs[R], sorted[R]
  uint16_t* runs = sh;
  uint16_t* sorted = sh + R;
  const int64_t cp = blockIdx.x;
  const int t = threadIdx.x;
  const int p = static_cast<int>(cp % P);
  const int r = (p + 1 < P ? rstart[(cp + 1) * R + t] : rowlen[(cp / P) * R + t]) -
                rstart[cp * R + t];
  runs[t] = static_cast<uint16_t>(r);
  __syncthreads();
  int rank = 0;
  for (int j = 0; j < R; ++j) {
    const int rj = runs[j];
    rank += (rj > r) || (rj == r && j < t);
  }
  perm[cp * R + rank] = static_cast<uint16_t>(t);
  srun[cp * R + rank] = static_cast<uint16_t>(r);
  sorted[rank] = static_cast<uint16_t>(r);
  __syncthreads();
  if (t == 0) {
    uint32_t base = 0;
    const int NG = R / 32;
    for (int gq = 0; gq < NG; ++gq) {
      gbase[cp * NG + gq] = base;
      base += 32u * sorted[32 * gq];  // sorted descending: the group's longest run
    }
    nepad[cp] = base;
  }
}

// one CTA per (cta, panel): header, columns and / or values into the blob
__global__ void sweep_fill_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                  const double* __restrict__ va, const int32_t* __restrict__ crow,
                                  int R, int P, int W, const uint16_t* __restrict__ perm,
                                  const uint16_t* __restrict__ srun,
                                  const uint32_t* __restrict__ gbase,
                                  const uint32_t* __restrict__ nepad,
                                  const int32_t* __restrict__ rstart,
                                  const int64_t* __restrict__ blob_off, unsigned char* blobs,
                                  int do_struct, int do_vals) {
  const int64_t cp = blockIdx.x;
  const int c = static_cast<int>(cp / P), p = static_cast<int>(cp % P);
  const int t = threadIdx.x;
  const int NG = R / 32;
  unsigned char* blob = blobs + blob_off[cp];
  const uint32_t ne = nepad[cp];
  uint32_t* hdr = reinterpret_cast<uint32_t*>(blob);
  uint16_t* bperm = reinterpret_cast<uint16_t*>(blob + 16 + 4 * NG);
  uint16_t* brun = bperm + R;
  uint16_t* bcols = brun + R;
  double* bvals = reinterpret_cast<double*>(bcols + ne);
  const int lr = perm[cp * R + t];
  const int run = srun[cp * R + t];
  if (do_struct) {
    if (t < 4) hdr[t] = t == 0 ? ne : 0u;
    if (t < NG) hdr[4 + t] = gbase[cp * NG + t];
    bperm[t] = static_cast<uint16_t>(lr);
    brun[t] = static_cast<uint16_t>(run);
  }
  if (run == 0) return;
  const int32_t row = crow[static_cast<int64_t>(c) * R + lr];
  const int64_t src = rp[row] + rstart[cp * R + lr];
  const uint32_t e0 = gbase[cp * NG + (t >> 5)] + (t & 31);
  const int32_t cbase = p * W;
  for (int k = 0; k < run; ++k) {
    if (do_struct) bcols[e0 + 32u * k] = static_cast<uint16_t>(ci[src + k] - cbase);
    if (do_vals) bvals[e0 + 32u * k] = va[src + k];
  }
}

}  // namespace

size_t sweep_smem_bytes(const SweepArgs& sw) {
  return (static_cast<size_t>(sw.width) * 8 + sw.blob_max) * sw.stages +
         static_cast<size_t>(sw.rmax) * 8 + 2 * sizeof(unsigned long long) * sw.stages +
         static_cast<size_t>(sw.npanels + 1) * 8;
}

cudaError_t launch_sweep(const double* x, double* rowsum, const SweepArgs& sw, cudaStream_t s) {
  if (sw.nctas == 0) return cudaSuccess;
  static std::atomic<unsigned long long> done{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ULL << (dev & 63);
  if (!(done.load() & bit)) {
    e = cudaFuncSetAttribute(sweep_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(sweep_kernel<928>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024);
    if (e != cudaSuccess) return e;
    done.fetch_or(bit);
  }
  const unsigned threads = 32 + sw.rmax;
  if (threads <= 512)  // more registers per thread for the pipelined chains
    sweep_kernel<512><<<static_cast<unsigned>(sw.nctas), threads, sweep_smem_bytes(sw), s>>>(
        x, rowsum, sw);
  else
    sweep_kernel<928><<<static_cast<unsigned>(sw.nctas), threads, sweep_smem_bytes(sw), s>>>(
        x, rowsum, sw);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_sweep_runs(const int64_t* rp, const int32_t* ci, const int32_t* crow, int ncta,
                              int R, int P, int W, int32_t* rstart, int32_t* rowlen,
                              cudaStream_t s) {
  const int64_t n = static_cast<int64_t>(ncta) * R * P;
  if (n == 0) return cudaSuccess;
  sweep_runs_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(rp, ci, crow, ncta, R, P,
                                                                          W, rstart, rowlen);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_sweep_sort(const int32_t* rstart, const int32_t* rowlen, int ncta, int R, int P,
                              uint16_t* perm, uint16_t* srun, uint32_t* gbase, uint32_t* nepad,
                              cudaStream_t s) {
  const int64_t n = static_cast<int64_t>(ncta) * P;
  if (n == 0) return cudaSuccess;
  sweep_sort_kernel<<<static_cast<unsigned>(n), R, 4 * R, s>>>(rstart, rowlen, R, P, perm, srun,
                                                              gbase, nepad);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_sweep_fill(const int64_t* rp, const int32_t* ci, const double* va,
                              const int32_t* crow, int ncta, int R, int P, int W,
                              const uint16_t* perm, const uint16_t* srun, const uint32_t* gbase,
                              const uint32_t* nepad, const int32_t* rstart, const int64_t* blob_off,
                              unsigned char* blobs, bool do_struct, bool do_vals, cudaStream_t s) {
  const int64_t n = static_cast<int64_t>(ncta) * P;
  if (n == 0) return cudaSuccess;
  sweep_fill_kernel<<<static_cast<unsigned>(n), R, 0, s>>>(rp, ci, va, crow, R, P, W, perm, srun,
                                                          gbase, nepad, rstart, blob_off, blobs,
                                                          do_struct ? 1 : 0, do_vals ? 1 : 0);
  count_launch(s);
  return cudaGetLastError();
}

}  // namespace eqb
