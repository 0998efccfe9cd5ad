// transpose.cu -- K2: CSR(A^T) built on the device, bit-exact to
// ExplicitMatrix::transposed() (src/explicit_matrix.cpp:117-125).
//
// transposed() emits {j, i, v} in CSR order and sparse() sorts by (j, i)
// (:28-31); CSR order is ascending in i, so CSR(A^T) is the STABLE counting
// sort of A's entries by column.  Hand-written as an MSD partition of the
// column index in a few levels (level_bits: <= 7 bits each):
//
//   count    one warp per chunk of <= kChunkE consecutive entries of a segment
//            (the entries whose columns share the bits above this level) counts
//            its entries per bucket in warp-private shared memory (match_any
//            aggregation, no atomics);
//   scan     one exclusive scan over all counts, laid out segment-major, then
//            bucket, then chunk, gives every (chunk, bucket) run its output
//            offset -- runs of a bucket in chunk (= input) order, so stable;
//   scatter  each warp re-reads its chunk in order and writes every entry to its
//            run at its rank (match_any + popc: lane order = input order),
//            staged in shared memory so runs leave in whole 64-byte granules.
//
// At the last level a bucket is one column and the offsets ARE CSR(A^T)'s
// positions.  The segments come from CSR(A^T)'s row pointers on the host.
// Only columns are needed, so all of this runs while A's values are still
// crossing PCIe; the values then take one gather (transpose_values).
#include <algorithm>
#include <cstdint>
#include <vector>

#include "internal.h"

namespace eqb {
namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 8;  // elements per thread per scan block

// -------------------------------------------------------------- exclusive scan
template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const T o = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += o;
  }
  return v;
}

// block-wide exclusive scan of one value per thread; returns the block total
template <class T>
__device__ __forceinline__ T block_excl_scan(T v, T& total) {
  __shared__ T wsum[32];
  __shared__ T wtot;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T inc = warp_incl_scan(v);
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    const T w = lane < nw ? wsum[lane] : T(0);
    const T wi = warp_incl_scan(w);
    if (lane < nw) wsum[lane] = wi - w;
    if (lane == 31) wtot = wi;
  }
  __syncthreads();
  const T out = inc - v + wsum[warp];
  total = wtot;
  __syncthreads();
  return out;
}

// phase 1: per-block sums
template <class T>
__global__ void __launch_bounds__(kScanThreads) scan_sums_kernel(const T* __restrict__ in, int64_t n,
                                                               T* __restrict__ sums) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanThreads * kScanItems;
  T acc = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t k = base + static_cast<int64_t>(j) * kScanThreads + threadIdx.x;
    if (k < n) acc += in[k];
  }
  T total;
  block_excl_scan(acc, total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// phase 2: exclusive scan of the block sums (one CTA, sequential chunks)
template <class T>
__global__ void __launch_bounds__(kScanThreads) scan_top_kernel(T* __restrict__ sums, int64_t nb) {
  T carry = 0;
  for (int64_t c = 0; c < nb; c += kScanThreads) {
    const int64_t k = c + threadIdx.x;
    const T v = k < nb ? sums[k] : T(0);
    T total;
    const T ex = block_excl_scan(v, total);
    if (k < nb) sums[k] = carry + ex;
    carry += total;
  }
}

// phase 3: out[k] = offset of the block + exclusive scan inside it (thread t
// owns kScanItems consecutive elements so the block scan stays in order)
template <class T>
__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(const T* __restrict__ in,
                                                                int64_t n,
                                                                const T* __restrict__ sums,
                                                                T* __restrict__ out) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanThreads * kScanItems;
  const int64_t my = base + static_cast<int64_t>(threadIdx.x) * kScanItems;
  T v[kScanItems];
  T acc = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    v[j] = my + j < n ? in[my + j] : T(0);
    acc += v[j];
  }
  T total;
  T run = block_excl_scan(acc, total) + sums[blockIdx.x];
#pragma unroll
  for (int j = 0; j < kScanItems; ++j)
    if (my + j < n) {
      const T x = v[j];
      out[my + j] = run;
      run += x;
    }
}

// ------------------------------------------------------------ column counts
// CSR(A^T) row pointers: per-column counts (one atomic per distinct column in
// a warp's 32 entries), then an exclusive scan.  cnt has cols + 1 slots and
// receives the row pointers in place.
__global__ void col_hist_kernel(const int32_t* __restrict__ col, int64_t nnz,
                                unsigned long long* __restrict__ cnt) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
       k += stride) {
    const int32_t c = __ldg(col + k);
    const unsigned peers = __match_any_sync(__activemask(), c);
    const int leader = __ffs(peers) - 1;
    if ((threadIdx.x & 31) == leader) atomicAdd(cnt + c, static_cast<unsigned long long>(__popc(peers)));
  }
}

// row index of every entry (rows ascending, empty rows skipped): thread per
// 32-entry run, binary search for the first, then a forward walk
constexpr int kExpand = 32;
__global__ void expand_rows_kernel(const int64_t* __restrict__ rp, int64_t rows, int64_t nnz,
                                   int32_t* __restrict__ rowidx) {
  const int64_t k0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) * kExpand;
  if (k0 >= nnz) return;
  int64_t lo = 0, hi = rows;  // rp[lo] <= k0 < rp[hi]
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (rp[mid] <= k0) lo = mid; else hi = mid;
  }
  int64_t next = rp[lo + 1];
  const int64_t k1 = k0 + kExpand < nnz ? k0 + kExpand : nnz;
  for (int64_t k = k0; k < k1; ++k) {
    while (k >= next) next = rp[++lo + 1];
    rowidx[k] = static_cast<int32_t>(lo);
  }
}

// ------------------------------------------------------- partition levels
// One level of the MSD partition: the entries of every segment (a contiguous
// range whose columns share the high bits above shift + bits) are split into
// 2^bits buckets by (col >> shift) & mask, stably.  Work unit = one warp-chunk
// (<= kChunkE consecutive entries inside one segment).  A chunk's count of
// bucket b lives at cbase + b * nch + idx (segment-major, then bucket, then
// chunk), so one exclusive scan over all counts gives every (chunk, bucket) run
// its output offset, runs of a bucket in chunk (= input) order.
struct PartChunk {
  int64_t start, end;  // entry range
  int64_t cbase;       // counts base of the segment
  int32_t nch, idx;    // chunks in the segment, this chunk's index
};
constexpr int kChunkE = 16384;
constexpr int kPartWarps = 4;

__global__ void __launch_bounds__(32 * kPartWarps)
part_count_kernel(const int32_t* __restrict__ col, const PartChunk* __restrict__ chunks,
                  int nchunks, int shift, int bits, int32_t* __restrict__ cnt) {
  __shared__ int32_t sc[kPartWarps][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ci = blockIdx.x * kPartWarps + warp;
  const int nb = 1 << bits;
  for (int j = lane; j < nb; j += 32) sc[warp][j] = 0;
  __syncwarp();
  if (ci >= nchunks) return;
  const PartChunk ch = chunks[ci];
  for (int64_t b = ch.start; b < ch.end; b += 32) {
    const int64_t k = b + lane;
    const int bk = k < ch.end ? (__ldg(col + k) >> shift) & (nb - 1) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, bk);
    if (bk >= 0 && lane == __ffs(peers) - 1) sc[warp][bk] += __popc(peers);
    __syncwarp();
  }
  for (int j = lane; j < nb; j += 32) cnt[ch.cbase + static_cast<int64_t>(j) * ch.nch + ch.idx] = sc[warp][j];
}

// Scatter with write staging: every (chunk, bucket) run is written in whole
// 16-entry granules (64 bytes, the DRAM access granule) from a per-warp
// shared-memory line per bucket; only a run's first and last granules can be
// partial.  Scattered 4-byte stores instead measured ~3.5x the algorithmic
// DRAM bytes (read-modify-write of partially written granules evicted early).
// src null on the first level (src = entry index); ocol null on the last
// (CSR(A^T)'s column is the entry's row, kept in orow).
constexpr int kLine = 16;
constexpr int kMaxBuckets = 128;
struct ScatterSmem {
  int32_t cur[kMaxBuckets];    // next output position of the bucket's run
  int32_t first[kMaxBuckets];  // the run's first position (mask of its first granule)
  int32_t line[3][kMaxBuckets][kLine];
};

__device__ __forceinline__ void flush_line(ScatterSmem& S, int bk, int32_t ln, int lo, int hi,
                                           int32_t* __restrict__ o0, int32_t* __restrict__ o1,
                                           int32_t* __restrict__ o2, int lane) {
  // lanes 0-15: arrays 0 / 2; lanes 16-31: array 1
  const int l = lane & (kLine - 1);
  const int64_t p = static_cast<int64_t>(ln) * kLine + l;
  if (l >= lo && l < hi) {
    if (lane < kLine) {
      if (o0) o0[p] = S.line[0][bk][l];
    } else {
      o1[p] = S.line[1][bk][l];
    }
  }
  if (lane < kLine && l >= lo && l < hi) o2[p] = S.line[2][bk][l];
}

__global__ void __launch_bounds__(32 * kPartWarps)
part_scatter_kernel(const int32_t* __restrict__ col, const int32_t* __restrict__ row,
                    const int32_t* __restrict__ src, const PartChunk* __restrict__ chunks,
                    int nchunks, int shift, int bits, const int32_t* __restrict__ off,
                    int32_t* __restrict__ ocol, int32_t* __restrict__ orow,
                    int32_t* __restrict__ osrc, int64_t total) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  ScatterSmem& S = reinterpret_cast<ScatterSmem*>(smraw)[warp];
  const int ci = blockIdx.x * kPartWarps + warp;
  if (ci >= nchunks) return;
  const int nb = 1 << bits;
  const PartChunk ch = chunks[ci];
  for (int j = lane; j < nb; j += 32) {
    const int32_t o = off[ch.cbase + static_cast<int64_t>(j) * ch.nch + ch.idx];
    S.cur[j] = o;
    S.first[j] = o;
  }
  __syncwarp();
  const unsigned lt = (1u << lane) - 1u;
  // one step ahead: this lane's next entry
  int64_t k = ch.start + lane;
  int32_t c = 0, r = 0, sr = 0;
  if (k < ch.end) {
    c = __ldg(col + k);
    r = __ldg(row + k);
    sr = src ? __ldg(src + k) : static_cast<int32_t>(k);
  }
  for (int64_t b = ch.start; b < ch.end; b += 32) {
    const bool ok = k < ch.end;
    const int32_t cc = c, rr = r, ss = sr;
    k += 32;
    if (k < ch.end) {
      c = __ldg(col + k);
      r = __ldg(row + k);
      sr = src ? __ldg(src + k) : static_cast<int32_t>(k);
    }
    const int bk = ok ? (cc >> shift) & (nb - 1) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, bk);
    const int leader = __ffs(peers) - 1;
    const int cnt = __popc(peers);
    int32_t base = 0;
    if (ok && lane == leader) base = S.cur[bk];
    base = __shfl_sync(0xffffffffu, base, leader);
    const int32_t pos = base + __popc(peers & lt);
    EQ_CHECK(!ok || (pos >= 0 && pos < total));
    const int32_t l0 = base / kLine;  // positions are >= 0
    // a bucket's entries of this step span at most 3 granules: fill, flush full ones
    for (int ph = 0; ph < 3; ++ph) {
      if (ok && pos / kLine - l0 == ph) {
        S.line[0][bk][pos % kLine] = cc;
        S.line[1][bk][pos % kLine] = rr;
        S.line[2][bk][pos % kLine] = ss;
      }
      __syncwarp();
      // granule l0 + ph is complete if this step's run passes its end
      const bool full = ok && lane == leader && base + cnt >= (l0 + ph + 1) * kLine;
      unsigned fm = __ballot_sync(0xffffffffu, full);
      while (fm) {
        const int src_lane = __ffs(fm) - 1;
        fm &= fm - 1;
        const int fb = __shfl_sync(0xffffffffu, bk, src_lane);
        const int32_t fl = __shfl_sync(0xffffffffu, l0, src_lane) + ph;
        const int32_t fst = S.first[fb];
        const int lo = fst > fl * kLine ? fst - fl * kLine : 0;
        flush_line(S, fb, fl, lo, kLine, ocol, orow, osrc, lane);
      }
      __syncwarp();
    }
    if (ok && lane == leader) S.cur[bk] = base + cnt;
    __syncwarp();
  }
  // the last, partial granule of every run
  for (int j = 0; j < nb; ++j) {
    const int32_t cur = S.cur[j];
    if (cur % kLine == 0 || cur == S.first[j]) continue;
    const int32_t fl = cur / kLine;
    const int32_t fst = S.first[j];
    const int lo = fst > fl * kLine ? fst - fl * kLine : 0;
    flush_line(S, j, fl, lo, cur % kLine, ocol, orow, osrc, lane);
  }
}

// CSR(A^T)'s values: AT.val[q] = val[srcT[q]]
__global__ void gather_values_kernel(const double* __restrict__ val,
                                     const int32_t* __restrict__ srcT, int64_t n,
                                     double* __restrict__ out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n;
       q += stride)
    __stcs(out + q, __ldg(val + __ldcs(srcT + q)));
}

int sm_count() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaGetLastError();
  return sms;
}

}  // namespace

template <class T>
cudaError_t exclusive_scan(const T* in, T* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t per = static_cast<int64_t>(kScanThreads) * kScanItems;
  const int64_t nb = (n + per - 1) / per;
  T* sums = nullptr;
  cudaError_t e = cudaMallocAsync(&sums, nb * sizeof(T), s);
  if (e) return e;
  scan_sums_kernel<T><<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(in, n, sums);
  scan_top_kernel<T><<<1, kScanThreads, 0, s>>>(sums, nb);
  scan_apply_kernel<T><<<static_cast<unsigned>(nb), kScanThreads, 0, s>>>(in, n, sums, out);
  count_launch(s, 3);
  e = cudaGetLastError();
  cudaFreeAsync(sums, s);
  return e;
}
template cudaError_t exclusive_scan<int32_t>(const int32_t*, int32_t*, int64_t, cudaStream_t);
template cudaError_t exclusive_scan<int64_t>(const int64_t*, int64_t*, int64_t, cudaStream_t);
template cudaError_t exclusive_scan<unsigned long long>(const unsigned long long*,
                                                        unsigned long long*, int64_t,
                                                        cudaStream_t);

cudaError_t launch_col_rowptr(const int32_t* col, int64_t nnz, int64_t cols, int64_t* rp,
                              cudaStream_t s) {
  // counts into rp[0, cols), then rp = exclusive scan over cols + 1 slots
  cudaError_t e = cudaMemsetAsync(rp, 0, (cols + 1) * 8, s);
  if (e) return e;
  if (nnz > 0) {
    const int64_t blocks = std::min<int64_t>((nnz + 255) / 256, 8LL * sm_count() * 8);
    col_hist_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(
        col, nnz, reinterpret_cast<unsigned long long*>(rp));
    count_launch(s);
    if ((e = cudaGetLastError())) return e;
  }
  return exclusive_scan(reinterpret_cast<const unsigned long long*>(rp),
                        reinterpret_cast<unsigned long long*>(rp), cols + 1, s);
}

TransposeWork::~TransposeWork() { release(); }

void TransposeWork::release() {
  if (srcT) cudaFreeAsync(srcT, stream);
  srcT = nullptr;
}

// Level plan: the bits of the column index split MSD-first into levels of
// <= 7 bits (the last level's buckets are single columns).
static std::vector<int> level_bits(int64_t n) {
  int total = 0;
  while ((1LL << total) < n) ++total;
  const int nl = std::max(1, (total + 6) / 7);
  std::vector<int> lv;
  int rest = std::max(total, 1);
  for (int i = 0; i < nl; ++i) {  // as even as possible, the larger ones first
    const int b = (rest + (nl - i) - 1) / (nl - i);
    lv.push_back(b);
    rest -= b;
  }
  return lv;
}

// rpT_host: CSR(A^T)'s row pointers on the host (n + 1); AT.row_ptr on the
// device.  Writes AT.col; keeps the source index of every CSR(A^T) entry in w
// for transpose_values.
cudaError_t transpose_structure(const DevCsr& A, DevCsr& AT, const int64_t* rpT_host,
                                TransposeWork& w, cudaStream_t s, const HostUpload& upload) {
  const int64_t nnz = A.nnz, n = A.cols;
  AT.rows = A.cols;
  AT.cols = A.rows;
  AT.nnz = nnz;
  w.release();
  w.stream = s;
  w.nnz = nnz;
  if (nnz == 0) return cudaSuccess;
  if (nnz >= (1LL << 31) || A.rows >= (1LL << 31) || n >= (1LL << 31))
    return cudaErrorInvalidValue;
  cudaError_t e;
  const std::vector<int> lv = level_bits(n);
  int32_t *rowidx = nullptr, *bufc[2] = {nullptr, nullptr}, *bufr[2] = {nullptr, nullptr},
          *bufs[2] = {nullptr, nullptr}, *cnt = nullptr;
  PartChunk* dch = nullptr;
  auto cleanup = [&] {
    for (int32_t* p : {rowidx, bufc[0], bufc[1], bufr[0], bufr[1], bufs[0], bufs[1], cnt})
      if (p) cudaFreeAsync(p, s);
    if (dch) cudaFreeAsync(dch, s);
  };
  do {
    if ((e = cudaMallocAsync(reinterpret_cast<void**>(&w.srcT), nnz * 4, s))) break;
    if ((e = cudaMallocAsync(reinterpret_cast<void**>(&rowidx), nnz * 4, s))) break;
    for (int i = 0; i < 2 && lv.size() > 1; ++i) {
      if ((e = cudaMallocAsync(reinterpret_cast<void**>(&bufc[i]), nnz * 4, s))) break;
      if ((e = cudaMallocAsync(reinterpret_cast<void**>(&bufr[i]), nnz * 4, s))) break;
      if ((e = cudaMallocAsync(reinterpret_cast<void**>(&bufs[i]), nnz * 4, s))) break;
    }
    if (e) break;
    const int64_t nexp = (nnz + kExpand - 1) / kExpand;
    expand_rows_kernel<<<static_cast<unsigned>((nexp + 255) / 256), 256, 0, s>>>(
        A.row_ptr, A.rows, nnz, rowidx);
    count_launch(s);
    const int32_t* icol = A.col;
    const int32_t* irow = rowidx;
    const int32_t* isrc = nullptr;
    int shift = 0;
    for (int b : lv) shift += b;
    std::vector<PartChunk> ch;
    cudaFuncSetAttribute(part_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kPartWarps * sizeof(ScatterSmem)));
    for (size_t l = 0; l < lv.size(); ++l) {
      const int bits = lv[l];
      const int seg_shift = shift;  // segments: columns sharing col >> seg_shift
      shift -= bits;
      const bool final = l + 1 == lv.size();
      // chunks of every segment (segment p covers columns [p << seg_shift, ...))
      ch.clear();
      int64_t cbase = 0;
      const int64_t nseg = seg_shift >= 62 ? 1 : ((n - 1) >> seg_shift) + 1;
      for (int64_t p = 0; p < nseg; ++p) {
        const int64_t c0 = p << seg_shift, c1 = std::min(n, (p + 1) << seg_shift);
        const int64_t e0 = rpT_host[c0], e1 = rpT_host[c1];
        const int32_t nc = static_cast<int32_t>((e1 - e0 + kChunkE - 1) / kChunkE);
        for (int32_t i = 0; i < nc; ++i)
          ch.push_back({e0 + static_cast<int64_t>(i) * kChunkE,
                        std::min(e1, e0 + static_cast<int64_t>(i + 1) * kChunkE), cbase, nc, i});
        cbase += static_cast<int64_t>(nc) << bits;
      }
      if (ch.empty()) break;
      if (dch) cudaFreeAsync(dch, s);
      if (cnt) cudaFreeAsync(cnt, s);
      dch = nullptr;
      cnt = nullptr;
      if ((e = cudaMallocAsync(reinterpret_cast<void**>(&dch), ch.size() * sizeof(PartChunk), s))) break;
      if (upload) {
        upload(dch, ch.data(), ch.size() * sizeof(PartChunk));
      } else if ((e = cudaMemcpyAsync(dch, ch.data(), ch.size() * sizeof(PartChunk),
                                      cudaMemcpyHostToDevice, s))) {
        break;
      }
      if ((e = cudaMallocAsync(reinterpret_cast<void**>(&cnt), cbase * 4, s))) break;
      const int nchunks = static_cast<int>(ch.size());
      const unsigned grid = static_cast<unsigned>((nchunks + kPartWarps - 1) / kPartWarps);
      part_count_kernel<<<grid, 32 * kPartWarps, 0, s>>>(icol, dch, nchunks, shift, bits, cnt);
      count_launch(s);
      if ((e = cudaGetLastError())) break;
      if ((e = exclusive_scan(cnt, cnt, cbase, s))) break;
      const int o = static_cast<int>(l & 1);
      int32_t* oc = final ? nullptr : bufc[o];
      int32_t* orow = final ? AT.col : bufr[o];
      int32_t* osrc = final ? w.srcT : bufs[o];
      part_scatter_kernel<<<grid, 32 * kPartWarps, kPartWarps * sizeof(ScatterSmem), s>>>(
          icol, irow, isrc, dch, nchunks, shift, bits, cnt, oc, orow, osrc, nnz);
      count_launch(s);
      if ((e = cudaGetLastError())) break;
      icol = oc;
      irow = orow;
      isrc = osrc;
    }
  } while (0);
  cleanup();
  return e;
}

cudaError_t transpose_values(const DevCsr& A, DevCsr& AT, TransposeWork& w, cudaStream_t s) {
  if (w.nnz == 0) return cudaSuccess;
  if (!w.srcT) return cudaErrorInvalidValue;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((w.nnz + 255) / 256,
                                                                  16LL * sm_count()));
  gather_values_kernel<<<blocks, 256, 0, s>>>(A.val, w.srcT, w.nnz, AT.val);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t transpose_csr(const DevCsr& A, DevCsr& AT, const int64_t* rpT_host, cudaStream_t s,
                          cudaEvent_t val_ready) {
  TransposeWork w;
  cudaError_t e = transpose_structure(A, AT, rpT_host, w, s);
  if (e) return e;
  if (val_ready && (e = cudaStreamWaitEvent(s, val_ready, 0))) return e;
  return transpose_values(A, AT, w, s);  // w's buffer is freed stream-ordered
}

}  // namespace eqb
