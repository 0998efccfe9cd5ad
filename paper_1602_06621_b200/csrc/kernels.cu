// kernels.cu -- sm_100a kernels for the equilibration hot path.
//
//   K1 sign stream    mt_jump_kernel / mt_gen_kernel  (src/rng.cpp:19-64)
//   K2 transpose      transpose_csr (stable radix by column; explicit_matrix.cpp:117-125)
//   K3/K4 SGD pass    sgd_iter_kernel: CSR(A) rows and CSR(A^T) rows in one
//                     launch, products staged in shared memory, each row summed
//                     sequentially in CSR order (explicit_matrix.cpp:70-78 and the
//                     ascending-row scatter :85-92), fused u/v epilogue
//                     (equilibrate.cpp:106-129) that also writes next e.*s, d.*w
//   K5 dense          dense_rows_kernel / dense_cols_* (canonical GEMV order)
//   K7 LSQR           pass_kernel + canonical reductions + vector updates
//                     (lsqr.cpp:36-80)
//
// Every floating-point operation that feeds the trajectory is an explicit
// round-to-nearest intrinsic; the library is also built with --fmad=false.
#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "internal.h"
#include "mt64_host.h"
#include "sgd_common.cuh"

namespace eqb {

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) {
  return a < b ? a : b;
}

// Kernel-launch accounting for bench.py's "gpu_launches" (launches issued while
// a stream is being captured are counted when the graph is replayed instead).
static std::atomic<long long> g_launches{0};
void note_launches(long long n) { g_launches += n; }
long long launch_count() { return g_launches.load(); }
void count_launch(cudaStream_t s, int n) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &st) != cudaSuccess) {
    cudaGetLastError();
    st = cudaStreamCaptureStatusNone;
  }
  if (st == cudaStreamCaptureStatusNone) g_launches += n;
}

#define EQ_CUDA_TRY(x)                   \
  do {                                   \
    cudaError_t e_ = (x);                \
    if (e_ != cudaSuccess) return e_;    \
  } while (0)

// ---------------------------------------------------------------------------
// K1: MT19937-64 sign stream
// ---------------------------------------------------------------------------
namespace {

constexpr uint64_t kMtA = 0xB5026F5AA96619E9ULL;
constexpr uint64_t kMtUM = 0xFFFFFFFF80000000ULL;
constexpr uint64_t kMtLM = 0x000000007FFFFFFFULL;
constexpr int kJumpWords = mt::kDegree + mt::kN - 1;  // 20248 generated words
constexpr int kMtThreads = 320;                       // >= 312, whole warps
constexpr int kPackOutputs = 312 * 32;                // outputs per pack round

__device__ __forceinline__ uint64_t mt_next(uint64_t a, uint64_t b, uint64_t c) {
  const uint64_t y = (a & kMtUM) | (b & kMtLM);
  return c ^ (y >> 1) ^ ((y & 1ULL) ? kMtA : 0ULL);
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

// One CTA per jump: W[dst0 + b] = sum_i r_i W_{p+i}, p = position of W[src0 + b].
// The set bits of r are given as a host-expanded list of positions (uint16,
// padded to a multiple of 8 with kJumpWords, whose window reads zeros).
// kJumpGroups thread groups of kMtThreads split the position list and XOR
// their partial sums (GF(2): any order gives the same words).
constexpr int kJumpGroups = 3;
__global__ void __launch_bounds__(kMtThreads * kJumpGroups)
mt_jump_kernel(uint64_t* __restrict__ windows, int src0, int dst0,
               const uint4* __restrict__ pos8, int npos8) {
  extern __shared__ uint64_t sx[];  // kJumpWords + kN zero words, then the partials
  const int tid = threadIdx.x;
  const uint64_t* src = windows + static_cast<size_t>(src0 + blockIdx.x) * mt::kN;
  for (int j = tid; j < mt::kN; j += blockDim.x) {
    sx[j] = src[j];
    sx[kJumpWords + j] = 0;
  }
  __syncthreads();
  for (int q = 0; q + mt::kN < kJumpWords; q += mt::kN) {
    const int j = tid;
    if (j < mt::kM && q + mt::kN + j < kJumpWords)
      sx[q + mt::kN + j] = mt_next(sx[q + j], sx[q + j + 1], sx[q + mt::kM + j]);
    __syncthreads();
    if (j >= mt::kM && j < mt::kN && q + mt::kN + j < kJumpWords)
      sx[q + mt::kN + j] = mt_next(sx[q + j], sx[q + j + 1], sx[q + mt::kM + j]);
    __syncthreads();
  }
  const int grp = tid / kMtThreads, t = tid - grp * kMtThreads;
  uint64_t* part = sx + kJumpWords + mt::kN;  // [kJumpGroups - 1][kN]
  if (t < mt::kN) {
    uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    const uint64_t* x = sx + t;
    const int q0 = npos8 * grp / kJumpGroups, q1 = npos8 * (grp + 1) / kJumpGroups;
    for (int q = q0; q < q1; ++q) {
      const uint4 p = __ldg(pos8 + q);  // 8 positions, warp-uniform (broadcast)
      a0 ^= x[p.x & 0xffff];
      a1 ^= x[p.x >> 16];
      a2 ^= x[p.y & 0xffff];
      a3 ^= x[p.y >> 16];
      a0 ^= x[p.z & 0xffff];
      a1 ^= x[p.z >> 16];
      a2 ^= x[p.w & 0xffff];
      a3 ^= x[p.w >> 16];
    }
    if (grp > 0) part[(grp - 1) * mt::kN + t] = (a0 ^ a1) ^ (a2 ^ a3);
    a0 ^= a1;
    a2 ^= a3;
    a0 ^= a2;
    if (grp == 0) part[(kJumpGroups - 1) * mt::kN + t] = a0;
  }
  __syncthreads();
  if (grp == 0 && t < mt::kN) {
    uint64_t w = part[(kJumpGroups - 1) * mt::kN + t];
    for (int g = 0; g < kJumpGroups - 1; ++g) w ^= part[g * mt::kN + t];
    windows[static_cast<size_t>(dst0 + blockIdx.x) * mt::kN + t] = w;
  }
}

// One CTA per segment: outputs [g*L, min((g+1)*L, total)) -> sign bits.
__global__ void __launch_bounds__(kMtThreads)
mt_gen_kernel(const uint64_t* __restrict__ windows, uint64_t seg_len,
              uint64_t total, uint32_t* __restrict__ bits) {
  __shared__ uint64_t ring[2 * mt::kN];
  __shared__ uint8_t sbit[kPackOutputs];
  const int tid = threadIdx.x;
  const uint64_t g = blockIdx.x;
  const uint64_t start = g * seg_len;
  const uint64_t len = min(seg_len, total - start);
  for (int j = tid; j < mt::kN; j += blockDim.x)
    ring[j] = windows[g * mt::kN + j];
  __syncthreads();
  // local word index p (p >= 312) lives at ring[p % 624]; output k = p - 312.
  for (uint64_t base = 0; base < len; base += kPackOutputs) {
    const uint64_t blen = min(static_cast<uint64_t>(kPackOutputs), len - base);
    for (int b = 0; b < static_cast<int>(blen); b += mt::kN) {
      // base is a multiple of 624, so the batch's first word p0 = base + b + 312
      // sits in ring slot 312 on even batches and slot 0 on odd ones
      const int j = tid;
      const int s0 = ((b / mt::kN) & 1) ? 0 : mt::kN;  // slot of p0
      const int sp = s0 + j;                             // slot of p = p0 + j
      const int sm312 = mt::kN - s0 + j;                 // slot of p - 312
      const int sm311 = sm312 + 1 == 2 * mt::kN ? 0 : sm312 + 1;
      const int sm156 = sp >= mt::kM ? sp - mt::kM : sp + 2 * mt::kN - mt::kM;
      if (j < mt::kM) {
        const uint64_t w = mt_next(ring[sm312], ring[sm311], ring[sm156]);
        ring[sp] = w;
        sbit[b + j] = static_cast<uint8_t>(mt_temper(w) >> 63);
      }
      __syncthreads();
      if (j >= mt::kM && j < mt::kN) {
        const uint64_t w = mt_next(ring[sm312], ring[sm311], ring[sm156]);
        ring[sp] = w;
        sbit[b + j] = static_cast<uint8_t>(mt_temper(w) >> 63);
      }
      __syncthreads();
    }
    // pack: word wi covers outputs base + 32*wi .. +31 (start is 32-aligned)
    const int nwords = static_cast<int>((blen + 31) / 32);
    for (int wi = tid; wi < nwords; wi += blockDim.x) {
      uint32_t word = 0;
      for (int k = 0; k < 32; ++k) {
        const uint64_t o = static_cast<uint64_t>(wi) * 32 + k;
        if (o < blen && sbit[o]) word |= 1u << k;
      }
      bits[(start + base) / 32 + wi] = word;
    }
    __syncthreads();
  }
}

int ceil_log2(uint64_t x) {
  int k = 0;
  while ((1ULL << k) < x) ++k;
  return k;
}

// Segment length L = 2^k: trade jump-tree levels against the sequential length
// each segment generates.  Model (B200, measured): a jump wave (one CTA per SM,
// 172 KB of shared memory) ~0.09 ms; generation ~0.76 us per 1000 outputs per
// CTA, six CTAs per SM.
int choose_seg_log2(uint64_t total) {
  int best = 14;
  double best_cost = 1e300;
  for (int k = 14; k <= 40; ++k) {
    const uint64_t L = 1ULL << k;
    const uint64_t G = (total + L - 1) / L;
    const int levels = ceil_log2(G);
    double cost = 0.0;
    for (int a = 0; a < levels; ++a) {
      const uint64_t cnt = std::min<uint64_t>(1ULL << a, G - (1ULL << a));
      cost += static_cast<double>((cnt + 147) / 148) * 0.09;
    }
    cost += static_cast<double>((G + 148 * 6 - 1) / (148 * 6)) *
            static_cast<double>(std::min(L, total)) * 7.6e-7;
    if (cost < best_cost) {
      best_cost = cost;
      best = k;
    }
    if (L >= total) break;
  }
  return best;
}

}  // namespace

constexpr int kPosCap = 20000;  // >= 19937 set bits, padded to a multiple of 8

size_t sign_stream_scratch_bytes(uint64_t total) {
  if (total == 0) return 0;
  const int k = choose_seg_log2(total);
  const uint64_t G = (total + (1ULL << k) - 1) >> k;
  const int levels = ceil_log2(G);
  return G * mt::kN * sizeof(uint64_t) +
         static_cast<size_t>(levels + 1) * kPosCap * sizeof(uint16_t);
}

cudaError_t sign_stream_generate(uint64_t seed, uint64_t stream, uint64_t total,
                                 uint32_t* bits, void* scratch,
                                 size_t scratch_bytes, cudaStream_t s) {
  if (total == 0) return cudaSuccess;
  if (scratch_bytes < sign_stream_scratch_bytes(total)) return cudaErrorInvalidValue;
  const int k = choose_seg_log2(total);
  const uint64_t L = 1ULL << k;
  const uint64_t G = (total + L - 1) / L;
  const int levels = ceil_log2(G);
  uint64_t* windows = static_cast<uint64_t*>(scratch);
  uint16_t* pos = reinterpret_cast<uint16_t*>(windows + G * mt::kN);
  // host: seeding state and, per tree level, the set-bit positions of the
  // jump polynomial x^(2^(k+a)) mod phi
  static thread_local std::vector<uint64_t> seedw(mt::kN);
  static thread_local std::vector<uint16_t> hpos;
  std::vector<int> npos8(levels);
  hpos.assign(static_cast<size_t>(levels) * kPosCap, static_cast<uint16_t>(kJumpWords));
  mt::seed_state(seed, stream, seedw.data());
  // set-bit positions of x^(2^j) mod phi: constants of the generator, computed
  // once per j and process (the per-call scan of 19937 bits per level was
  // host time the device waited for)
  struct JumpPositions {
    std::vector<uint16_t> pos;
    int cnt = 0;
  };
  static std::mutex jp_mu;
  static std::map<int, JumpPositions> jp_cache;
  for (int a = 0; a < levels; ++a) {
    const JumpPositions* jp = nullptr;
    {
      std::lock_guard<std::mutex> lk(jp_mu);
      auto it = jp_cache.find(k + a);
      if (it == jp_cache.end()) {
        std::vector<uint64_t> poly(mt::kPolyWords);
        if (!mt::jump_poly_pow2(k + a, poly.data())) return cudaErrorUnknown;
        JumpPositions j;
        for (int i = 0; i < mt::kDegree; ++i)
          if ((poly[i >> 6] >> (i & 63)) & 1ULL) j.pos.push_back(static_cast<uint16_t>(i));
        j.cnt = static_cast<int>(j.pos.size());
        it = jp_cache.emplace(k + a, std::move(j)).first;
      }
      jp = &it->second;  // map nodes are stable
    }
    std::copy(jp->pos.begin(), jp->pos.end(), hpos.begin() + static_cast<size_t>(a) * kPosCap);
    npos8[a] = (jp->cnt + 7) / 8;  // tail slots keep the zero-window sentinel
  }
  EQ_CUDA_TRY(cudaMemcpyAsync(windows, seedw.data(), mt::kN * sizeof(uint64_t),
                              cudaMemcpyHostToDevice, s));
  if (levels > 0)
    EQ_CUDA_TRY(cudaMemcpyAsync(pos, hpos.data(), hpos.size() * sizeof(uint16_t),
                                cudaMemcpyHostToDevice, s));
  const size_t smem = (kJumpWords + mt::kN + kJumpGroups * mt::kN) * sizeof(uint64_t);
  // the attribute belongs to the device context: set it once per device
  static std::atomic<unsigned long long> attr_done{0};
  int dev = 0;
  EQ_CUDA_TRY(cudaGetDevice(&dev));
  const unsigned long long bit = 1ULL << (dev & 63);
  if (!(attr_done.load() & bit)) {
    EQ_CUDA_TRY(cudaFuncSetAttribute(mt_jump_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    attr_done.fetch_or(bit);
  }
  for (int a = 0; a < levels; ++a) {
    const uint64_t lo = 1ULL << a;
    const uint64_t cnt = std::min(lo, G - lo);
    mt_jump_kernel<<<static_cast<unsigned>(cnt), kMtThreads * kJumpGroups, smem, s>>>(
        windows, 0, static_cast<int>(lo),
        reinterpret_cast<const uint4*>(pos + static_cast<size_t>(a) * kPosCap), npos8[a]);
    count_launch(s);
    EQ_CUDA_TRY(cudaGetLastError());
  }
  mt_gen_kernel<<<static_cast<unsigned>(G), kMtThreads, 0, s>>>(windows, L, total,
                                                                bits); count_launch(s);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Input validation (ExplicitMatrix::sparse's preconditions, explicit_matrix.cpp:21-39,
// restated for canonical CSR input: rows ascending, columns strictly ascending)
// ---------------------------------------------------------------------------
namespace {
// (row_ptr itself is validated on the host before upload, so these reads
// stay inside the arrays.)  One warp per row, coalesced.  The reported error is deterministic and follows
// the reference's order of checks: the first out-of-range entry
// (explicit_matrix.cpp:23-28) before the first duplicate (:33-39); a column
// order violation (only possible for non-canonical CSR) ranks last.  `where`
// receives min over (class << 40 | entry index).
__global__ void validate_cols_kernel(const int64_t* rp, const int32_t* ci,
                                     int64_t rows, int64_t cols, int* err,
                                     unsigned long long* where) {
  const int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= rows) return;
  const int64_t k0 = rp[i], k1 = rp[i + 1];
  unsigned long long best = ~0ULL;
  for (int64_t k = k0 + lane; k < k1; k += 32) {
    const int32_t c = __ldg(ci + k);
    unsigned long long key = ~0ULL;
    if (c < 0 || c >= cols) {
      key = static_cast<unsigned long long>(k);
    } else if (k > k0) {
      const int32_t p = __ldg(ci + k - 1);
      if (p == c) key = (1ULL << 40) | static_cast<unsigned long long>(k);
      else if (p > c && p >= 0 && p < cols) key = (2ULL << 40) | static_cast<unsigned long long>(k);
    }
    best = key < best ? key : best;
  }
  for (int h = 16; h >= 1; h >>= 1) {
    const unsigned long long o = __shfl_down_sync(0xffffffffu, best, h);
    best = o < best ? o : best;
  }
  if (lane == 0 && best != ~0ULL) {
    atomicMin(where, best);
    *err = 1;
  }
}
}  // namespace

cudaError_t launch_validate_csr(const DevCsr& A, int* err, unsigned long long* where,
                                cudaStream_t s) {
  if (A.rows == 0) return cudaSuccess;
  const int bs = 256;  // 8 rows per CTA
  validate_cols_kernel<<<static_cast<unsigned>((A.rows * 32 + bs - 1) / bs), bs, 0, s>>>(
      A.row_ptr, A.col, A.rows, A.cols, err, where);
  count_launch(s);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Device flag barrier across the ranks of a fused all-gather (one CTA).  Stream
// order puts it after this rank's SGD kernels, whose threads fenced their peer
// stores system-wide (__threadfence_system) before exiting.  Each rank bumps its
// epoch, release-stores it into flag[rank] of every peer, and acquire-spins
// until every other rank's flag in its own array has reached the epoch; the
// kernels after it (a new launch: L1 starts empty) then read the peers' stores.
// A wait longer than ~6 s gives up and sets the error word (checked on the host
// after the loop) instead of hanging.
// ---------------------------------------------------------------------------
namespace {
struct PeerDeltas {
  int64_t d[EQ_MAX_PEERS];
};
__global__ void peer_barrier_kernel(unsigned long long* bar, int rank, int world,
                                    PeerDeltas pd, int npeer) {
  __shared__ unsigned long long ep;
  if (threadIdx.x == 0) {
    ep = bar[kBarEpoch] + 1;
    bar[kBarEpoch] = ep;
  }
  __syncthreads();
  const unsigned long long e = ep;
  if (static_cast<int>(threadIdx.x) < npeer) {
    unsigned long long* dst = bar + rank + pd.d[threadIdx.x];
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst), "l"(e) : "memory");
  }
  if (static_cast<int>(threadIdx.x) < world && static_cast<int>(threadIdx.x) != rank) {
    unsigned long long v = 0;
    for (long long spin = 0; spin < (1LL << 26); ++spin) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(bar + threadIdx.x) : "memory");
      if (v >= e) break;
      __nanosleep(100);
    }
    if (v < e) atomicExch(bar + kBarError, 1ULL);
  }
  __syncthreads();
}
}  // namespace

cudaError_t launch_peer_barrier(unsigned long long* bar, int rank, int world,
                                const int64_t* peer_delta, int npeer, cudaStream_t s) {
  if (npeer > EQ_MAX_PEERS || world > kBarEpoch) return cudaErrorInvalidValue;
  PeerDeltas pd{};
  for (int g = 0; g < npeer; ++g) pd.d[g] = peer_delta[g];
  peer_barrier_kernel<<<1, 32, 0, s>>>(bar, rank, world, pd, npeer);
  count_launch(s);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Host -> device copy pulled by the SMs from mapped pinned memory: during
// matrix setup the copy engine is busy with A's values, and a small plan
// upload queued behind them would wait for the whole transfer.
// ---------------------------------------------------------------------------
namespace {
__global__ void pull_copy_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                 int64_t n16, unsigned char* __restrict__ dtail,
                                 const unsigned char* __restrict__ stail, int tail) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  for (int64_t k = t0; k < n16; k += stride) dst[k] = src[k];
  if (t0 < tail) dtail[t0] = stail[t0];
}
}  // namespace

cudaError_t launch_pull_copy(void* dst, const void* src_mapped, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return cudaSuccess;
  // both 16-byte aligned (pool / arena allocations)
  const int64_t n16 = static_cast<int64_t>(bytes / 16);
  const int tail = static_cast<int>(bytes % 16);
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n16 + 255) / 256, 1184));
  pull_copy_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(
      static_cast<uint4*>(dst), static_cast<const uint4*>(src_mapped), n16,
      static_cast<unsigned char*>(dst) + n16 * 16,
      static_cast<const unsigned char*>(src_mapped) + n16 * 16, tail);
  count_launch(s);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// COO ingest = ExplicitMatrix::sparse (src/explicit_matrix.cpp:19-57) on device:
// range check in input order (:21-28), sort by (row, col) (:28-31), duplicate
// rejection in sorted order (:32-39), CSR by counting (:41-56).
// ---------------------------------------------------------------------------
namespace {
__global__ void coo_range_kernel(const int64_t* __restrict__ r, const int64_t* __restrict__ c,
                                 int64_t nnz, int64_t m, int64_t n,
                                 unsigned long long* first_bad, uint64_t* key,
                                 int32_t* perm) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= nnz) return;
  const int64_t i = r[k], j = c[k];
  const bool ok = i >= 0 && i < m && j >= 0 && j < n;
  if (!ok) atomicMin(first_bad, static_cast<unsigned long long>(k));
  key[k] = ok ? static_cast<uint64_t>(i) * static_cast<uint64_t>(n) + static_cast<uint64_t>(j) : 0;
  perm[k] = static_cast<int32_t>(k);
}
__global__ void coo_build_kernel(const uint64_t* __restrict__ skey,
                                 const int32_t* __restrict__ sperm,
                                 const double* __restrict__ v, int64_t nnz, int64_t n,
                                 unsigned long long* first_dup, int32_t* __restrict__ col,
                                 double* __restrict__ val) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= nnz) return;
  const uint64_t key = skey[p];
  if (p > 0 && skey[p - 1] == key) atomicMin(first_dup, static_cast<unsigned long long>(p));
  col[p] = static_cast<int32_t>(key % static_cast<uint64_t>(n));
  val[p] = v[sperm[p]];
}
__global__ void coo_rowptr_kernel(const uint64_t* __restrict__ skey, int64_t nnz, int64_t n,
                                  int64_t m, int64_t* __restrict__ rp) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p > nnz) return;
  const int64_t prev = p == 0 ? -1 : static_cast<int64_t>(skey[p - 1] / static_cast<uint64_t>(n));
  const int64_t cur = p == nnz ? m : static_cast<int64_t>(skey[p] / static_cast<uint64_t>(n));
  for (int64_t i = prev + 1; i <= cur && i <= m; ++i) rp[i] = p;
}
}  // namespace

cudaError_t coo_to_csr(int64_t m, int64_t n, int64_t nnz, const int64_t* rows,
                       const int64_t* cols, const double* vals, DevCsr& out,
                       unsigned long long* bad, int* bad_kind, cudaStream_t s) {
  *bad_kind = 0;
  uint64_t *key = nullptr, *skey = nullptr;
  int32_t *perm = nullptr, *sperm = nullptr;
  unsigned long long* flags = nullptr;
  void* temp = nullptr;
  size_t temp_bytes = 0;
  const int end_bit = std::max(1, ceil_log2(static_cast<uint64_t>(m) * static_cast<uint64_t>(n)));
  const unsigned nb = static_cast<unsigned>((nnz + 255) / 256);
  cudaError_t e = cudaSuccess;
  unsigned long long h[2] = {~0ULL, ~0ULL};
  do {
    e = cudaMallocAsync(&flags, 2 * sizeof(unsigned long long), s); if (e) break;
    e = cudaMemsetAsync(flags, 0xff, 2 * sizeof(unsigned long long), s); if (e) break;
    if (nnz > 0) {
      e = cudaMallocAsync(&key, nnz * 8, s); if (e) break;
      e = cudaMallocAsync(&skey, nnz * 8, s); if (e) break;
      e = cudaMallocAsync(&perm, nnz * 4, s); if (e) break;
      e = cudaMallocAsync(&sperm, nnz * 4, s); if (e) break;
      coo_range_kernel<<<nb, 256, 0, s>>>(rows, cols, nnz, m, n, flags, key, perm);
      count_launch(s);
      e = cudaMemcpyAsync(h, flags, 8, cudaMemcpyDeviceToHost, s); if (e) break;
      e = cudaStreamSynchronize(s); if (e) break;
      if (h[0] != ~0ULL) {  // first out-of-range entry in input order
        *bad = h[0];
        *bad_kind = 1;
        break;
      }
      e = cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, key, skey, perm, sperm, nnz, 0,
                                          end_bit, s);
      if (e) break;
      e = cudaMallocAsync(&temp, temp_bytes, s); if (e) break;
      e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, key, skey, perm, sperm, nnz, 0,
                                          end_bit, s);
      if (e) break;
      coo_build_kernel<<<nb, 256, 0, s>>>(skey, sperm, vals, nnz, n, flags + 1, out.col,
                                          out.val);
      count_launch(s);
    }
    coo_rowptr_kernel<<<static_cast<unsigned>((nnz + 1 + 255) / 256), 256, 0, s>>>(
        skey, nnz, n, m, out.row_ptr);
    count_launch(s);
    e = cudaMemcpyAsync(h + 1, flags + 1, 8, cudaMemcpyDeviceToHost, s); if (e) break;
    e = cudaStreamSynchronize(s); if (e) break;
    if (h[1] != ~0ULL) {  // first duplicate in sorted order: report its key
      uint64_t dk = 0;
      e = cudaMemcpy(&dk, skey + h[1], 8, cudaMemcpyDeviceToHost); if (e) break;
      *bad = dk;
      *bad_kind = 2;
    }
  } while (0);
  if (temp) cudaFreeAsync(temp, s);
  if (key) cudaFreeAsync(key, s);
  if (skey) cudaFreeAsync(skey, s);
  if (perm) cudaFreeAsync(perm, s);
  if (sperm) cudaFreeAsync(sperm, s);
  if (flags) cudaFreeAsync(flags, s);
  return e;
}

// ---------------------------------------------------------------------------
// K3/K4: the fused SGD iteration over CSR(A) and CSR(A^T)
// ---------------------------------------------------------------------------
namespace {

// kind 2 (run_tile): one warp runs one slice; warps never wait on each other,
// so on an SM the memory-bound staging of some warps overlaps the
// latency-bound sequential chains of others.
//
// kind 3 (run_long_slice) is CTA-cooperative: the 4 warps of a CTA own the same
// "long slice" of up to 32 rows longer than kTileNnz (length-sorted).  Each
// round all 128 threads stage the next kLongChunk products of every active row
// (coalesced, aligned chunks) into a padded [32][kLongStride] buffer, then warp
// 0's 32 lanes each extend one row's sequential sum with conflict-free 16-byte
// reads -- 32 chains in parallel instead of one lane-0 chain per warp.
// NV = 2 (LSQR's fused pass): a second gathered vector xg2 rides along; its
// products go to a second staging buffer and a second sequential chain.
template <class Epi, int NV = 1>
__device__ __forceinline__ void run_long_slice(const Tile& t, const int64_t* __restrict__ rp,
                                               const int32_t* __restrict__ ci,
                                               const double* __restrict__ va,
                                               const double* __restrict__ xg,
                                               const int32_t* __restrict__ rowlist,
                                               double* sp, SliceMeta& sm, Epi& epi,
                                               const double* __restrict__ xg2 = nullptr) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cnt = t.r1;
  int myrow = -1, mk0 = 0, mlen = 0, rounds = 0;
  double acc0 = 0.0;  // running sum carried in (column-block rounds)
  if (warp == 0) {
    myrow = lane < cnt ? rowlist[t.r0 + lane] : -1;
    int64_t k0 = 0, k1 = 0;
    if (myrow >= 0) epi.span(rp, myrow, k0, k1, acc0);
    const int64_t kb = k0 & ~static_cast<int64_t>(kLongChunk - 1);
    rounds = k1 > k0 ? static_cast<int>((k1 - kb + kLongChunk - 1) / kLongChunk) : 0;
    mk0 = static_cast<int>(k0 - kb);
    mlen = static_cast<int>(k1 - kb);
    sm.r[lane] = RowMeta{kb, mk0, mlen};
    const int maxr = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(rounds)));
    if (lane == 0) sm.maxr = maxr;
  }
  __syncthreads();
  const int maxr = sm.maxr;
  double acc = acc0, acc2 = 0.0;
  double* sp2 = sp + 32 * kLongStride;  // NV == 2 only
  for (int b = 0; b < maxr; ++b) {
    const int off = b * kLongChunk;
    // warp w stages rows w, w+4, ... : kLongChunk / 32 products per lane per row
    constexpr int kPer = kLongChunk / 32;
#pragma unroll 1
    for (int q0 = warp; q0 < cnt; q0 += 4 * kLongBatch) {
      int32_t c[kPer * kLongBatch];
      double v[kPer * kLongBatch];
      bool ok[kPer * kLongBatch];
#pragma unroll
      for (int u = 0; u < kLongBatch; ++u) {
        const int q = q0 + 4 * u;
        RowMeta rm{0, 1, 0};
        if (q < cnt) rm = sm.r[q];
#pragma unroll
        for (int h = 0; h < kPer; ++h) {
          const int rel = off + lane + 32 * h;
          const int i = kPer * u + h;
          ok[i] = rel >= rm.k0 && rel < rm.len;
          if (ok[i]) {
            c[i] = ld_na(ci + rm.start + rel);
            v[i] = ld_na(va + rm.start + rel);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kLongBatch; ++u)
#pragma unroll
        for (int h = 0; h < kPer; ++h)
          if (ok[kPer * u + h]) {
            const int at = (q0 + 4 * u) * kLongStride + lane + 32 * h;
            sp[at] = __dmul_rn(v[kPer * u + h], __ldg(xg + c[kPer * u + h]));
            if constexpr (NV == 2) sp2[at] = __dmul_rn(v[kPer * u + h], __ldg(xg2 + c[kPer * u + h]));
          }
    }
    __syncthreads();
    if (warp == 0 && rounds > b) {
      acc = chain_sum(acc, sp + lane * kLongStride, max(0, mk0 - off),
                      min(kLongChunk, mlen - off));
      if constexpr (NV == 2)
        acc2 = chain_sum(acc2, sp2 + lane * kLongStride, max(0, mk0 - off),
                         min(kLongChunk, mlen - off));
    }
    __syncthreads();
  }
  if (warp == 0 && myrow >= 0) {
    if constexpr (NV == 2) epi(myrow, acc, acc2);
    else epi(myrow, acc);
  }
}

template <class Epi, int NV = 1>
__device__ __forceinline__ void run_tile(const Tile& t, const int64_t* __restrict__ rp,
                                         const int32_t* __restrict__ ci,
                                         const double* __restrict__ va,
                                         const double* __restrict__ xg,
                                         const int32_t* __restrict__ rowlist, double* sp,
                                         SliceMeta& sm, int lane, Epi& epi,
                                         const double* __restrict__ xg2 = nullptr) {
  {
    // Slice: up to 32 rows (sorted by length, longest first), one per lane, in
    // lock-step rounds of kSliceChunk products per row.  Each round the warp
    // stages the rows' next chunks with coalesced half-warp loads into a padded
    // [row][kSliceStride] buffer (conflict-free 16B reads), then every lane
    // extends its own row's sequential sum.
    // Chunks are aligned to kSliceChunk elements in absolute CSR position, so a
    // 128-byte line of values / 64 bytes of columns is fetched once per row
    // (the first and last chunk of a row are partial).
    const int cnt = t.r1;
    const int myrow = lane < cnt ? rowlist[t.r0 + lane] : -1;
    int64_t k0 = 0, k1 = 0;
    double acc0 = 0.0;
    if (myrow >= 0) epi.span(rp, myrow, k0, k1, acc0);
    const int64_t kb = k0 & ~static_cast<int64_t>(kSliceChunk - 1);
    const int rounds = k1 > k0 ? static_cast<int>((k1 - kb + kSliceChunk - 1) / kSliceChunk) : 0;
    const int mk0 = static_cast<int>(k0 - kb), mlen = static_cast<int>(k1 - kb);
    sm.r[lane] = RowMeta{kb, mk0, mlen};
    const int maxr = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(rounds)));
    __syncwarp();
    const int half = lane >> 4, e = lane & 15;
    double acc = acc0, acc2 = 0.0;
    double* sp2 = sp + 32 * kSliceStride;  // NV == 2 only
    for (int b = 0; b < maxr; ++b) {
      const int off = b * kSliceChunk;
#if EQ_SLICE_PREFETCH
      // pull this lane's row chunk EQ_SLICE_PREFETCH rounds ahead into L2, so the
      // column-index loads of later rounds (which the gathers depend on) do not
      // wait on DRAM
      if (rounds > b + EQ_SLICE_PREFETCH) {
        const int64_t nx = kb + off + EQ_SLICE_PREFETCH * kSliceChunk;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(ci + nx));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(va + nx));
      }
#endif
      // rows still active this round (rows are length-sorted, so nearly a prefix)
      const int act = 32 - __clz(__ballot_sync(0xffffffffu, rounds > b));
      for (int q0 = 0; q0 < act; q0 += 2 * kSliceBatch) {
        int32_t c[kSliceBatch];
        double v[kSliceBatch];
        bool ok[kSliceBatch];
#pragma unroll
        for (int u = 0; u < kSliceBatch; ++u) {
          const int q = q0 + 2 * u + half;
          const int rel = off + e;  // position relative to the row's aligned base
          RowMeta rm{0, 1, 0};
          if (q < act) rm = sm.r[q];  // one 16-byte shared load per row chunk
          ok[u] = rel >= rm.k0 && rel < rm.len;
          if (ok[u]) {
            const int64_t k = rm.start + rel;
            c[u] = ld_na(ci + k);
            v[u] = ld_na(va + k);
          }
        }
#pragma unroll
        for (int u = 0; u < kSliceBatch; ++u) {
          const int q = q0 + 2 * u + half;
          if (ok[u]) {
            sp[q * kSliceStride + e] = __dmul_rn(v[u], __ldg(xg + c[u]));
            if constexpr (NV == 2) sp2[q * kSliceStride + e] = __dmul_rn(v[u], __ldg(xg2 + c[u]));
          }
        }
      }
      __syncwarp();
      if (rounds > b) {
        const int lo = max(0, mk0 - off);
        const int hi = min(kSliceChunk, mlen - off);
        acc = chain_sum(acc, sp + lane * kSliceStride, lo, hi);
        if constexpr (NV == 2) acc2 = chain_sum(acc2, sp2 + lane * kSliceStride, lo, hi);
      }
      __syncwarp();
    }
    if (myrow >= 0) {
      if constexpr (NV == 2) epi(myrow, acc, acc2);
      else epi(myrow, acc);
    }
  }
}

// With column blocks (nblk > 1) a row's entries are visited block by block in
// separate launches (rounds); the running sum waits in `carry` between them and
// the epilogue runs in the last round.  Blocks are contiguous column ranges and
// columns ascend within a row, so every row is still summed in CSR order.
struct SgdEpi {
  const SgdIterArgs& a;
  int mat;
  unsigned fl;
  __device__ void span(const int64_t* rp, int64_t r, int64_t& k0, int64_t& k1,
                       double& acc0) const {
    const int nb = a.nblk[mat];
    k0 = rp[r];
    k1 = rp[r + 1];
    acc0 = 0.0;
    if (nb <= 1) return;
    const int32_t* bb = a.bnd[mat] + r * (nb - 1);
    const int64_t base = k0;
    if (a.round > 0) {
      k0 = base + bb[a.round - 1];
      acc0 = a.carry[mat][r];
    }
    if (a.round < nb - 1) k1 = base + bb[a.round];
  }
  __device__ void operator()(int64_t r, double acc) {
    if (a.round < a.nblk[mat] - 1) {
      a.carry[mat][r] = acc;
      return;
    }
    sgd_epilogue(a, mat, r, acc, fl);
  }
};

// KINDS: bit 0 = warp slices (kind 2), bit 1 = CTA long slices (kind 3);
// tile_base offsets into the tile list (for launches over a sub-range).
template <int MINB, int KINDS>
__global__ void __launch_bounds__(kTileThreads, MINB)
sgd_iter_kernel(const SgdIterArgs a, int tile_base, int ntiles) {
  __shared__ __align__(16) double sp[kTileWarps][kWarpSmem];
  __shared__ SliceMeta sm[kTileWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tid = blockIdx.x * kTileWarps + warp;
  if (tid >= ntiles) return;
  const Tile t = a.tiles[tile_base + tid];
  const int mat = t.mat;
  if (a.round >= a.nblk[mat]) return;  // this matrix has fewer column blocks
  SgdEpi epi{a, mat, 0u};
  if ((KINDS & 2) && t.kind == 3)  // CTA-cooperative (all 4 warps hold this tile)
    run_long_slice<SgdEpi, 1>(t, a.rp[mat], a.ci[mat], a.va[mat], mat ? a.xw_cur : a.xs_cur,
                              a.rl[mat], &sp[0][0], sm[0], epi);
  else if (KINDS & 1)
    run_tile<SgdEpi, 1>(t, a.rp[mat], a.ci[mat], a.va[mat], mat ? a.xw_cur : a.xs_cur,
                        a.rl[mat], sp[warp], sm[warp], lane, epi);
  // peer stores performed system-wide before the kernel completes (the
  // barrier that follows orders every peer's next reads after them)
  if (a.npeer) __threadfence_system();
  if (epi.fl) atomicOr(a.flags, epi.fl);
}

__global__ void sgd_init_kernel(double* xs, double* xw, double* u, double* ub,
                                double* v, double* vb, const uint32_t* signs,
                                int64_t m_loc, int64_t n_loc, int64_t a_goff,
                                int64_t at_goff, int64_t a_poff, int64_t at_poff,
                                int64_t n_glob, const int32_t* wslot, const int32_t* sslot) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < m_loc) {  // d = exp(0) = 1: xw = w (iteration 1: outputs n + i)
    u[k] = 0.0;
    ub[k] = 0.0;
    xw[wslot ? wslot[k] : a_poff + k] = sign_bit(signs, n_glob + a_goff + k) ? 1.0 : -1.0;
  }
  if (k < n_loc) {  // e = 1: xs = s (outputs j)
    v[k] = 0.0;
    vb[k] = 0.0;
    xs[sslot ? sslot[k] : at_poff + k] = sign_bit(signs, at_goff + k) ? 1.0 : -1.0;
  }
}

__global__ void remap_cols_by_map_kernel(int32_t* __restrict__ dst, const int32_t* __restrict__ src,
                                         const int32_t* __restrict__ map, int64_t nnz) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < nnz) dst[k] = map[src[k]];
}

__global__ void exp_kernel(const double* __restrict__ x, double* __restrict__ y,
                           int64_t n, double scale) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < n) y[k] = det_exp(scale == 1.0 ? x[k] : __dmul_rn(scale, x[k]));
}

}  // namespace

cudaError_t launch_sgd_init(double* xs, double* xw, double* u, double* ub,
                            double* v, double* vb, int64_t, int64_t,
                            const uint32_t* signs, int64_t m_loc, int64_t n_loc,
                            int64_t a_goff, int64_t at_goff, int64_t a_poff,
                            int64_t at_poff, int64_t, int64_t n_glob, const int32_t* wslot,
                            const int32_t* sslot, cudaStream_t s) {
  const int64_t nmax = std::max(m_loc, n_loc);
  if (nmax == 0) return cudaSuccess;
  sgd_init_kernel<<<static_cast<unsigned>((nmax + 255) / 256), 256, 0, s>>>(
      xs, xw, u, ub, v, vb, signs, m_loc, n_loc, a_goff, at_goff, a_poff, at_poff,
      n_glob, wslot, sslot); count_launch(s);
  return cudaGetLastError();
}

namespace {
// key of row i of rank g: g * 128 + (len == 0 ? 64 : clz(len)) -> longest rows first
__global__ void slot_keys_kernel(const int64_t* __restrict__ rp, int64_t rows,
                                 const int64_t* __restrict__ bounds, int G,
                                 uint32_t* __restrict__ key, int32_t* __restrict__ idx, int flat) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= rows) return;
  int g = 0;
  while (g + 1 < G && bounds[g + 1] <= i) ++g;
  const int64_t len = rp[i + 1] - rp[i];
  // flat: every row of a rank gets the same key, so the (stable) sort keeps
  // the row order and the slot map is the identity
  key[i] = static_cast<uint32_t>(g) * 128u +
           (flat || len <= 0 ? 64u : static_cast<uint32_t>(__clzll(static_cast<long long>(len))));
  idx[i] = static_cast<int32_t>(i);
}
// sorted position s holds row perm[s]: map[pad(perm[s])] = g * maxcnt + (s - bounds[g])
__global__ void slot_map_kernel(const int32_t* __restrict__ perm, int64_t rows,
                                const int64_t* __restrict__ bounds, int G, int64_t maxcnt,
                                int32_t* __restrict__ map_pad) {
  const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (s >= rows) return;
  const int64_t i = perm[s];
  int g = 0;
  while (g + 1 < G && bounds[g + 1] <= i) ++g;  // rank of row i == rank of position s
  const int64_t base = G == 1 ? 0 : g * maxcnt;
  map_pad[base + (i - bounds[g])] = static_cast<int32_t>(base + (s - bounds[g]));
}
}  // namespace

cudaError_t launch_slot_map(const int64_t* rp, int64_t rows, const int64_t* bounds, int G,
                            int64_t maxcnt, int32_t* map_pad, cudaStream_t s, bool flat) {
  if (rows == 0) return cudaSuccess;
  uint32_t *k0 = nullptr, *k1 = nullptr;
  int32_t *i0 = nullptr, *i1 = nullptr;
  void* temp = nullptr;
  size_t tb = 0;
  int bits = 7;
  while ((1 << (bits - 7)) < G) ++bits;
  cudaError_t e = cudaSuccess;
  do {
    e = cudaMallocAsync(&k0, rows * 4, s); if (e) break;
    e = cudaMallocAsync(&k1, rows * 4, s); if (e) break;
    e = cudaMallocAsync(&i0, rows * 4, s); if (e) break;
    e = cudaMallocAsync(&i1, rows * 4, s); if (e) break;
    const unsigned grid = static_cast<unsigned>((rows + 255) / 256);
    slot_keys_kernel<<<grid, 256, 0, s>>>(rp, rows, bounds, G, k0, i0, flat ? 1 : 0);
    count_launch(s);
    e = cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, i0, i1, rows, 0, bits, s);
    if (e) break;
    e = cudaMallocAsync(&temp, tb, s); if (e) break;
    e = cub::DeviceRadixSort::SortPairs(temp, tb, k0, k1, i0, i1, rows, 0, bits, s);  // stable
    if (e) break;
    slot_map_kernel<<<grid, 256, 0, s>>>(i1, rows, bounds, G, maxcnt, map_pad);
    count_launch(s);
    e = cudaGetLastError();
  } while (0);
  for (void* q : {static_cast<void*>(k0), static_cast<void*>(k1), static_cast<void*>(i0),
                  static_cast<void*>(i1), temp})
    if (q) cudaFreeAsync(q, s);
  return e;
}

cudaError_t launch_remap_cols(int32_t* dst, const int32_t* src, const int32_t* map, int64_t nnz,
                              cudaStream_t s) {
  if (nnz == 0) return cudaSuccess;
  remap_cols_by_map_kernel<<<static_cast<unsigned>((nnz + 255) / 256), 256, 0, s>>>(dst, src, map,
                                                                                   nnz);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_sgd_iter(const SgdIterArgs& a, int ntiles, cudaStream_t s) {
  if (ntiles == 0) return cudaSuccess;
  const unsigned g = static_cast<unsigned>((ntiles + kTileWarps - 1) / kTileWarps);
  sgd_iter_kernel<kTileMinBlocks, 3><<<g, kTileThreads, 0, s>>>(a, 0, ntiles);
  count_launch(s);
  return cudaGetLastError();
}

// tiles [tile_base, tile_base + ntiles) of one kind class (long: kind-3 CTA
// groups, else warp tiles) -- for launching the two classes on separate streams
cudaError_t launch_sgd_iter_part(const SgdIterArgs& a, int tile_base, int ntiles, bool long_part,
                                 int minb, cudaStream_t s) {
  if (ntiles <= 0) return cudaSuccess;
  const unsigned g = static_cast<unsigned>((ntiles + kTileWarps - 1) / kTileWarps);
  if (long_part) {
    if (minb >= 8) sgd_iter_kernel<8, 2><<<g, kTileThreads, 0, s>>>(a, tile_base, ntiles);
    else sgd_iter_kernel<6, 2><<<g, kTileThreads, 0, s>>>(a, tile_base, ntiles);
  } else {
    if (minb >= 8) sgd_iter_kernel<8, 1><<<g, kTileThreads, 0, s>>>(a, tile_base, ntiles);
    else sgd_iter_kernel<6, 1><<<g, kTileThreads, 0, s>>>(a, tile_base, ntiles);
  }
  count_launch(s);
  return cudaGetLastError();
}

namespace {
// per row: the nb - 1 interior column-block boundaries as offsets into the row
// (first entry with column >= b * width), columns ascending within rows
__global__ void block_bounds_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                    int64_t rows, int nb, int64_t width,
                                    int32_t* __restrict__ bnd) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  const int64_t k0 = rp[r], k1 = rp[r + 1];
  for (int b = 1; b < nb; ++b) {
    const int64_t key = b * width;
    int64_t lo = k0, hi = k1;  // lower bound of key in ci[k0, k1)
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ci[mid] < key) lo = mid + 1; else hi = mid;
    }
    bnd[r * (nb - 1) + (b - 1)] = static_cast<int32_t>(lo - k0);
  }
}
}  // namespace

cudaError_t launch_block_bounds(const DevCsr& M, int nb, int64_t width, int32_t* bnd,
                                cudaStream_t s) {
  if (M.rows == 0 || nb <= 1) return cudaSuccess;
  block_bounds_kernel<<<static_cast<unsigned>((M.rows + 255) / 256), 256, 0, s>>>(
      M.row_ptr, M.col, M.rows, nb, width, bnd);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_exp(const double* x, double* y, int64_t n, double scale,
                       cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  exp_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(x, y, n, scale); count_launch(s);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Generic single-matrix pass (LSQR, plain apply): same traversal, other epilogues
// ---------------------------------------------------------------------------
namespace {

__device__ __forceinline__ void full_row(const int64_t* rp, int64_t r, int64_t& k0, int64_t& k1,
                                         double& acc0) {
  k0 = rp[r];
  k1 = rp[r + 1];
  acc0 = 0.0;
}
struct PassEpi {
  const PassArgs& a;
  __device__ void span(const int64_t* rp, int64_t r, int64_t& k0, int64_t& k1,
                       double& acc0) const {
    full_row(rp, r, k0, k1, acc0);
  }
  __device__ void operator()(int64_t r, double acc) { pass_epilogue(a, r, acc); }
};
struct PassEpi2 {
  const PassArgs& a;
  const PassArgs& b;
  __device__ void span(const int64_t* rp, int64_t r, int64_t& k0, int64_t& k1,
                       double& acc0) const {
    full_row(rp, r, k0, k1, acc0);
  }
  __device__ void operator()(int64_t r, double acc, double acc2) {
    pass_epilogue(a, r, acc);
    pass_epilogue(b, r, acc2);
  }
};

// NV = 2: two passes over the same matrix in one traversal (shared value and
// column streams, two gathers per entry, two sequential sums per row)
template <int NV>
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks)
pass_kernel(const PassArgs a, const PassArgs b, int tile_base, int ntiles) {
  constexpr int kWarpDoubles = NV == 2 ? 2 * 32 * kSliceStride : kWarpSmem;
  static_assert(NV == 1 || 2 * 32 * kLongStride <= kTileWarps * kWarpDoubles, "long staging");
  __shared__ __align__(16) double sp[kTileWarps][kWarpDoubles];
  __shared__ SliceMeta sm[kTileWarps];
  if (a.skip && *a.skip) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tid = blockIdx.x * kTileWarps + warp;
  if (tid >= ntiles) return;
  const Tile t = a.tiles[tile_base + tid];
  if constexpr (NV == 1) {
    PassEpi epi{a};
    if (t.kind == 3)
      run_long_slice<PassEpi, 1>(t, a.rp, a.ci, a.va, a.xg, a.rl, &sp[0][0], sm[0], epi);
    else
      run_tile<PassEpi, 1>(t, a.rp, a.ci, a.va, a.xg, a.rl, &sp[warp][0], sm[warp], lane, epi);
  } else {
    PassEpi2 epi{a, b};
    if (t.kind == 3)
      run_long_slice<PassEpi2, 2>(t, a.rp, a.ci, a.va, a.xg, a.rl, &sp[0][0], sm[0], epi, b.xg);
    else
      run_tile<PassEpi2, 2>(t, a.rp, a.ci, a.va, a.xg, a.rl, &sp[warp][0], sm[warp], lane, epi,
                            b.xg);
  }
}

}  // namespace

cudaError_t launch_pass_range(const PassArgs& a, const PassArgs* b, int tile_base, int ntiles,
                              cudaStream_t s) {
  if (ntiles <= 0) return cudaSuccess;
  const unsigned g = static_cast<unsigned>((ntiles + kTileWarps - 1) / kTileWarps);
  if (b)
    pass_kernel<2><<<g, kTileThreads, 0, s>>>(a, *b, tile_base, ntiles);
  else
    pass_kernel<1><<<g, kTileThreads, 0, s>>>(a, a, tile_base, ntiles);
  count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_pass(const PassArgs& a, int ntiles, cudaStream_t s) {
  return launch_pass_range(a, nullptr, 0, ntiles, s);
}

cudaError_t launch_pass_dual(const PassArgs& a, const PassArgs& b, int ntiles, cudaStream_t s) {
  return launch_pass_range(a, &b, 0, ntiles, s);
}

// ---------------------------------------------------------------------------
// Canonical reduction (det_math.cuh): level 1 per 2048-chunk, level 2 by the
// last CTA to finish (fixed-order read of all chunk partials).
// ---------------------------------------------------------------------------
namespace {

// fold s[0..lanes) in place, lanes power of two, blockDim.x == 256
__device__ double block_fold(double* s, int lanes) {
  for (int h = lanes / 2; h >= 1; h >>= 1) {
    for (int l = threadIdx.x; l < h; l += blockDim.x) s[l] = __dadd_rn(s[l], s[l + h]);
    __syncthreads();
  }
  return s[0];
}

__global__ void __launch_bounds__(256)
canon_reduce_kernel(const double* __restrict__ x, int64_t len, int kind, double coef,
                    double* __restrict__ part, unsigned* counter,
                    double* __restrict__ out, int sqrt_out, int64_t part_cap) {
  __shared__ double s[kLanes2];
  EQ_CHECK(part_cap < 0 || static_cast<int64_t>(blockIdx.x) < part_cap);
  __shared__ bool last;
  const int64_t nc = (len + kChunk - 1) / kChunk;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kChunk;
  const int64_t clen = imin64(kChunk, len - base);
  const int l = threadIdx.x;
  double acc = 0.0;
  for (int64_t k = l; k < clen; k += kLanes1) {
    const double v = x[base + k];
    const double term = kind == 0 ? __dmul_rn(v, v) : (kind == 1 ? v : __dmul_rn(coef, v));
    acc = __dadd_rn(acc, term);
  }
  s[l] = acc;
  __syncthreads();
  const double p = block_fold(s, kLanes1);
  if (l == 0) {
    part[blockIdx.x] = p;
    __threadfence();
    // (an empty input still runs one CTA, which must finish the reduction)
    last = (atomicAdd(counter, 1u) == static_cast<unsigned>((nc > 0 ? nc : 1) - 1));
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int q = l; q < kLanes2; q += blockDim.x) {
    double a2 = 0.0;
    for (int64_t k = q; k < nc; k += kLanes2) a2 = __dadd_rn(a2, __ldcg(part + k));
    s[q] = a2;
  }
  __syncthreads();
  const double r = block_fold(s, kLanes2);
  if (l == 0) {
    *out = sqrt_out ? __dsqrt_rn(r) : r;
    *counter = 0;  // re-arm
  }
}

}  // namespace

cudaError_t launch_canon_reduce(const double* x, int64_t len, int kind, double coef,
                                double* partials, unsigned* counter, double* out,
                                int sqrt_out, cudaStream_t s, int64_t part_cap) {
  const int64_t nc = std::max<int64_t>(1, (len + kChunk - 1) / kChunk);
  canon_reduce_kernel<<<static_cast<unsigned>(nc), 256, 0, s>>>(
      x, len, kind, coef, partials, counter, out, sqrt_out, part_cap); count_launch(s);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// LSQR elementwise kernels (lsqr.cpp:41-52, :66-67)
// ---------------------------------------------------------------------------
namespace {

// if *norm > 0: dst = src / norm; scaled_out = scale .* dst (or dst)
// else: *invariant = 1 (and if skip_in: propagate skip)
__global__ void lsqr_normalize_kernel(double* dst, const double* src,
                                      const double* norm_dev, double* scaled_out,
                                      const double* scale, int64_t len,
                                      int* invariant, int* skip_in, int64_t ostride,
                                      const int32_t* slot) {
  if (skip_in && *skip_in) return;
  const double nrm = *norm_dev;
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (!(nrm > 0.0) && invariant) {
    if (k == 0) *invariant = 1;
    return;
  }
  if (k >= len) return;
  const double q = __ddiv_rn(src[k], nrm);
  dst[k] = q;
  const int64_t o = slot ? static_cast<int64_t>(slot[k]) : k;
  if (scaled_out) scaled_out[o * ostride] = scale ? __dmul_rn(scale[k], q) : q;
}

__global__ void lsqr_xw_kernel(double* x, double* w, const double* v, double c1,
                               double c2, const double* e, double* ex, int64_t n,
                               int64_t ostride, const int32_t* slot) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  const double wk = w[k];
  const double xk = __dadd_rn(x[k], __dmul_rn(c1, wk));  // x += (phi/rho) w
  x[k] = xk;
  w[k] = __dsub_rn(v[k], __dmul_rn(c2, wk));           // w = v - (theta/rho) w
  const int64_t o = slot ? static_cast<int64_t>(slot[k]) : k;
  if (ex) ex[o * ostride] = e ? __dmul_rn(e[k], xk) : xk;
}

}  // namespace

cudaError_t launch_lsqr_normalize(double* dst, const double* src,
                                  const double* norm_dev, double* scaled_out,
                                  const double* scale, int64_t len,
                                  int* invariant, int* skip_in, cudaStream_t s,
                                  int64_t ostride, const int32_t* slot) {
  const int64_t nb = std::max<int64_t>(1, (len + 255) / 256);
  lsqr_normalize_kernel<<<static_cast<unsigned>(nb), 256, 0, s>>>(
      dst, src, norm_dev, scaled_out, scale, len, invariant, skip_in, ostride, slot); count_launch(s);
  return cudaGetLastError();
}

cudaError_t launch_lsqr_xw_update(double* x, double* w, const double* v,
                                  double c1, double c2, const double* e,
                                  double* ex, int64_t n, cudaStream_t s, int64_t ostride,
                                  const int32_t* slot) {
  if (n == 0) return cudaSuccess;
  lsqr_xw_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(x, w, v, c1, c2,
                                                                        e, ex, n, ostride, slot); count_launch(s);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Diagnostics helper: per-row sqrt(sum_k ((a*a)*eu_i)*ev_j) - target, squared
// (metrics.cpp:24-56), rows of A (mat 0) or A^T (mat 1), sequential per row.
// ---------------------------------------------------------------------------
namespace {
__global__ void rms_terms_kernel(int mat, const int64_t* __restrict__ rp,
                                 const int32_t* __restrict__ ci,
                                 const double* __restrict__ va, int64_t rows,
                                 const double* __restrict__ eu,
                                 const double* __restrict__ ev,
                                 double* __restrict__ out, int64_t goff,
                                 double target) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  const int64_t g = goff + r;
  double acc = 0.0;
  for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
    const double a = va[k];
    const double ei = mat ? eu[ci[k]] : eu[g];
    const double ej = mat ? ev[g] : ev[ci[k]];
    acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(__dmul_rn(a, a), ei), ej));
  }
  const double d = __dsub_rn(__dsqrt_rn(acc), target);
  out[r] = __dmul_rn(d, d);
}
}  // namespace

cudaError_t launch_rms_terms(int mat, const DevCsr& M, const double* eu,
                             const double* ev, double* out, int64_t goff,
                             double target, cudaStream_t s) {
  if (M.rows == 0) return cudaSuccess;
  rms_terms_kernel<<<static_cast<unsigned>((M.rows + 255) / 256), 256, 0, s>>>(
      mat, M.row_ptr, M.col, M.val, M.rows, eu, ev, out, goff, target); count_launch(s);
  return cudaGetLastError();
}

}  // namespace eqb

namespace eqb {
// objective (src/equilibrate.cpp:10-22): per-row sequential sum over CSR(A) of
// (a*a) * exp(2*(u_i + v_j)), zero entries skipped (glibc exp -> det_exp here)
namespace {
__global__ void obj_terms_kernel(const int64_t* __restrict__ rp,
                                 const int32_t* __restrict__ ci,
                                 const double* __restrict__ va, int64_t rows,
                                 const double* __restrict__ u,
                                 const double* __restrict__ v,
                                 double* __restrict__ out) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  double acc = 0.0;
  const double ui = u[r];
  for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
    const double a = va[k];
    if (a == 0.0) continue;
    const double ex = det_exp(__dmul_rn(2.0, __dadd_rn(ui, v[ci[k]])));
    acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(a, a), ex));
  }
  out[r] = acc;
}
__global__ void mul_kernel(double* out, const double* a, const double* b, int64_t n) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < n) out[k] = __dmul_rn(a[k], b[k]);
}
}  // namespace

cudaError_t launch_obj_terms(const DevCsr& A, const double* u, const double* v,
                             double* out, cudaStream_t s) {
  if (A.rows == 0) return cudaSuccess;
  obj_terms_kernel<<<static_cast<unsigned>((A.rows + 255) / 256), 256, 0, s>>>(
      A.row_ptr, A.col, A.val, A.rows, u, v, out); count_launch(s);
  return cudaGetLastError();
}
cudaError_t launch_mul(double* out, const double* a, const double* b, int64_t n,
                       cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  mul_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(out, a, b, n); count_launch(s);
  return cudaGetLastError();
}
}  // namespace eqb
