// engine.cu -- host engine and C ABI (include/equil_b200.h): matrix creation
// and sharding, traversal plans, the SGD driver and LSQR.
//
// Owns the device-resident matrix (CSR(A), CSR(A^T) shards or dense A), the
// traversal plans, the sign stream and the SGD / LSQR drivers.  The T-iteration
// SGD loop is captured once as a CUDA graph per (T, targets, gamma, M) and
// replayed; LSQR keeps its scalar recurrence on the host (std::hypot, exactly
// as src/lsqr.cpp:58-64) with one device->host round trip per norm.  The
// variants, the lasso, the public helpers and file I/O are in engine_ext.cu.
#include "engine_internal.h"

#include <fcntl.h>
#include <pthread.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>

namespace eqe {

// Grow-only mapped pinned staging for h2d's pull copies, one per host thread.
// A block is reused only by the next setup on the same thread, which starts
// after the previous one synchronised its stream.
struct PullArena {
  struct Block {
    char* host = nullptr;
    char* dev = nullptr;
    size_t cap = 0, used = 0;
  };
  std::vector<Block> blocks;
  ~PullArena() {
    for (Block& b : blocks) cudaFreeHost(b.host);
  }
  char* take(size_t bytes, char** dev) {
    bytes = (bytes + 255) & ~static_cast<size_t>(255);
    for (Block& b : blocks)
      if (b.cap - b.used >= bytes) {
        *dev = b.dev + b.used;
        char* h = b.host + b.used;
        b.used += bytes;
        return h;
      }
    Block b;
    b.cap = std::max<size_t>(bytes, 32u << 20);
    void* hp = nullptr;
    CK(cudaHostAlloc(&hp, b.cap, cudaHostAllocMapped | cudaHostAllocPortable));
    b.host = static_cast<char*>(hp);
    void* dp = nullptr;
    CK(cudaHostGetDevicePointer(&dp, hp, 0));
    b.dev = static_cast<char*>(dp);
    b.used = bytes;
    blocks.push_back(b);
    *dev = b.dev;
    return b.host;
  }
};
static PullArena& pull_arena() {
  thread_local PullArena a;
  return a;
}
void pull_arena_reset() {
  for (PullArena::Block& b : pull_arena().blocks) b.used = 0;
}

void h2d(equil_matrix* M, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return;
  if (!M->pull_uploads) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, M->stream));
    return;
  }
  char* dev = nullptr;
  char* h = pull_arena().take(bytes, &dev);
  std::memcpy(h, src, bytes);
  CK(eqb::launch_pull_copy(dst, dev, bytes, M->stream));
}

Plan plan_tiles(const int64_t* rp, int64_t rows, int mat) {
  Plan P;
  const int64_t nwin = (rows + eqb::kSliceWindow - 1) / eqb::kSliceWindow;
  const int nth = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()), nwin / 8)));
  struct Part {
    std::vector<eqb::Tile> slices;
    std::vector<int32_t> maxlen;  // of each slice: its first row's length
    std::vector<int32_t> rowlist;
    std::vector<std::pair<int64_t, int64_t>> longs;
  };
  std::vector<Part> parts(nth);
  auto work = [&](int t) {
    Part& pt = parts[t];
    const int64_t wa = nwin * t / nth, wb = nwin * (t + 1) / nth;
    pt.rowlist.reserve(static_cast<size_t>((wb - wa) * eqb::kSliceWindow));
    pt.slices.reserve(static_cast<size_t>((wb - wa) * (eqb::kSliceWindow / eqb::kSliceRows + 1)));
    pt.maxlen.reserve(pt.slices.capacity());
    // a window's rows by decreasing length, ties in row order (a stable
    // counting sort: lengths are at most kTileNnz)
    std::vector<int32_t> start(eqb::kTileNnz + 2);
    std::vector<int32_t> wlen(eqb::kSliceWindow);
    for (int64_t w = wa; w < wb; ++w) {
      const int64_t w0 = w * eqb::kSliceWindow;
      const int64_t w1 = std::min<int64_t>(rows, w0 + eqb::kSliceWindow);
      std::fill(start.begin(), start.end(), 0);
      int nshort = 0;
      for (int64_t i = w0; i < w1; ++i) {
        const int64_t len = rp[i + 1] - rp[i];
        if (len > eqb::kTileNnz) {
          pt.longs.push_back({len, i});
          wlen[i - w0] = -1;
        } else {
          wlen[i - w0] = static_cast<int32_t>(len);
          ++start[len];
          ++nshort;
        }
      }
      int32_t run = 0;  // start[l] = rows longer than l
      for (int l = eqb::kTileNnz; l >= 0; --l) {
        const int32_t c = start[l];
        start[l] = run;
        run += c;
      }
      const size_t base = pt.rowlist.size();
      pt.rowlist.resize(base + nshort);
      for (int64_t i = w0; i < w1; ++i) {
        const int32_t l = wlen[i - w0];
        if (l >= 0) pt.rowlist[base + start[l]++] = static_cast<int32_t>(i);
      }
      for (int q = 0; q < nshort; q += eqb::kSliceRows) {
        const int cnt = std::min<int>(eqb::kSliceRows, nshort - q);
        pt.slices.push_back({static_cast<int32_t>(base + q), cnt, 2, static_cast<int16_t>(mat), 0});
        const int32_t r = pt.rowlist[base + q];
        pt.maxlen.push_back(static_cast<int32_t>(rp[r + 1] - rp[r]));
      }
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nth; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  std::vector<std::pair<int64_t, int64_t>> longs;
  std::vector<int32_t> slice_max;  // parallel to P.slices until the mids are inserted
  {
    size_t ns = 0, nr = 0;
    for (const Part& pt : parts) ns += pt.slices.size(), nr += pt.rowlist.size();
    P.slices.reserve(ns);
    slice_max.reserve(ns);
    P.rowlist.reserve(static_cast<size_t>(rows));
    (void)nr;
  }
  for (Part& pt : parts) {
    const int32_t base = static_cast<int32_t>(P.rowlist.size());
    for (eqb::Tile s : pt.slices) {
      s.r0 += base;
      P.slices.push_back(s);
    }
    slice_max.insert(slice_max.end(), pt.maxlen.begin(), pt.maxlen.end());
    P.rowlist.insert(P.rowlist.end(), pt.rowlist.begin(), pt.rowlist.end());
    longs.insert(longs.end(), pt.longs.begin(), pt.longs.end());
  }
  // rows longer than a tile: CTA-cooperative long slices of 32 length-sorted
  // rows (kind 3), each replicated once per warp of the CTA
  std::stable_sort(longs.begin(), longs.end(),
                   [](const auto& a, const auto& b) { return a.first > b.first; });
  // mid-length rows (kTileNnz, EQ_MID_MAX]: warp slices of 32 globally
  // length-sorted rows, placed first among the slices (longest first)
  size_t nlong = longs.size();
  if (eqb::kMidMax > eqb::kTileNnz) {
    size_t first_mid = 0;
    while (first_mid < longs.size() && longs[first_mid].first > eqb::kMidMax) ++first_mid;
    std::vector<eqb::Tile> mids;
    for (size_t q = first_mid; q < longs.size(); q += eqb::kSliceRows) {
      const int cnt = static_cast<int>(std::min<size_t>(eqb::kSliceRows, longs.size() - q));
      mids.push_back({static_cast<int32_t>(P.rowlist.size()), cnt, 2, static_cast<int16_t>(mat), 0});
      for (int k = 0; k < cnt; ++k) P.rowlist.push_back(static_cast<int32_t>(longs[q + k].second));
    }
    P.slices.insert(P.slices.begin(), mids.begin(), mids.end());
    // globally sorted: a mid slice's first row is its longest
    std::vector<int32_t> mmax;
    for (size_t q = first_mid; q < longs.size(); q += eqb::kSliceRows)
      mmax.push_back(static_cast<int32_t>(longs[q].first));
    slice_max.insert(slice_max.begin(), mmax.begin(), mmax.end());
    nlong = first_mid;
  }
  for (size_t q = 0; q < nlong; ++q) P.long_nnz += longs[q].first;
  for (size_t q = 0; q < nlong; q += eqb::kLongRows) {
    const int cnt = static_cast<int>(std::min<size_t>(eqb::kLongRows, nlong - q));
    const eqb::Tile t{static_cast<int32_t>(P.rowlist.size()), cnt, 3,
                      static_cast<int16_t>(mat), 0};
    for (int k = 0; k < cnt; ++k) P.rowlist.push_back(static_cast<int32_t>(longs[q + k].second));
    for (int w = 0; w < eqb::kTileWarps; ++w) P.lng.push_back(t);
  }
  // interleaved-slice entries, longest first
  auto ent = [&](const eqb::Tile& t, int lng) {
    int64_t mx = 0;
    for (int k = 0; k < t.r1; ++k) {
      const int32_t r = P.rowlist[t.r0 + k];
      mx = std::max<int64_t>(mx, rp[r + 1] - rp[r]);
    }
    return SellEnt{static_cast<int32_t>(mx), static_cast<int16_t>(t.r1),
                   static_cast<int16_t>(lng), t.r0};
  };
  // (long groups first, longest first; then the warp slices in window order)
  P.sell.reserve(P.lng.size() / eqb::kTileWarps + P.slices.size());
  for (size_t q = 0; q < P.lng.size(); q += eqb::kTileWarps) P.sell.push_back(ent(P.lng[q], 1));
  // (every slice is sorted longest first, so its first row gives maxlen)
  for (size_t q = 0; q < P.slices.size(); ++q) {
    const eqb::Tile& t = P.slices[q];
    P.sell.push_back(SellEnt{slice_max[q], static_cast<int16_t>(t.r1), 0, t.r0});
  }
  return P;
}

std::vector<int64_t> partition_rows(const int64_t* rp, int64_t rows, int parts) {
  // contiguous ranges balanced by (nnz + rows): boundary g at the first row
  // whose prefix cost reaches g/parts of the total
  std::vector<int64_t> b(parts + 1, rows);
  b[0] = 0;
  const double total = static_cast<double>(rp[rows] + rows);
  int g = 1;
  for (int64_t i = 0; i <= rows && g < parts; ++i) {
    const double cost = static_cast<double>(rp[i] + i);
    while (g < parts && cost >= total * g / parts) b[g++] = i;
  }
  while (g < parts) b[g++] = rows;
  b[parts] = rows;
  return b;
}

__global__ void remap_cols_kernel(int32_t* col, int64_t nnz, const int64_t* bounds,
                                  int parts, int64_t maxcnt) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= nnz) return;
  const int64_t j = col[k];
  int g = 0;
  while (g + 1 < parts && bounds[g + 1] <= j) ++g;
  col[k] = static_cast<int32_t>(g * maxcnt + (j - bounds[g]));
}

// sharded setup: a constant added to every column (local A row -> padded slot)
__global__ void add_cols_kernel(int32_t* col, int64_t nnz, int64_t delta) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < nnz) col[k] = static_cast<int32_t>(col[k] + delta);
}
// row lengths from row pointers
__global__ void row_counts_kernel(const int64_t* rp, int64_t rows, int32_t* cnt) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < rows) cnt[k] = static_cast<int32_t>(rp[k + 1] - rp[k]);
}
// Merge of the received CSR(A^T) pieces: run (source g, local row j) of cnt
// entries moves from src_off to dst_off.  Sources arrive in rank order and each
// holds ascending rows of A, so row j's entries end up in ascending original
// row order -- CSR(A^T)'s order (explicit_matrix.cpp:117-125).
__global__ void merge_runs_kernel(const int64_t* src_off, const int64_t* dst_off,
                                  const int32_t* cnt, int64_t runs, const int32_t* ci_in,
                                  const double* va_in, int32_t* ci_out, double* va_out) {
  const int64_t q = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 3;
  const int sub = threadIdx.x & 7;  // 8 threads per run
  if (q >= runs) return;
  const int64_t s0 = src_off[q], d0 = dst_off[q];
  for (int k = sub; k < cnt[q]; k += 8) {
    ci_out[d0 + k] = ci_in[s0 + k];
    va_out[d0 + k] = va_in[s0 + k];
  }
}

__global__ void rebase_rowptr_kernel(int64_t* dst, const int64_t* src, int64_t cnt,
                                     int64_t base) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < cnt) dst[k] = src[k] - base;
}

__global__ void unpad_kernel(double* dst, const double* src, const int64_t* bounds,
                             int parts, int64_t maxcnt, int64_t len) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= len) return;
  int g = 0;
  while (g + 1 < parts && bounds[g + 1] <= k) ++g;
  dst[k] = src[g * maxcnt + (k - bounds[g])];
}

}  // namespace eqe

namespace eqe {

void setup_common(equil_matrix* M, const equil_device_cfg* cfg) {
  M->device = cfg ? cfg->device : 0;
  M->rank = cfg ? cfg->rank : 0;
  M->world = cfg ? std::max(1, cfg->world_size) : 1;
  if (const char* e = getenv("EQUIL_SLOTS")) M->use_slots = atoi(e) != 0;
  if (const char* e = getenv("EQUIL_SELL")) M->use_sell = atoi(e) != 0;
  if (const char* e = getenv("EQUIL_SELL_VARIANT")) M->sell_variant = atoi(e);
  if (const char* e = getenv("EQUIL_SELL_LONG")) M->sell_long = atoi(e);
  if (const char* e = getenv("EQUIL_SELL_QUAD")) M->sell_quad = atoi(e) != 0;
  if (const char* e = getenv("EQUIL_SELL_LVARIANT")) M->sell_lvariant = atoi(e);
  if (const char* e = getenv("EQUIL_SELL_PASSES")) M->sell_passes = atoi(e) != 0;
  if (const char* e = getenv("EQUIL_SELL_ORDER")) M->sell_order = atoi(e);
  if (const char* e = getenv("EQUIL_SELL_BLOCKED")) M->sell_blocked = atoi(e) != 0;
  if (const char* e = getenv("EQUIL_BLOCK_WIN")) M->block_win = atoi(e) != 0;
  if (const char* e = getenv("EQUIL_SPLIT_EPI")) M->split_epi = atoi(e) != 0;
  if (const char* e = getenv("EQUIL_SWEEP")) {
    M->use_sweep = atoi(e) != 0;
    M->sweep_forced = M->use_sweep;
  }
  if (const char* e = getenv("EQUIL_SWEEP_WIDTH")) M->sweep_width = std::max(256, atoi(e) & ~1);
  if (const char* e = getenv("EQUIL_SWEEP_STAGES")) M->sweep_stages = std::max(2, atoi(e));

  require(M->rank >= 0 && M->rank < M->world, "device cfg: rank out of range");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  require(M->device >= 0 && M->device < ndev, "device cfg: no such CUDA device");
  CK(cudaSetDevice(M->device));
  CK(cudaStreamCreateWithFlags(&M->stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&M->copy_stream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&M->ev_vals, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&M->ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&M->ev_join, cudaEventDisableTiming));
  {
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&M->sign_stream, cudaStreamNonBlocking, hi));
    CK(cudaEventCreateWithFlags(&M->sign_ev, cudaEventDisableTiming));
  }
  {  // keep stream-ordered scratch (transpose, reductions) cached across calls
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, M->device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
  }
  if (M->world > 1) {
    require(cfg->nccl_id != nullptr, "device cfg: world_size > 1 needs nccl_id");
    const char* hxe = getenv("EQUIL_HOST_EXCHANGE");
    if (hxe && atoi(hxe) == 2) {  // processes, shared memory + CUDA IPC, no NCCL
      M->hx = shm_exchange(cfg->nccl_id, M->world, M->rank);
    } else if (hxe && atoi(hxe) != 0) {  // test transport (ThreadExchange), no NCCL
      M->hx = host_exchange(cfg->nccl_id, M->world);
    } else {
      if (!nccl().ok) fail(EQUIL_ENCCL, "libnccl.so.2 could not be loaded");
      ncclUniqueId id;
      std::memcpy(&id, cfg->nccl_id, sizeof id);
      nccl_check(nccl().CommInitRank(&M->comm, M->world, id, M->rank), "ncclCommInitRank");
    }
  }
  M->flags.alloc(1);
  M->red_counter.alloc(1);
  CK(cudaMemset(M->red_counter.p, 0, sizeof(unsigned)));
  M->scal.alloc(64);
  CK(cudaEventCreate(&M->ev_loop0));
  CK(cudaEventCreate(&M->ev_loop1));
  CK(cudaMemset(M->scal.p, 0, 64 * sizeof(double)));
}

// Upload the traversal plans of the local CSR(A) / CSR(A^T) shards.  The SGD
// launch covers both matrices: every long row (longest first, so the longest
// sequential chains start first), then the slices of A and of A^T.
// Merge the two matrices' interleaved-slice lists (both longest first; ties
// take A first) into the launch order, and lay out each matrix's arrays in it.
// slices of at least this many entries per row are stored in the quad layout
// (EQUIL_SELL_QUAD=0: none; EQUIL_QUAD_MIN: the threshold, default 64)
int quad_min(const equil_matrix* M) {
  if (!M->sell_quad) return 0x7fffffff;
  static const int qm = getenv("EQUIL_QUAD_MIN") ? std::max(4, atoi(getenv("EQUIL_QUAD_MIN"))) : 64;
  return qm;
}

void plan_sell(equil_matrix* M, const Plan& pa, const Plan& pt) {
  equil_matrix::SellHost& H = M->sell_host;
  H = equil_matrix::SellHost{};
  struct Src {
    const SellEnt* e;
    int mat;
  };
  // Launch order: the long groups of both matrices longest first, then the
  // warp slices -- longest first (EQUIL_SELL_ORDER=0, default; c3: 1.5% faster)
  // or in window order (1: the epilogues' row accesses stay local, which
  // matters once u, v and the gathered vectors outgrow L2, e.g. with blocks).
  std::vector<Src> order;
  order.reserve(pa.sell.size() + pt.sell.size());
  for (int mat = 0; mat < 2; ++mat)
    for (const SellEnt& e : mat ? pt.sell : pa.sell)
      if (e.lng && M->sell_long) order.push_back({&e, mat});
  const size_t nlong = order.size();
  for (int mat = 0; mat < 2; ++mat)
    for (const SellEnt& e : mat ? pt.sell : pa.sell)
      if (!e.lng) order.push_back({&e, mat});
  auto by_len = [](const Src& a, const Src& b) { return a.e->maxlen > b.e->maxlen; };
  std::stable_sort(order.begin(), order.begin() + nlong, by_len);
  if (M->sell_order == 0) std::stable_sort(order.begin() + nlong, order.end(), by_len);
  const size_t ns = order.size();
  H.slices.resize(ns);
  for (int mat = 0; mat < 2; ++mat) H.kbp[mat].assign(1, 0);
  for (size_t w = 0; w < ns; ++w) {
    const SellEnt& e = *order[w].e;
    const int mat = order[w].mat;
    H.slices[w] = {H.total[mat], e.maxlen, e.cnt, static_cast<int16_t>(mat)};
    // long slices read by the warp-specialised kernel are stored in the quad
    // layout (128-bit stream loads), padded to a multiple of 4 entries
    const bool quad = e.maxlen >= quad_min(M);
    H.total[mat] += 32 * (quad ? eqb::sell_quad_len(e.maxlen) : static_cast<int64_t>(e.maxlen));
    if (e.maxlen > 0) {
      H.midx[mat].push_back(static_cast<int32_t>(w));
      H.kbp[mat].push_back(H.kbp[mat].back() + (e.maxlen + 31) / 32);
    }
  }
  H.r0.resize(ns);
  for (size_t w = 0; w < ns; ++w) {
    H.r0[w] = order[w].e->r0;
    const int mat = order[w].mat;
    H.pidx[mat].push_back(static_cast<int32_t>(w));
    if (order[w].e->maxlen > eqb::kTileNnz) ++H.plong[mat];
  }
}

// The generic passes' column arrays (padded coordinates) and per-matrix slice
// orders, on first use.

// per-matrix slice orders of the generic passes (both column flavours)
void ensure_sell_order(equil_matrix* M) {
  if (M->sell_order_up || !M->sell) return;
  const equil_matrix::SellHost& H = M->sell_host;
  for (int mat = 0; mat < 2; ++mat) {
    M->sell_pidx[mat].alloc(H.pidx[mat].size());
    if (!H.pidx[mat].empty())
      CK(cudaMemcpyAsync(M->sell_pidx[mat].p, H.pidx[mat].data(), H.pidx[mat].size() * 4,
                         cudaMemcpyHostToDevice, M->stream));
  }
  CK(cudaStreamSynchronize(M->stream));
  M->sell_order_up = true;
}

void ensure_sell_pass(equil_matrix* M) {
  if (M->sell_pass || !M->sell) return;
  ensure_sell_order(M);
  const equil_matrix::SellHost& H = M->sell_host;
  cudaStream_t s = M->stream;
  for (int mat = 0; mat < 2; ++mat) {
    M->sell_pci[mat].alloc(H.total[mat]);
    DevBuf<int64_t> dkbp;
    DevBuf<int32_t> didx;
    dkbp.alloc(H.kbp[mat].size());
    didx.alloc(H.midx[mat].size());
    CK(cudaMemcpyAsync(dkbp.p, H.kbp[mat].data(), H.kbp[mat].size() * 8, cudaMemcpyHostToDevice,
                       s));
    if (!H.midx[mat].empty())
      CK(cudaMemcpyAsync(didx.p, H.midx[mat].data(), H.midx[mat].size() * 4,
                         cudaMemcpyHostToDevice, s));
    const eqb::DevCsr& C = mat ? M->AT : M->A;
    CK(eqb::build_sell(C.row_ptr, C.col, nullptr, C.val, dkbp.p, H.kbp[mat].back(), didx.p,
                       static_cast<int>(H.midx[mat].size()), M->sell_slices.p, M->sell_row.p,
                       M->sell_len.p, nullptr, M->sell_pci[mat].p, nullptr, s, quad_min(M)));
    CK(cudaStreamSynchronize(s));
  }
  M->sell_pass = true;
}

// One generic pass (b: the dual pass) over matrix `mat` on the interleaved
// slices: long slices on the copy stream, warp slices on the main stream.
// slotted: the gathered vector is in the hot-first slot layout, so the SGD
// passes' slot-mapped column arrays serve (LSQR, engine.cu lsqr_core).
void sell_pass(equil_matrix* M, int mat, const eqb::PassArgs& a, const eqb::PassArgs* b,
               bool pair = false, bool slotted = false) {
  if (slotted) {
    ensure_sell_order(M);
  } else {
    ensure_sell_pass(M);
  }
  const equil_matrix::SellHost& H = M->sell_host;
  cudaStream_t s = M->stream;
  eqb::SellArgs sa{};
  sa.xlen[0] = sa.xlen[1] = mat ? M->m_pad() : M->n_pad();  // padded coordinates
  sa.quad_min = quad_min(M);
  sa.slices = M->sell_slices.p;
  sa.order = M->sell_pidx[mat].p;
  sa.row = M->sell_row.p;
  sa.len = M->sell_len.p;
  for (int k = 0; k < 2; ++k) {
    sa.ci[k] = slotted ? M->sell_ci[k].p : M->sell_pci[k].p;
    sa.va[k] = M->sell_va[k].p;
  }
  const int nl = H.plong[mat], nall = static_cast<int>(H.pidx[mat].size());
  if (nl > 0) {
    CK(cudaEventRecord(M->ev_fork, s));
    CK(cudaStreamWaitEvent(M->copy_stream, M->ev_fork, 0));
    eqb::SellArgs sl = sa;
    sl.first = 0;
    sl.nslices = nl;
    CK(eqb::launch_sell_pass(a, b, sl, true, pair, M->copy_stream));
  }
  sa.first = nl;
  sa.nslices = nall;
  CK(eqb::launch_sell_pass(a, b, sa, false, pair, s));
  if (nl > 0) {
    CK(cudaEventRecord(M->ev_join, M->copy_stream));
    CK(cudaStreamWaitEvent(s, M->ev_join, 0));
  }
}

// Device arrays of the interleaved slices, columns mapped to slots on the way
// (the slot layout must be built).
// Column blocks (build_block_layout): the interleaved arrays are laid out
// block-major -- block b holds, per slice, each lane's entries with columns in
// block b, interleaved and padded to the slice's longest range -- so round b of
// an iteration streams exactly the entries whose gathers fall in block b.
// Columns stay in padded coordinates (blocks are column ranges).
void build_sell_blocked(equil_matrix* M) {
  const equil_matrix::SellHost& H = M->sell_host;
  cudaStream_t s = M->stream;
  const int ns = M->n_sell;
  const int nbm = std::max(M->nblk[0], M->nblk[1]);
  const int64_t nq = 32LL * ns;
  DevBuf<int32_t> kst, maxb;
  kst.alloc(nbm * nq);
  maxb.alloc(static_cast<size_t>(nbm) * ns);
  M->sell_bln.alloc(nbm * nq);
  CK(eqb::launch_sell_block_lanes(M->sell_slices.p, ns, M->sell_row.p, M->sell_len.p,
                                  M->A.row_ptr, M->A.col, M->AT.row_ptr, M->AT.col, M->nblk[0],
                                  M->nblk[1], M->bwidth[0], M->bwidth[1], nbm, kst.p,
                                  M->sell_bln.p, maxb.p, s));
  std::vector<int32_t> hm(static_cast<size_t>(nbm) * ns);
  CK(cudaMemcpyAsync(hm.data(), maxb.p, hm.size() * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  std::vector<eqb::SellSlice> tab(static_cast<size_t>(nbm) * ns);
  int64_t tot[2] = {0, 0};
  std::vector<std::vector<int64_t>> kbp[2];
  std::vector<std::vector<int32_t>> midx[2];
  for (int mat = 0; mat < 2; ++mat) {
    kbp[mat].resize(nbm);
    midx[mat].resize(nbm);
  }
  for (int b = 0; b < nbm; ++b)
    for (int w = 0; w < ns; ++w) {
      const int mat = H.slices[w].mat;
      eqb::SellSlice& e = tab[static_cast<size_t>(b) * ns + w];
      e = {0, 0, 0, static_cast<int16_t>(mat)};
      if (b >= M->nblk[mat]) continue;  // this matrix has fewer blocks
      const int32_t ml = hm[static_cast<size_t>(b) * ns + w];
      e = {tot[mat], ml, H.slices[w].cnt, static_cast<int16_t>(mat)};
      tot[mat] += 32 * static_cast<int64_t>(ml);
      if (kbp[mat][b].empty()) kbp[mat][b].push_back(0);
      if (ml > 0) {
        midx[mat][b].push_back(w);
        kbp[mat][b].push_back(kbp[mat][b].back() + (ml + 31) / 32);
      }
    }
  M->sell_bslices.alloc(tab.size());
  CK(cudaMemcpyAsync(M->sell_bslices.p, tab.data(), tab.size() * sizeof(tab[0]),
                     cudaMemcpyHostToDevice, s));
  for (int mat = 0; mat < 2; ++mat) {
    M->sell_ci[mat].alloc(tot[mat]);
    M->sell_va[mat].alloc(tot[mat]);
    const eqb::DevCsr& C = mat ? M->AT : M->A;
    for (int b = 0; b < M->nblk[mat]; ++b) {
      if (midx[mat][b].empty()) continue;
      DevBuf<int64_t> dkbp;
      DevBuf<int32_t> didx;
      dkbp.alloc(kbp[mat][b].size());
      didx.alloc(midx[mat][b].size());
      CK(cudaMemcpyAsync(dkbp.p, kbp[mat][b].data(), kbp[mat][b].size() * 8,
                         cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(didx.p, midx[mat][b].data(), midx[mat][b].size() * 4,
                         cudaMemcpyHostToDevice, s));
      CK(eqb::build_sell(C.row_ptr, C.col, nullptr, C.val, dkbp.p, kbp[mat][b].back(), didx.p,
                         static_cast<int>(midx[mat][b].size()),
                         M->sell_bslices.p + static_cast<size_t>(b) * ns, M->sell_row.p,
                         M->sell_bln.p + b * nq, kst.p + b * nq, M->sell_ci[mat].p,
                         M->sell_va[mat].p, s));
      CK(cudaStreamSynchronize(s));
    }
  }
  M->sell_carry.alloc(nq);
  M->sell_nb = nbm;
}

// interleaved arrays of matrix `mat`: columns (mapped to slots) and / or values
// part 0: every slice of the matrix; 1: only its long slices (rows longer than
// kTileNnz, the leading entries of the launch order); 2: all but those
void build_sell_arrays(equil_matrix* M, int mat, bool cols, bool vals, int part = 0) {
  const equil_matrix::SellHost& H = M->sell_host;
  cudaStream_t s = M->stream;
  // A's long slices are not needed by a one-shot SGD call that runs them on the
  // column sweep (M->sell_skip_long; build_sweep_layout completes them if the
  // sweep does not come about)
  if (part == 0 && mat == 0 && M->sell_skip_long) part = 2;
  const size_t nl = std::min<size_t>(static_cast<size_t>(H.plong[mat]), H.midx[mat].size());
  const size_t i0 = part == 2 ? nl : 0, i1 = part == 1 ? nl : H.midx[mat].size();
  if (i1 <= i0) return;
  std::vector<int64_t> kbp(H.kbp[mat].begin() + i0, H.kbp[mat].begin() + i1 + 1);
  for (int64_t& k : kbp) k -= H.kbp[mat][i0];
  DevBuf<int64_t> dkbp;
  DevBuf<int32_t> didx;
  dkbp.alloc_on(kbp.size(), s);
  didx.alloc_on(i1 - i0, s);
  h2d(M, dkbp.p, kbp.data(), kbp.size() * 8);
  h2d(M, didx.p, H.midx[mat].data() + i0, (i1 - i0) * 4);
  if (!M->pull_uploads) CK(cudaStreamSynchronize(s));  // kbp is a local (pageable) vector
  const eqb::DevCsr& C = mat ? M->AT : M->A;
  CK(eqb::build_sell(C.row_ptr, C.col, mat ? M->wmap.p : M->smap.p, C.val, dkbp.p, kbp.back(),
                     didx.p, static_cast<int>(i1 - i0), M->sell_slices.p, M->sell_row.p,
                     M->sell_len.p, nullptr, cols ? M->sell_ci[mat].p : nullptr,
                     vals ? M->sell_va[mat].p : nullptr, s, quad_min(M)));
}

// the values half of build_sell_layout(M, false), after A's values (and
// CSR(A^T)'s) are on the device
void build_sell_values(equil_matrix* M) {
  if (!M->sell_values_pending) return;
  for (int mat = 0; mat < 2; ++mat) build_sell_arrays(M, mat, false, true);
  M->sell_values_pending = false;
}

void build_sell_layout(equil_matrix* M, bool with_values) {
  M->sell = false;
  M->sell_values_pending = false;
  M->sell_nb = 1;
  const bool blocked = M->nblk[0] > 1 || M->nblk[1] > 1;
  if (!M->use_sell || (!M->slots && !blocked)) return;
  if (blocked && (!M->sell_blocked || M->sell_long == 0)) return;
  const equil_matrix::SellHost& H = M->sell_host;
  cudaStream_t s = M->stream;
  // (allocations ordered on s: the host may be ahead of the device here, and a
  // host-synchronous pool allocation would grow the pool instead of reusing what
  // the transpose's temporaries free in stream order)
  auto upload = [&](auto& d, const auto& h) {
    d.alloc_async(h.size(), s);
    h2d(M, d.p, h.data(), h.size() * sizeof(h[0]));
  };
  upload(M->sell_slices, H.slices);
  M->n_sell = static_cast<int>(H.slices.size());
  {  // lane -> row and length, from the device row lists
    DevBuf<int32_t> dr0;
    dr0.alloc_on(H.r0.size(), s);
    h2d(M, dr0.p, H.r0.data(), H.r0.size() * 4);
    M->sell_row.alloc_async(32 * static_cast<size_t>(M->n_sell), s);
    M->sell_len.alloc_async(32 * static_cast<size_t>(M->n_sell), s);
    CK(eqb::launch_sell_rows(M->sell_slices.p, dr0.p, M->n_sell, M->rowlist_a.p,
                             M->rowlist_t.p, M->A.row_ptr, M->AT.row_ptr, M->sell_row.p,
                             M->sell_len.p, s));
  }
  M->n_sell_long = 0;
  while (M->n_sell_long < M->n_sell && H.slices[M->n_sell_long].maxlen > eqb::kTileNnz)
    ++M->n_sell_long;
  for (int mat = 0; mat < 2 && !blocked; ++mat) {
    M->sell_ci[mat].alloc_async(H.total[mat], s);
    M->sell_va[mat].alloc_async(H.total[mat], s);
    // columns of A index xs (slot map smap), columns of A^T index xw (wmap);
    // the values follow in build_sell_values once they are on the device
    build_sell_arrays(M, mat, true, with_values);
  }
  M->sell_values_pending = !blocked && !with_values;
  if (blocked) build_sell_blocked(M);
  if (M->sell_long || M->n_sgd_long == 0) {  // the staged kernel no longer runs
    M->a_ci_sgd.release();
    M->t_ci_sgd.release();
  }
  M->sell = true;
  M->sell_pass = false;
  if (M->sell_long == 0) M->sell_passes = false;  // long rows are not in the slices
  if (blocked) M->sell_passes = false;            // the passes' arrays are not blocked
}

// Column sweep of A's long rows (sweep.cu): deal the rows to one CTA per SM
// (longest first, boustrophedon, so every CTA gets the same count and a similar
// number of entries), cut each row into its runs per panel, sort every (CTA,
// panel)'s rows by run length and lay the blobs out.  The values follow in
// build_sweep_values once they are on the device.
// the layout construction's per-(CTA, panel, row) tables, once the blobs are complete
void release_sweep_scratch(equil_matrix* M) {
  cudaStream_t s = M->stream;
  M->sweep_rstart.release_on(s);
  M->sweep_perm.release_on(s);
  M->sweep_srun.release_on(s);
  M->sweep_gbase.release_on(s);
  M->sweep_nepad.release_on(s);
}

void build_sweep_values(equil_matrix* M) {
  if (!M->sweep || !M->sweep_values_pending) return;
  const eqb::SweepArgs& sw = M->sweep_args;
  CK(eqb::launch_sweep_fill(M->A.row_ptr, M->A.col, M->A.val, M->sweep_crow.p, sw.nctas, sw.rmax,
                            sw.npanels, sw.width, M->sweep_perm.p, M->sweep_srun.p,
                            M->sweep_gbase.p, M->sweep_nepad.p, M->sweep_rstart.p, M->sweep_off.p,
                            M->sweep_blobs.p, false, true, M->stream));
  M->sweep_values_pending = false;
  release_sweep_scratch(M);
}

// First half (plan_sweep_layout): deal the rows, pick the panel width, enqueue the
// run / sort kernels and the copy of the blob sizes to the host, and record an
// event -- no host wait, so the interleaved layout can be enqueued behind it.
// Second half (build_sweep_layout): wait for that event only, lay the blobs out
// and fill them.
namespace {
struct SweepPlan {
  bool ok = false;
  int G = 0, R = 0, NG = 0, W = 0, P = 0;
  size_t ncp = 0;
  int64_t hdr = 0;
};

void sweep_enqueue_runs(equil_matrix* M, SweepPlan& sp) {
  cudaStream_t s = M->stream;
  sp.P = static_cast<int>((M->n + sp.W - 1) / sp.W);
  sp.ncp = static_cast<size_t>(sp.G) * sp.P;
  DevBuf<int32_t> rowlen;
  rowlen.alloc_on(static_cast<size_t>(sp.G) * sp.R, s);
  M->sweep_rstart.alloc_async(sp.ncp * sp.R, s);
  M->sweep_perm.alloc_async(sp.ncp * sp.R, s);
  M->sweep_srun.alloc_async(sp.ncp * sp.R, s);
  M->sweep_gbase.alloc_async(sp.ncp * sp.NG, s);
  M->sweep_nepad.alloc_async(sp.ncp, s);
  CK(eqb::launch_sweep_runs(M->A.row_ptr, M->A.col, M->sweep_crow.p, sp.G, sp.R, sp.P, sp.W,
                            M->sweep_rstart.p, rowlen.p, s));
  CK(eqb::launch_sweep_sort(M->sweep_rstart.p, rowlen.p, sp.G, sp.R, sp.P, M->sweep_perm.p,
                            M->sweep_srun.p, M->sweep_gbase.p, M->sweep_nepad.p, s));
  // pinned landing buffer for the sizes: cached per host thread (pinning and
  // unpinning memory per handle cost tens of ms now and then, and cudaFreeHost
  // synchronises the device); build_sweep_layout reads it on the same thread
  struct PinnedScratch {
    uint32_t* p = nullptr;
    size_t cap = 0;
    ~PinnedScratch() {  // at thread exit (an error after runtime shutdown is moot)
      if (p) cudaFreeHost(p);
    }
  };
  static thread_local PinnedScratch ps;
  if (ps.cap < sp.ncp) {
    if (ps.p) cudaFreeHost(ps.p);
    ps.p = nullptr;
    ps.cap = 0;
    void* q = nullptr;
    CK(cudaHostAlloc(&q, sp.ncp * 4 * 2, cudaHostAllocDefault));
    ps.p = static_cast<uint32_t*>(q);
    ps.cap = sp.ncp * 2;
  }
  M->sweep_ne_host = ps.p;
  CK(cudaMemcpyAsync(M->sweep_ne_host, M->sweep_nepad.p, sp.ncp * 4, cudaMemcpyDeviceToHost, s));
  if (!M->ev_sweep) CK(cudaEventCreateWithFlags(&M->ev_sweep, cudaEventDisableTiming));
  CK(cudaEventRecord(M->ev_sweep, s));
}
}  // namespace

void plan_sweep_layout(equil_matrix* M) {
  M->sweep = false;
  M->sweep_values_pending = false;
  M->sweep_plan_ok = false;
  M->sell_skip_long = false;
  if (!M->sweep_candidate || !M->use_sell || !M->slots || M->sell_long != 2 || !M->split_epi ||
      M->nblk[0] > 1 || M->nblk[1] > 1)
    return;
  const equil_matrix::SellHost& H = M->sell_host;
  const std::vector<int32_t>& rows = M->sweep_rows_host;
  if (rows.empty() || H.plong[1] != 0) return;  // (A^T's long rows stay on the long kernel)
  cudaStream_t s = M->stream;
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, M->device));
  SweepPlan sp;
  sp.G = static_cast<int>(std::min<size_t>(nsm, rows.size()));
  const int per = static_cast<int>((rows.size() + sp.G - 1) / sp.G);
  sp.R = (per + 127) / 128 * 128;
  if (sp.R > 896) return;  // 32 producer + R consumer threads per CTA
  sp.NG = sp.R / 32;
  const int G = sp.G, R = sp.R;
  std::vector<int32_t> crow(static_cast<size_t>(G) * R, -1);
  for (size_t i = 0; i < rows.size(); ++i) {
    const size_t round = i / G, pos = i % G;
    const size_t c = (round & 1) ? G - 1 - pos : pos;
    crow[c * R + round] = rows[i];
  }
  M->sweep_crow.alloc_async(crow.size(), s);
  h2d(M, M->sweep_crow.p, crow.data(), crow.size() * 4);
  if (!M->pull_uploads) CK(cudaStreamSynchronize(s));  // crow is a local (pageable) vector
  // Panel width: two stages of (panel + the CTA's largest blob) must fit in
  // shared memory.  A CTA's blob holds about W / n of its entries at 10 bytes
  // each plus padding; start from that estimate and narrow if the layout
  // disagrees (EQUIL_SWEEP_WIDTH fixes the first try).
  sp.hdr = 16 + 4 * sp.NG + 4 * R;
  sp.W = M->sweep_width;
  if (sp.W <= 0) {
    const double ent_per_col = static_cast<double>(M->sweep_long_nnz) / G / static_cast<double>(M->n);
    const double budget = 227.0 * 1024 / 2 - sp.hdr - 4.0 * R - 4096;
    sp.W = static_cast<int>(budget / (8.0 + 15.0 * ent_per_col));
    sp.W = std::max(128, std::min(sp.W, 16384) / 512 * 512);
  }
  sweep_enqueue_runs(M, sp);
  sp.ok = true;
  M->sweep_plan_ok = true;
  M->sell_skip_long = M->oneshot_hint;  // (see build_sell_arrays)
  M->sweep_plan_G = sp.G;
  M->sweep_plan_R = sp.R;
  M->sweep_plan_W = sp.W;
}

static void build_sweep_layout_impl(equil_matrix* M, bool with_values);
void build_sweep_layout(equil_matrix* M, bool with_values) {
  if (!M->sweep_plan_ok) return;
  M->sweep_plan_ok = false;
  build_sweep_layout_impl(M, with_values);
  // A's long interleaved slices were left out for the sweep: if it did not come
  // about, the long-slice kernel needs them after all
  if (M->sell_skip_long && !M->sweep) {
    M->sell_skip_long = false;
    if (M->sell) build_sell_arrays(M, 0, true, with_values, 1);
  }
}

static void build_sweep_layout_impl(equil_matrix* M, bool with_values) {
  if (!M->sell || M->sell_nb != 1) return;
  if (getenv("EQUIL_SWEEP_FAIL")) return;  // test hook: the layout "does not fit"
  cudaStream_t s = M->stream;
  SweepPlan sp;
  sp.G = M->sweep_plan_G;
  sp.R = M->sweep_plan_R;
  sp.W = M->sweep_plan_W;
  sp.NG = sp.R / 32;
  sp.hdr = 16 + 4 * sp.NG + 4 * sp.R;
  sp.P = static_cast<int>((M->n + sp.W - 1) / sp.W);
  sp.ncp = static_cast<size_t>(sp.G) * sp.P;
  const int G = sp.G, R = sp.R;
  eqb::SweepArgs sw{};
  std::vector<int64_t> off;
  for (int attempt = 0;; ++attempt) {
    if (attempt == 6) return;  // the rows do not fit this scheme
    CK(cudaEventSynchronize(M->ev_sweep));  // the blob sizes are on the host
    const uint32_t* ne = M->sweep_ne_host;
    off.assign(sp.ncp + 1, 0);
    int64_t bmax = 0;
    for (size_t q = 0; q < sp.ncp; ++q) {
      const int64_t b = sp.hdr + 10 * static_cast<int64_t>(ne[q]);
      off[q + 1] = off[q] + b;
      bmax = std::max(bmax, b);
    }
    sw = eqb::SweepArgs{};
    sw.nctas = G;
    sw.rmax = R;
    sw.npanels = sp.P;
    sw.width = sp.W;
    sw.ncols = M->n;
    sw.blob_max = static_cast<unsigned>(bmax);
    sw.stages = M->sweep_stages;
    while (sw.stages > 2 && eqb::sweep_smem_bytes(sw) > 227 * 1024) --sw.stages;
    if (eqb::sweep_smem_bytes(sw) <= 227 * 1024) break;
    // narrower panels, smaller blobs: scale by what the largest blob may take
    const double room = 227.0 * 1024 / 2 - 4.0 * R - 4.0 * sp.P - 256 - 8.0 * sp.W;
    const double f = room > 4096 ? room / static_cast<double>(bmax) : 0.25;
    const int Wn = static_cast<int>(sp.W * std::min(0.8, 0.9 * f)) / 64 * 64;
    if (Wn < 128) return;
    sp.W = Wn;
    sweep_enqueue_runs(M, sp);
  }
  const int P = sp.P, W = sp.W;
  const size_t ncp = sp.ncp;
  M->sweep_off.alloc_async(off.size(), s);
  h2d(M, M->sweep_off.p, off.data(), off.size() * 8);
  M->sweep_blobs.alloc_async(static_cast<size_t>(off[ncp]), s);
  CK(cudaMemsetAsync(M->sweep_blobs.p, 0, static_cast<size_t>(off[ncp]), s));
  CK(eqb::launch_sweep_fill(M->A.row_ptr, M->A.col, M->A.val, M->sweep_crow.p, G, R, P, W,
                            M->sweep_perm.p, M->sweep_srun.p, M->sweep_gbase.p, M->sweep_nepad.p,
                            M->sweep_rstart.p, M->sweep_off.p, M->sweep_blobs.p, true, with_values,
                            s));
  if (!M->pull_uploads) CK(cudaStreamSynchronize(s));  // off is a local (pageable) vector
  sw.blobs = M->sweep_blobs.p;
  sw.blob_off = M->sweep_off.p;
  sw.crow = M->sweep_crow.p;
  M->sweep_args = sw;
  M->sweep = true;
  M->sweep_values_pending = !with_values;
  if (with_values) release_sweep_scratch(M);
  if (getenv("EQUIL_VERBOSE"))
    fprintf(stderr, "[equil] sweep: %d CTAs x %d rows, %d panels of %d, %d stages, blobs %.1f MB (max %u B)\n",
            G, R, P, W, sw.stages, off[ncp] / 1048576.0, sw.blob_max);
}

void upload_plans(equil_matrix* M, const Plan& pa, const Plan& pt) {
  if (M->use_sell) plan_sell(M, pa, pt);
  M->sweep_rows_host.clear();
  M->sweep_long_nnz = pa.long_nnz;
  if (M->sweep_candidate)  // A's long rows, longest first (each group is listed once per warp)
    for (size_t q = 0; q < pa.lng.size(); q += eqb::kTileWarps)
      for (int k = 0; k < pa.lng[q].r1; ++k)
        M->sweep_rows_host.push_back(pa.rowlist[pa.lng[q].r0 + k]);
  // kind-3 groups (4 entries each) first, so every group starts on a CTA
  std::vector<eqb::Tile> sgd = pa.lng;
  sgd.insert(sgd.end(), pt.lng.begin(), pt.lng.end());
  sgd.insert(sgd.end(), pa.slices.begin(), pa.slices.end());
  sgd.insert(sgd.end(), pt.slices.begin(), pt.slices.end());
  std::vector<eqb::Tile> ta = pa.lng, tt = pt.lng;
  ta.insert(ta.end(), pa.slices.begin(), pa.slices.end());
  tt.insert(tt.end(), pt.slices.begin(), pt.slices.end());
  auto upload = [&](auto& d, const auto& h) {
    d.alloc(h.size());
    h2d(M, d.p, h.data(), h.size() * sizeof(h[0]));
    return static_cast<int>(h.size());
  };
  M->n_sgd = upload(M->tiles_sgd, sgd);
  M->n_sgd_long = static_cast<int>(pa.lng.size() + pt.lng.size());
  M->n_la = static_cast<int>(pa.lng.size());
  M->n_sa = static_cast<int>(pa.slices.size());
  M->n_a = upload(M->tiles_a, ta);
  M->n_t = upload(M->tiles_t, tt);
  upload(M->rowlist_a, pa.rowlist);
  upload(M->rowlist_t, pt.rowlist);
}

void allgather_padded(equil_matrix* M, double* buf, int64_t maxcnt) {
  if (M->world == 1) return;
  if (M->hx) {  // host exchange: own slice out, barrier, peers' slices in, barrier
    const size_t bytes = static_cast<size_t>(maxcnt) * 8;
    CK(cudaStreamSynchronize(M->stream));
    std::vector<char> mine(bytes);
    if (bytes) CK(cudaMemcpy(mine.data(), buf + M->rank * maxcnt, bytes, cudaMemcpyDeviceToHost));
    M->hx->put(M->rank, mine.data(), bytes);
    M->hx->barrier();
    for (int g = 0; g < M->world; ++g)
      if (g != M->rank && bytes)
        h2d_sync(M->stream, buf + g * maxcnt, M->hx->slot(g), bytes);
    M->hx->barrier();
    return;
  }
  nccl_check(nccl().AllGather(buf + M->rank * maxcnt, buf, static_cast<size_t>(maxcnt),
                              ncclFloat64, M->comm, M->stream),
             "ncclAllGather");
}

// Fused all-gather of the SGD loop.  With world > 1 every rank maps every peer's
// gathered-vector buffer (xbuf, same layout on all ranks): CUDA IPC handles are
// all-gathered over NCCL and opened with peer access (NVLink / NVSwitch), or,
// under the host exchange, the in-process pointers are passed directly.  The SGD
// epilogue then stores each next value into all copies and the iteration ends
// with a one-word barrier instead of two padded all-gathers.  Negotiated once
// (collectively, at the first SGD call); any rank unable to map turns it off
// for all.  EQUIL_P2P=0 keeps the NCCL all-gathers.
static int64_t elem_delta(const void* peer, const double* mine) {
  // both allocations are 256-byte aligned, so the offset is whole doubles
  return (static_cast<int64_t>(reinterpret_cast<intptr_t>(peer)) -
          static_cast<int64_t>(reinterpret_cast<intptr_t>(mine))) /
         static_cast<int64_t>(sizeof(double));
}

// Cross-process host exchange (EQUIL_HOST_EXCHANGE=2): one POSIX shared-memory
// segment per communicator id -- a header with a process-shared barrier, then
// one slot of EQUIL_SHM_SLOT_MB (default 8) per rank.  Rank 0 initialises the
// header; the others wait for its magic word.  The name is unlinked once every
// rank has attached (the mappings stay valid).
struct ShmExchange : HostExchange {
  struct Header {
    std::atomic<unsigned long long> magic;
    pthread_barrier_t bar;
    int world;
    size_t cap;
  };
  static constexpr unsigned long long kMagic = 0x6571756c73686d31ULL;  // "equlshm1"
  Header* h = nullptr;
  char* base = nullptr;
  size_t total = 0;
  size_t cap = 0;
  std::string name;
  ShmExchange(const void* id128, int world_, int rank) {
    world = world_;
    const unsigned char* id = static_cast<const unsigned char*>(id128);
    uint64_t hsh = 1469598103934665603ULL;  // FNV-1a of the id
    for (int k = 0; k < 128; ++k) hsh = (hsh ^ id[k]) * 1099511628211ULL;
    char nm[64];
    snprintf(nm, sizeof nm, "/equil_%016llx", static_cast<unsigned long long>(hsh));
    name = nm;
    double mb = 8.0;
    if (const char* e = getenv("EQUIL_SHM_SLOT_MB")) mb = std::max(0.001, atof(e));
    cap = static_cast<size_t>(mb * (1 << 20));
    total = 4096 + cap * world;
    const int fd = shm_open(name.c_str(), O_CREAT | O_RDWR, 0600);
    if (fd < 0) fail(EQUIL_ERUNTIME, "host exchange: shm_open failed");
    if (ftruncate(fd, static_cast<off_t>(total)) != 0) {
      close(fd);
      fail(EQUIL_ERUNTIME, "host exchange: ftruncate failed");
    }
    void* p = mmap(nullptr, total, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) fail(EQUIL_ERUNTIME, "host exchange: mmap failed");
    h = static_cast<Header*>(p);
    base = static_cast<char*>(p) + 4096;
    if (rank == 0) {
      pthread_barrierattr_t at;
      pthread_barrierattr_init(&at);
      pthread_barrierattr_setpshared(&at, PTHREAD_PROCESS_SHARED);
      pthread_barrier_init(&h->bar, &at, static_cast<unsigned>(world));
      pthread_barrierattr_destroy(&at);
      h->world = world;
      h->cap = cap;
      h->magic.store(kMagic, std::memory_order_release);
    } else {
      for (int k = 0; h->magic.load(std::memory_order_acquire) != kMagic; ++k) {
        if (k > 600000) fail(EQUIL_ERUNTIME, "host exchange: rank 0 never attached");
        std::this_thread::sleep_for(std::chrono::microseconds(100));
      }
    }
    barrier();
    if (rank == 0) shm_unlink(name.c_str());
  }
  ~ShmExchange() override {
    if (h) munmap(h, total);
  }
  void barrier() override { pthread_barrier_wait(&h->bar); }
  void put(int rank, const void* data, size_t bytes) override {
    if (bytes > cap) fail(EQUIL_ERUNTIME, "host exchange: slot too small (EQUIL_SHM_SLOT_MB)");
    std::memcpy(base + rank * cap, data, bytes);
  }
  const char* slot(int g) override { return base + g * cap; }
  bool in_process() const override { return false; }
  size_t capacity() const override { return cap; }
};

std::shared_ptr<HostExchange> shm_exchange(const void* id128, int world, int rank) {
  return std::make_shared<ShmExchange>(id128, world, rank);
}

// bytes of every rank, in rank order, through the handle's transport
static std::vector<char> allgather_bytes(equil_matrix* M, const void* mine, size_t bytes) {
  const int G = M->world;
  std::vector<char> all(G * bytes);
  if (M->hx) {
    M->hx->put(M->rank, mine, bytes);
    M->hx->barrier();
    for (int g = 0; g < G; ++g) std::memcpy(all.data() + g * bytes, M->hx->slot(g), bytes);
    M->hx->barrier();
    return all;
  }
  DevBuf<char> buf;
  buf.alloc(G * bytes);
  cudaStream_t s = M->stream;
  CK(cudaMemcpyAsync(buf.p + M->rank * bytes, mine, bytes, cudaMemcpyHostToDevice, s));
  nccl_check(nccl().AllGather(buf.p + M->rank * bytes, buf.p, bytes, ncclUint8, M->comm, s),
             "ncclAllGather");
  CK(cudaMemcpyAsync(all.data(), buf.p, G * bytes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return all;
}

void setup_peers(equil_matrix* M) {
  M->p2p_state = -1;
  const int G = M->world, r = M->rank;
  int want = (!M->dense && G - 1 <= EQ_MAX_PEERS) ? 1 : 0;
  if (const char* e = getenv("EQUIL_P2P")) want = want && atoi(e) != 0;
  CK(cudaStreamSynchronize(M->stream));
  const bool local = M->hx && M->hx->in_process();
  struct Rec {
    int32_t ok;
    int32_t pad;
    double* base;  // in-process transport: the buffer itself
    cudaIpcMemHandle_t h;
  } mine{};
  mine.ok = want;
  mine.base = M->xbuf.p;
  if (want && !local) {
    mine.ok = cudaIpcGetMemHandle(&mine.h, M->xbuf.p) == cudaSuccess;
    cudaGetLastError();
  }
  std::vector<char> raw = allgather_bytes(M, &mine, sizeof mine);
  std::vector<Rec> all(G);
  std::memcpy(all.data(), raw.data(), G * sizeof(Rec));
  bool ok = true;
  for (const Rec& x : all) ok = ok && x.ok;
  if (!ok) return;  // every rank saw the same records
  std::vector<int64_t> delta;
  unsigned opened = 1;
  for (int g = 0; g < G; ++g) {
    if (g == r) continue;
    if (local) {
      delta.push_back(elem_delta(all[g].base, M->xbuf.p));
      continue;
    }
    void* q = nullptr;
    if (cudaIpcOpenMemHandle(&q, all[g].h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) {
      M->peer_mapped.push_back(q);
      delta.push_back(elem_delta(q, M->xbuf.p));
    } else {
      opened = 0;
    }
    cudaGetLastError();
  }
  // every rank must have mapped every peer
  raw = allgather_bytes(M, &opened, sizeof opened);
  for (int g = 0; g < G; ++g) {
    unsigned v = 0;
    std::memcpy(&v, raw.data() + g * sizeof v, sizeof v);
    opened = opened && v;
  }
  if (!opened) {
    for (void* q : M->peer_mapped) cudaIpcCloseMemHandle(q);
    M->peer_mapped.clear();
    return;
  }
  M->peer_delta = delta;
  M->bar.alloc(1);
  CK(cudaMemsetAsync(M->bar.p, 0, sizeof(unsigned), M->stream));
  CK(cudaMemsetAsync(M->xbar(), 0, eqb::kBarWords * sizeof(unsigned long long), M->stream));
  CK(cudaStreamSynchronize(M->stream));
  allgather_bytes(M, &opened, sizeof opened);  // no rank signals before all flags are zero
  M->p2p_state = 1;
}

// End of a fused-all-gather iteration: no rank starts iteration t+1 (which
// overwrites the buffers its peers read in iteration t) before every rank's
// passes and peer stores of iteration t are complete.  Host transports: a host
// barrier.  NCCL: a device flag barrier on the peer-mapped buffers
// (peer_barrier_kernel: release-store of the epoch into every peer's flag for
// this rank, acquire-spin on the own flags), graph-capturable and without a
// collective; EQUIL_P2P_BARRIER=nccl keeps a one-word ncclAllReduce instead.
void rank_barrier(equil_matrix* M) {
  if (M->hx) {
    CK(cudaStreamSynchronize(M->stream));
    M->hx->barrier();
    return;
  }
  static const bool use_nccl = getenv("EQUIL_P2P_BARRIER") &&
                               std::string(getenv("EQUIL_P2P_BARRIER")) == "nccl";
  if (use_nccl) {
    nccl_check(nccl().AllReduce(M->bar.p, M->bar.p, 1, ncclUint32, ncclMax, M->comm, M->stream),
               "ncclAllReduce");
    return;
  }
  CK(eqb::launch_peer_barrier(M->xbar(), M->rank, M->world, M->peer_delta.data(),
                              static_cast<int>(M->peer_delta.size()), M->stream));
}

// Column blocks for gathered vectors larger than L2.  When the vector a pass
// gathers from (xs for A, xw for A^T) exceeds EQUIL_BLOCK_MB (default 60 MB,
// measured best on c5 among 20-80 MB: blocks of 40-53 MB), its coordinates are cut
// into nb contiguous blocks and each iteration visits every row block by block
// in nb launches, carrying the row's running sum between them (SgdEpi::span).
// A row's entries of one block are contiguous and blocks ascend, so the sum
// order is unchanged.  The slot layout is not used with blocks.
void build_block_layout(equil_matrix* M) {
  M->nblk[0] = M->nblk[1] = 1;
  double mb = 60.0;
  if (const char* e = getenv("EQUIL_BLOCK_MB")) {
    const double v = atof(e);
    if (v > 0.0) mb = v;
  }
  const int64_t lens[2] = {M->n_pad(), M->m_pad()};
  for (int mat = 0; mat < 2; ++mat) {
    const double bytes = static_cast<double>(lens[mat]) * 8.0;
    // (at most 1024 blocks: the per-row block boundaries take rows * (nb - 1) ints)
    const int nb = static_cast<int>(std::min(1024.0, std::ceil(bytes / (mb * 1e6))));
    if (nb <= 1) continue;
    const eqb::DevCsr& C = mat ? M->AT : M->A;
    const int64_t width = (lens[mat] + nb - 1) / nb;
    M->nblk[mat] = nb;
    M->bwidth[mat] = width;
    M->bnd[mat].alloc(std::max<int64_t>(1, C.rows * (nb - 1)));
    M->carry[mat].alloc(std::max<int64_t>(1, C.rows));
    CK(eqb::launch_block_bounds(C, nb, width, M->bnd[mat].p, M->stream));
  }
  if (M->nblk[0] > 1 || M->nblk[1] > 1) M->use_slots = false;
}

// Hot-first slot layout.  In the A^T pass every entry of A's row i gathers
// xw[i], so row i is read len(row i) times per iteration; with Zipf row lengths
// a few thousand rows take most gathers (c3: the 20k longest rows, 156 KB, take
// 57%).  Scattered over the 16 MB vector, each of them pins its own 128-byte L1
// line; packed together they fit in L1.  Rows are ordered by decreasing
// floor(log2(length)) (stable), per rank inside its own padded range, and the
// same is done for the columns feeding xs.  Only memory placement changes:
// every row sum keeps its entries and their order.  Built on the device from
// the global row pointers (a 7-bit stable radix sort per matrix).
void build_slot_layout(equil_matrix* M, const int64_t* rpA_dev, const int64_t* rpT_dev) {
  M->slots = false;
  if (!M->use_slots) return;
  cudaStream_t s = M->stream;
  const int G = M->world;
  DevBuf<int64_t> ab, tb;
  const int64_t* abd = M->a_bounds_d.p;
  const int64_t* tbd = M->t_bounds_d.p;
  if (G == 1) {  // bounds {0, rows}
    ab.alloc_on(2, s);
    tb.alloc_on(2, s);
    const int64_t a2[2] = {0, M->m}, t2[2] = {0, M->n};
    h2d(M, ab.p, a2, 16);
    h2d(M, tb.p, t2, 16);
    abd = ab.p;
    tbd = tb.p;
  }
  M->wmap.alloc(M->m_pad());
  M->smap.alloc(M->n_pad());
  CK(eqb::launch_slot_map(rpA_dev, M->m, abd, G, M->a_max, M->wmap.p, s));
  // the column sweep walks xs in column order: A's columns keep their positions
  CK(eqb::launch_slot_map(rpT_dev, M->n, tbd, G, M->t_max, M->smap.p, s, M->sweep_candidate));
  if (!M->use_sell || M->sell_long == 0) {  // slot-mapped columns of the staged traversal
    M->a_ci_sgd.alloc(M->A.nnz);
    M->t_ci_sgd.alloc(M->AT.nnz);
    CK(eqb::launch_remap_cols(M->a_ci_sgd.p, M->A.col, M->smap.p, M->A.nnz, s));
    CK(eqb::launch_remap_cols(M->t_ci_sgd.p, M->AT.col, M->wmap.p, M->AT.nnz, s));
  }
  M->slots = true;  // complete when `stream` reaches here (setup ends with a sync)
}

// Build local shards from the full device CSR(A) and CSR(A^T).
void shard_sparse(equil_matrix* M, eqb::DevCsr& fullA, eqb::DevCsr& fullT,
                  const std::vector<int64_t>& rpA_host,
                  const std::vector<int64_t>& rpT_host) {
  const int G = M->world, r = M->rank;
  M->a_bounds = G == 1 ? std::vector<int64_t>{0, M->m}
                       : partition_rows(rpA_host.data(), M->m, G);
  M->t_bounds = G == 1 ? std::vector<int64_t>{0, M->n}
                       : partition_rows(rpT_host.data(), M->n, G);
  M->a_max = 0;
  M->t_max = 0;
  for (int g = 0; g < G; ++g) {
    M->a_max = std::max(M->a_max, M->a_bounds[g + 1] - M->a_bounds[g]);
    M->t_max = std::max(M->t_max, M->t_bounds[g + 1] - M->t_bounds[g]);
  }
  M->a_bounds_d.alloc(G + 1);
  M->t_bounds_d.alloc(G + 1);
  h2d_sync(M->stream, M->a_bounds_d.p, M->a_bounds.data(), (G + 1) * 8);
  h2d_sync(M->stream, M->t_bounds_d.p, M->t_bounds.data(), (G + 1) * 8);

  auto take = [&](eqb::DevCsr& full, const std::vector<int64_t>& rph,
                  const std::vector<int64_t>& bounds, const std::vector<int64_t>& colb,
                  int64_t colmax, eqb::DevCsr& out, DevBuf<int64_t>& rp,
                  DevBuf<int32_t>& ci, DevBuf<double>& va) {
    const int64_t r0 = bounds[r], r1 = bounds[r + 1];
    const int64_t k0 = rph[r0], k1 = rph[r1];
    out.rows = r1 - r0;
    out.cols = full.cols;
    out.nnz = k1 - k0;
    rp.alloc(out.rows + 1);
    ci.alloc(out.nnz);
    va.alloc(out.nnz);
    rebase_rowptr_kernel<<<static_cast<unsigned>((out.rows + 1 + 255) / 256), 256, 0,
                           M->stream>>>(rp.p, full.row_ptr + r0, out.rows + 1, k0);
    CK(cudaGetLastError());
    if (out.nnz) {
      CK(cudaMemcpyAsync(ci.p, full.col + k0, out.nnz * 4, cudaMemcpyDeviceToDevice, M->stream));
      CK(cudaMemcpyAsync(va.p, full.val + k0, out.nnz * 8, cudaMemcpyDeviceToDevice, M->stream));
      if (G > 1) {
        DevBuf<int64_t> cb;
        cb.alloc(G + 1);
        h2d_sync(M->stream, cb.p, colb.data(), (G + 1) * 8);
        remap_cols_kernel<<<static_cast<unsigned>((out.nnz + 255) / 256), 256, 0,
                            M->stream>>>(ci.p, out.nnz, cb.p, G, colmax);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(M->stream));
      }
    }
    out.row_ptr = rp.p;
    out.col = ci.p;
    out.val = va.p;
  };
  take(fullA, rpA_host, M->a_bounds, M->t_bounds, M->t_max, M->A, M->a_rp, M->a_ci, M->a_va);
  take(fullT, rpT_host, M->t_bounds, M->a_bounds, M->a_max, M->AT, M->t_rp, M->t_ci, M->t_va);
  CK(cudaStreamSynchronize(M->stream));

  auto local_rp = [&](const std::vector<int64_t>& rph, const std::vector<int64_t>& b) {
    std::vector<int64_t> out(rph.begin() + b[r], rph.begin() + b[r + 1] + 1);
    const int64_t base = out[0];
    for (auto& x : out) x -= base;
    return out;
  };
  const std::vector<int64_t> la = local_rp(rpA_host, M->a_bounds);
  const std::vector<int64_t> lt = local_rp(rpT_host, M->t_bounds);
  upload_plans(M, plan_tiles(la.data(), static_cast<int64_t>(la.size()) - 1, 0),
               plan_tiles(lt.data(), static_cast<int64_t>(lt.size()) - 1, 1));
  build_block_layout(M);
  build_slot_layout(M, fullA.row_ptr, fullT.row_ptr);
  build_sell_layout(M, true);
}

// ---- rank collectives of the sharded setup ---------------------------------
// Every transport: NCCL (grouped send / receive, all-reduce) or the host
// exchange (one process per GPU over shared memory, or ranks as threads of one
// process; chunked through the exchange slots).

// Device all-to-all of bytes: send[soff[h], soff[h+1]) goes to rank h, and
// recv[roff[g], roff[g+1]) arrives from rank g.
void alltoallv_bytes(equil_matrix* M, const char* send, const std::vector<int64_t>& soff,
                     char* recv, const std::vector<int64_t>& roff) {
  const int G = M->world, r = M->rank;
  cudaStream_t s = M->stream;
  if (!M->hx) {
    nccl_check(nccl().GroupStart(), "ncclGroupStart");
    for (int h = 0; h < G; ++h) {
      const size_t sb = static_cast<size_t>(soff[h + 1] - soff[h]);
      const size_t rb = static_cast<size_t>(roff[h + 1] - roff[h]);
      if (h == r) {
        if (sb) CK(cudaMemcpyAsync(recv + roff[h], send + soff[h], sb, cudaMemcpyDeviceToDevice, s));
        continue;
      }
      if (sb) nccl_check(nccl().Send(send + soff[h], sb, ncclUint8, h, M->comm, s), "ncclSend");
      if (rb) nccl_check(nccl().Recv(recv + roff[h], rb, ncclUint8, h, M->comm, s), "ncclRecv");
    }
    nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
    CK(cudaStreamSynchronize(s));
    return;
  }
  // host exchange: every rank's whole send buffer passes through its slot in
  // chunks of the slot capacity; each rank copies out the part addressed to it
  CK(cudaStreamSynchronize(s));
  const size_t total = static_cast<size_t>(soff[G]);
  std::vector<char> host(total);
  if (total) CK(cudaMemcpy(host.data(), send, total, cudaMemcpyDeviceToHost));
  // everyone's send offsets (to find the piece addressed to this rank)
  const std::vector<char> offs =
      allgather_bytes(M, soff.data(), static_cast<size_t>(G + 1) * sizeof(int64_t));
  auto off_of = [&](int g, int h) {
    int64_t v;
    std::memcpy(&v, offs.data() + (static_cast<size_t>(g) * (G + 1) + h) * sizeof(int64_t), 8);
    return v;
  };
  const size_t cap = std::min<size_t>(M->hx->capacity(), size_t(1) << 30);
  int64_t maxtot = 0;
  for (int g = 0; g < G; ++g) maxtot = std::max(maxtot, off_of(g, G));
  const int64_t rounds = (maxtot + static_cast<int64_t>(cap) - 1) / static_cast<int64_t>(cap);
  std::vector<char> mine(static_cast<size_t>(roff[G]));
  for (int64_t c = 0; c < rounds; ++c) {
    const int64_t lo = c * static_cast<int64_t>(cap);
    const int64_t hi = std::min<int64_t>(lo + static_cast<int64_t>(cap), static_cast<int64_t>(total));
    M->hx->put(r, host.data() + std::min<int64_t>(lo, total), hi > lo ? static_cast<size_t>(hi - lo) : 0);
    M->hx->barrier();
    for (int g = 0; g < G; ++g) {
      const int64_t a = std::max(off_of(g, r), lo);
      const int64_t b = std::min(off_of(g, r + 1), lo + static_cast<int64_t>(cap));
      if (b > a)
        std::memcpy(mine.data() + roff[g] + (a - off_of(g, r)), M->hx->slot(g) + (a - lo),
                    static_cast<size_t>(b - a));
    }
    M->hx->barrier();
  }
  h2d_sync(s, recv, mine.data(), static_cast<size_t>(roff[G]));
}

// In-place sum of an int64 device array over the ranks.
void allreduce_sum_i64(equil_matrix* M, int64_t* dev, int64_t count) {
  cudaStream_t s = M->stream;
  if (!M->hx) {
    nccl_check(nccl().AllReduce(dev, dev, static_cast<size_t>(count), ncclInt64, ncclSum, M->comm, s),
               "ncclAllReduce");
    CK(cudaStreamSynchronize(s));
    return;
  }
  CK(cudaStreamSynchronize(s));
  const size_t bytes = static_cast<size_t>(count) * 8;
  const size_t cap = std::min<size_t>(M->hx->capacity(), size_t(1) << 30) / 8 * 8;
  std::vector<int64_t> mine(static_cast<size_t>(count)), sum(static_cast<size_t>(count), 0);
  CK(cudaMemcpy(mine.data(), dev, bytes, cudaMemcpyDeviceToHost));
  for (size_t lo = 0; lo < bytes; lo += cap) {
    const size_t len = std::min(cap, bytes - lo);
    M->hx->put(M->rank, reinterpret_cast<const char*>(mine.data()) + lo, len);
    M->hx->barrier();
    for (int g = 0; g < M->world; ++g) {
      const int64_t* p = reinterpret_cast<const int64_t*>(M->hx->slot(g));
      for (size_t k = 0; k < len / 8; ++k) sum[lo / 8 + k] += p[k];
    }
    M->hx->barrier();
  }
  h2d_sync(s, dev, sum.data(), bytes);
}

// ExplicitMatrix::sparse's message for the first invalid entry (class, global
// entry index), in the reference's order of checks (explicit_matrix.cpp:21-39)
[[noreturn]] void fail_invalid_entry(unsigned long long wh, const int64_t* row_ptr, int64_t m,
                                     const int32_t* col) {
  const int cls = static_cast<int>(wh >> 40);
  const int64_t k = static_cast<int64_t>(wh & ((1ULL << 40) - 1));
  const int64_t i = std::upper_bound(row_ptr, row_ptr + m + 1, k) - row_ptr - 1;
  const std::string at = "(" + std::to_string(i) + ", " + std::to_string(col[k]) + ")";
  if (cls == 0) fail(EQUIL_EINVAL, "ExplicitMatrix::sparse: entry " + at + " out of range");
  if (cls == 1) fail(EQUIL_EINVAL, "ExplicitMatrix::sparse: duplicate entry " + at);
  fail(EQUIL_EINVAL, "ExplicitMatrix::sparse: columns not ascending at entry " + at +
                         " (canonical CSR required)");
}

// Sharded setup (world > 1).  Rank r uploads only its rows [a0, a1) of A,
// validates them (the first error over all ranks wins, so every rank throws
// the single-GPU message), and transposes them locally.  CSR(A^T)'s global
// row pointers are the sum of the ranks' local prefix sums (one all-reduce),
// which fixes the A^T partition.  An all-to-all then sends every rank the rows
// of its A^T range from every other rank's local transpose (counts, columns,
// values), and a merge lays them out in rank order -- ascending original row,
// CSR(A^T)'s own order -- so the shards equal those cut from the full
// transpose, bit for bit, with 1/world of the upload and transpose work.
void create_sharded(equil_matrix* M, const int64_t* row_ptr, const int32_t* col,
                    const double* val, PhaseTimer& pt) {
  const int G = M->world, r = M->rank;
  const int64_t m = M->m, n = M->n;
  cudaStream_t s = M->stream;
  M->a_bounds = partition_rows(row_ptr, m, G);
  const int64_t a0 = M->a_bounds[r], a1 = M->a_bounds[r + 1];
  const int64_t k0 = row_ptr[a0], k1 = row_ptr[a1];
  const int64_t ml = a1 - a0, nl = k1 - k0;
  // this rank's rows of A (row pointers rebased) and the global row pointers
  // (the slot layout of the gathered vectors needs every row's length)
  DevBuf<int64_t> rpA_full;
  rpA_full.alloc(m + 1);
  CK(cudaMemcpyAsync(rpA_full.p, row_ptr, (m + 1) * 8, cudaMemcpyHostToDevice, s));
  std::vector<int64_t> rph(static_cast<size_t>(ml) + 1);
  for (int64_t i = 0; i <= ml; ++i) rph[i] = row_ptr[a0 + i] - k0;
  M->a_rp.alloc(ml + 1);
  M->a_ci.alloc(nl);
  M->a_va.alloc(nl);
  CK(cudaMemcpyAsync(M->a_rp.p, rph.data(), (ml + 1) * 8, cudaMemcpyHostToDevice, s));
  if (nl) {
    CK(cudaMemcpyAsync(M->a_ci.p, col + k0, nl * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(M->a_va.p, val + k0, nl * 8, cudaMemcpyHostToDevice, s));
  }
  eqb::DevCsr locA{ml, n, nl, M->a_rp.p, M->a_ci.p, M->a_va.p};
  pt.mark(s, "upload (shard)");
  // validation of the local rows; the smallest (class, global entry) over ranks
  DevBuf<unsigned long long> where;
  where.alloc(1);
  CK(cudaMemsetAsync(M->flags.p, 0, sizeof(unsigned), s));
  CK(cudaMemsetAsync(where.p, 0xff, 8, s));
  CK(eqb::launch_validate_csr(locA, reinterpret_cast<int*>(M->flags.p), where.p, s));
  unsigned long long wh = ~0ULL;
  CK(cudaMemcpyAsync(&wh, where.p, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (wh != ~0ULL) wh += static_cast<unsigned long long>(k0);  // class bits untouched
  {
    const std::vector<char> all = allgather_bytes(M, &wh, 8);
    for (int g = 0; g < G; ++g) {
      unsigned long long o;
      std::memcpy(&o, all.data() + 8 * g, 8);
      wh = std::min(wh, o);
    }
  }
  if (wh != ~0ULL) fail_invalid_entry(wh, row_ptr, m, col);
  pt.mark(s, "validate (shard)");
  // local transpose: n rows (A's columns) x ml (this rank's rows of A)
  DevBuf<int64_t> trl;
  DevBuf<int32_t> tcl;
  DevBuf<double> tvl;
  trl.alloc(n + 1);
  tcl.alloc(nl);
  tvl.alloc(nl);
  CK(eqb::launch_col_rowptr(M->a_ci.p, nl, n, trl.p, s));
  std::vector<int64_t> trl_h(static_cast<size_t>(n) + 1);
  CK(cudaMemcpyAsync(trl_h.data(), trl.p, (n + 1) * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  eqb::DevCsr locT{n, ml, nl, trl.p, tcl.p, tvl.p};
  {
    eqb::TransposeWork tw;
    CK(eqb::transpose_structure(locA, locT, trl_h.data(), tw, s));
    CK(eqb::transpose_values(locA, locT, tw, s));
    CK(cudaStreamSynchronize(s));
  }
  pt.mark(s, "transpose (shard)");
  // CSR(A^T)'s global row pointers: the sum of the local prefix sums
  DevBuf<int64_t> rpT_full;
  rpT_full.alloc(n + 1);
  CK(cudaMemcpyAsync(rpT_full.p, trl.p, (n + 1) * 8, cudaMemcpyDeviceToDevice, s));
  allreduce_sum_i64(M, rpT_full.p, n + 1);
  std::vector<int64_t> rpT(static_cast<size_t>(n) + 1);
  CK(cudaMemcpy(rpT.data(), rpT_full.p, (n + 1) * 8, cudaMemcpyDeviceToHost));
  M->t_bounds = partition_rows(rpT.data(), n, G);
  M->a_max = 0;
  M->t_max = 0;
  for (int g = 0; g < G; ++g) {
    M->a_max = std::max(M->a_max, M->a_bounds[g + 1] - M->a_bounds[g]);
    M->t_max = std::max(M->t_max, M->t_bounds[g + 1] - M->t_bounds[g]);
  }
  M->a_bounds_d.alloc(G + 1);
  M->t_bounds_d.alloc(G + 1);
  h2d_sync(M->stream, M->a_bounds_d.p, M->a_bounds.data(), (G + 1) * 8);
  h2d_sync(M->stream, M->t_bounds_d.p, M->t_bounds.data(), (G + 1) * 8);
  // A^T's columns are A's rows: local row -> this rank's padded slot range
  if (nl)
    add_cols_kernel<<<static_cast<unsigned>((nl + 255) / 256), 256, 0, s>>>(tcl.p, nl,
                                                                        r * M->a_max);
  // A's columns are A^T's rows: global column -> padded slot
  if (nl)
    remap_cols_kernel<<<static_cast<unsigned>((nl + 255) / 256), 256, 0, s>>>(
        M->a_ci.p, nl, M->t_bounds_d.p, G, M->t_max);
  CK(cudaGetLastError());
  // all-to-all: rank h gets rows [t_bounds[h], t_bounds[h+1]) of every local
  // transpose -- first each row's count, then the columns and the values
  const int64_t t0 = M->t_bounds[r], t1 = M->t_bounds[r + 1], tl = t1 - t0;
  DevBuf<int32_t> cnt_all;
  cnt_all.alloc(n);
  row_counts_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(trl.p, n, cnt_all.p);
  CK(cudaGetLastError());
  std::vector<int64_t> so(G + 1), ro(G + 1);
  for (int h = 0; h <= G; ++h) so[h] = M->t_bounds[h] * 4;
  for (int g = 0; g <= G; ++g) ro[g] = static_cast<int64_t>(g) * tl * 4;
  DevBuf<int32_t> cnt_in;
  cnt_in.alloc(static_cast<size_t>(G) * tl);
  CK(cudaStreamSynchronize(s));
  alltoallv_bytes(M, reinterpret_cast<const char*>(cnt_all.p), so,
                  reinterpret_cast<char*>(cnt_in.p), ro);
  // entry offsets: what this rank sends to h, and (counts summed) what it gets
  std::vector<int32_t> cin(static_cast<size_t>(G) * tl);
  if (!cin.empty())
    CK(cudaMemcpy(cin.data(), cnt_in.p, cin.size() * 4, cudaMemcpyDeviceToHost));
  std::vector<int64_t> se(G + 1), re(G + 1, 0);
  for (int h = 0; h <= G; ++h) se[h] = trl_h[M->t_bounds[h]];
  for (int g = 0; g < G; ++g) {
    int64_t c = 0;
    for (int64_t j = 0; j < tl; ++j) c += cin[static_cast<size_t>(g) * tl + j];
    re[g + 1] = re[g] + c;
  }
  const int64_t nt = re[G];  // this rank's entries of A^T
  require(nt == rpT[t1] - rpT[t0], "sharded setup: A^T entry count mismatch");
  DevBuf<int32_t> ci_in;
  DevBuf<double> va_in;
  ci_in.alloc(nt);
  va_in.alloc(nt);
  {
    std::vector<int64_t> sb(G + 1), rb(G + 1);
    for (int h = 0; h <= G; ++h) sb[h] = se[h] * 4, rb[h] = re[h] * 4;
    alltoallv_bytes(M, reinterpret_cast<const char*>(tcl.p), sb,
                    reinterpret_cast<char*>(ci_in.p), rb);
    for (int h = 0; h <= G; ++h) sb[h] = se[h] * 8, rb[h] = re[h] * 8;
    alltoallv_bytes(M, reinterpret_cast<const char*>(tvl.p), sb,
                    reinterpret_cast<char*>(va_in.p), rb);
  }
  pt.mark(s, "all-to-all");
  // merge: row j of the shard = the runs of sources 0, 1, ..., G-1 in order
  std::vector<int64_t> src_off(static_cast<size_t>(G) * tl), dst_off(src_off.size());
  {
    std::vector<int64_t> pos(static_cast<size_t>(tl));
    for (int64_t j = 0; j < tl; ++j) pos[j] = rpT[t0 + j] - rpT[t0];
    for (int g = 0; g < G; ++g) {
      int64_t sp = re[g];
      for (int64_t j = 0; j < tl; ++j) {
        const size_t q = static_cast<size_t>(g) * tl + j;
        src_off[q] = sp;
        dst_off[q] = pos[j];
        sp += cin[q];
        pos[j] += cin[q];
      }
    }
  }
  DevBuf<int64_t> so_d, do_d;
  so_d.alloc(src_off.size());
  do_d.alloc(dst_off.size());
  M->t_rp.alloc(tl + 1);
  M->t_ci.alloc(nt);
  M->t_va.alloc(nt);
  std::vector<int64_t> trp(static_cast<size_t>(tl) + 1);
  for (int64_t j = 0; j <= tl; ++j) trp[j] = rpT[t0 + j] - rpT[t0];
  CK(cudaMemcpyAsync(M->t_rp.p, trp.data(), (tl + 1) * 8, cudaMemcpyHostToDevice, s));
  if (!src_off.empty()) {
    CK(cudaMemcpyAsync(so_d.p, src_off.data(), src_off.size() * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(do_d.p, dst_off.data(), dst_off.size() * 8, cudaMemcpyHostToDevice, s));
    const int64_t runs = static_cast<int64_t>(src_off.size());
    merge_runs_kernel<<<static_cast<unsigned>((runs * 8 + 255) / 256), 256, 0, s>>>(
        so_d.p, do_d.p, cnt_in.p, runs, ci_in.p, va_in.p, M->t_ci.p, M->t_va.p);
    CK(cudaGetLastError());
  }
  CK(cudaStreamSynchronize(s));
  pt.mark(s, "merge");
  M->A = {ml, n, nl, M->a_rp.p, M->a_ci.p, M->a_va.p};
  M->AT = {tl, m, nt, M->t_rp.p, M->t_ci.p, M->t_va.p};
  const std::vector<int64_t>& la = rph;
  upload_plans(M, plan_tiles(la.data(), ml, 0), plan_tiles(trp.data(), tl, 1));
  build_block_layout(M);
  build_slot_layout(M, rpA_full.p, rpT_full.p);
  build_sell_layout(M, true);
  CK(cudaStreamSynchronize(s));
  pt.mark(s, "plan");
}

void alloc_workspaces(equil_matrix* M, PhaseTimer* pt = nullptr);

// From a validated device CSR(A) (ownership taken) and its host row_ptr: build
// CSR(A^T) on device (K2), plan the traversal (planA may already be running on
// `planner`), shard for world_size > 1, allocate workspaces.
void finish_sparse(equil_matrix* M, DevBuf<int64_t>& rp, DevBuf<int32_t>& ci,
                   DevBuf<double>& va, const int64_t* row_ptr, PhaseTimer& pt, Plan* planA,
                   std::thread* planner) {
  const int64_t m = M->m, n = M->n, nnz = M->nnz;
  cudaStream_t s = M->stream;
  eqb::DevCsr fullA{m, n, nnz, rp.p, ci.p, va.p};
  DevBuf<int64_t> trp;
  DevBuf<int32_t> tci;
  DevBuf<double> tva;
  trp.alloc(n + 1);
  tci.alloc(nnz);
  tva.alloc(nnz);
  eqb::DevCsr fullT{n, m, nnz, trp.p, tci.p, tva.p};
  // CSR(A^T)'s row pointers first (column counts), so the host can plan the
  // A^T traversal while the device transposes
  std::vector<int64_t> rpT(n + 1);
  CK(eqb::launch_col_rowptr(ci.p, nnz, n, trp.p, s));
  CK(cudaMemcpyAsync(rpT.data(), trp.p, (n + 1) * 8, cudaMemcpyDeviceToHost, s));
  cudaEvent_t ev_rp = nullptr;
  CK(cudaEventCreateWithFlags(&ev_rp, cudaEventDisableTiming));
  struct EvGuard {
    cudaEvent_t e;
    ~EvGuard() { cudaEventDestroy(e); }
  } evg{ev_rp};
  CK(cudaEventRecord(ev_rp, s));
  Plan planT;
  std::thread tplanner;
  struct Joiner {
    std::thread& t;
    ~Joiner() {
      if (t.joinable()) t.join();
    }
  } tj{tplanner};
  if (M->world == 1)
    tplanner = std::thread([&] {
      if (cudaEventSynchronize(ev_rp) != cudaSuccess) return;
      const auto t0 = std::chrono::steady_clock::now();
      planT = plan_tiles(rpT.data(), n, 1);
      if (pt.mode == 2)
        fprintf(stderr, "[equil] plan_tiles(A^T) %.2f ms\n",
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    });
  // K2's structure needs only the columns (and CSR(A^T)'s row pointers, which
  // the partition plan reads on the host); A's values may still be uploading
  CK(cudaEventSynchronize(ev_rp));
  // until the values have arrived, uploads must not queue behind them on the
  // copy engine: plans go up through pull kernels
  struct PullScope {
    equil_matrix* M;
    explicit PullScope(equil_matrix* m) : M(m) {
      pull_arena_reset();
      M->pull_uploads = M->world == 1;
    }
    ~PullScope() {
      M->pull_uploads = false;
      cudaStreamSynchronize(M->stream);  // nothing may still read the arena
    }
  } pull_scope(M);
  eqb::TransposeWork tw;
  CK(eqb::transpose_structure(fullA, fullT, rpT.data(), tw, s,
                              [M](void* d, const void* h, size_t b) { h2d(M, d, h, b); }));
  pt.mark(s, "transpose");
  // everything below until the values step reads only row pointers and columns
  auto values_arrived = [&] {
    CK(cudaStreamWaitEvent(s, M->ev_vals, 0));  // every later use of A's values
    CK(eqb::transpose_values(fullA, fullT, tw, s));
    M->pull_uploads = false;
    pt.mark(s, "values");
  };
  if (M->world == 1) {
    // adopt the full arrays as the shard (no copy)
    M->a_bounds = {0, m};
    M->t_bounds = {0, n};
    M->a_max = m;
    M->t_max = n;
    M->a_rp.swap(rp);
    M->a_ci.swap(ci);
    M->a_va.swap(va);
    M->t_rp.swap(trp);
    M->t_ci.swap(tci);
    M->t_va.swap(tva);
    M->A = {m, n, nnz, M->a_rp.p, M->a_ci.p, M->a_va.p};
    M->AT = {n, m, nnz, M->t_rp.p, M->t_ci.p, M->t_va.p};
    fullA = M->A;
    fullT = M->AT;
    build_block_layout(M);
    // column sweep of A's long rows (sweep.cu): decided here because it wants xs
    // in column order (identity slot map); needs long rows in A, one GPU, no
    // column blocks, and an even n (16-byte aligned panels of both xs buffers)
    M->sweep_candidate = false;
    if (M->use_sweep && M->use_sell && M->use_slots && M->sell_long == 2 && M->split_epi &&
        M->nblk[0] <= 1 && M->nblk[1] <= 1 && (n & 1) == 0)
    {
      for (int64_t i = 0; i < m && !M->sweep_candidate; ++i)
        M->sweep_candidate = row_ptr[i + 1] - row_ptr[i] > eqb::kTileNnz;
      // long rows in A^T need the long-slice kernel, and then the sweep stands down
      // (plan_sweep_layout): keep the hot-first layout of xs for such matrices
      for (int64_t j = 0; j < n && M->sweep_candidate; ++j)
        if (rpT[j + 1] - rpT[j] > eqb::kTileNnz) M->sweep_candidate = false;
    }
    build_slot_layout(M, M->A.row_ptr, M->AT.row_ptr);  // device work
    if (tplanner.joinable()) tplanner.join();  // planned during the transpose
    pt.mark(s, "plan A^T");
    if (planner && planner->joinable()) planner->join();
    pt.mark(s, "plan A (join)");
    if (planA)  // computed concurrently by the caller
      upload_plans(M, *planA, planT);
    else
      upload_plans(M, plan_tiles(row_ptr, m, 0), planT);
    pt.mark(s, "upload plans");
    // values are needed from here on only by the blocked layouts
    const bool late_values = M->nblk[0] <= 1 && M->nblk[1] <= 1;
    if (!late_values) values_arrived();
    plan_sweep_layout(M);  // (its kernels run ahead of the interleaved layout's)
    build_sell_layout(M, !late_values);
    build_sweep_layout(M, !late_values);
    pt.mark(s, "sell");
    if (late_values) {
      values_arrived();
      build_sell_values(M);
      build_sweep_values(M);
      pt.mark(s, "sell values");
    }
  } else {
    values_arrived();
    const std::vector<int64_t> rpA(row_ptr, row_ptr + m + 1);
    shard_sparse(M, fullA, fullT, rpA, rpT);
  }
  pt.mark(s, "plan");
  alloc_workspaces(M, &pt);
  CK(cudaStreamSynchronize(s));
  pt.mark(s, "workspaces");
}

// L2 access-policy window of stream st: [base, base + bytes) persisting (as much
// of it as the carve-out holds), or with bytes == 0 the handle's default
// (base == xbuf: the gathered vectors; nullptr: none).
void set_l2_window(equil_matrix* M, cudaStream_t st, const void* base, size_t bytes) {
  if (M->l2_carve == 0) return;
  cudaStreamAttrValue attr{};
  if (bytes == 0 && base) {
    bytes = M->l2_default_bytes;
  }
  if (base && bytes) {
    const size_t win = std::min(bytes, M->l2_max_window);
    attr.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    attr.accessPolicyWindow.num_bytes = win;
    attr.accessPolicyWindow.hitRatio =
        static_cast<float>(std::min(1.0, static_cast<double>(M->l2_carve) / win));
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  }
  cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &attr);
  cudaGetLastError();  // a hint; never fail on it
}

void alloc_workspaces(equil_matrix* M, PhaseTimer* pt) {
  // each vector padded to whole 32 KB granules (aligned bases for every copy)
  auto whole = [](int64_t x) { return (x + 4095) / 4096 * 4096; };
  const int64_t np = whole(M->n_pad()), mp = whole(M->m_pad());
  // the gathered vectors, then the device barrier words (fused all-gather)
  const int64_t xlen = 2 * (np + mp) + eqb::kBarWords;
  M->xbar_off = 2 * (np + mp);
  if (M->world > 1 && !(M->hx && M->hx->in_process())) {
    // pool memory cannot be exported over CUDA IPC
    double* q = nullptr;
    CK(cudaMalloc(&q, xlen * sizeof(double)));
    M->xbuf.adopt(q, xlen);
  } else {
    M->xbuf.alloc(xlen);
  }
  CK(cudaMemset(M->xbuf.p, 0, xlen * sizeof(double)));
  if (pt) pt->mark(M->stream, "xbuf");
  for (int b = 0; b < 2; ++b) {
    M->xs[b].p = M->xbuf.p + b * np;
    M->xw[b].p = M->xbuf.p + 2 * np + b * mp;
  }
  // Keep the gather targets resident in L2 while CSR(A)/CSR(A^T) stream past;
  // dense: keep A itself (c2: 67 MB, read twice per iteration) persisting.
  int dev = 0, max_persist = 0, max_window = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
  cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
  const void* wbase = M->dense ? static_cast<const void*>(M->Ad.p) : M->xbuf.p;
  const size_t bytes = M->dense ? static_cast<size_t>(M->m * M->n) * sizeof(double)
                                : static_cast<size_t>(2 * (np + mp)) * sizeof(double);
  static const bool l2win = !getenv("EQUIL_L2WIN") || atoi(getenv("EQUIL_L2WIN")) != 0;
  if (l2win && max_persist > 0 && max_window > 0 && bytes > 0) {
    const size_t win = std::min(bytes, static_cast<size_t>(max_window));
    const size_t carve = std::min(win, static_cast<size_t>(max_persist));
    M->l2_max_window = static_cast<size_t>(max_window);
    M->l2_default_bytes = bytes;
    // the limit is device-wide and setting it is slow (~2 ms): only when it changes
    size_t cur = 0;
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    if (cur == carve || cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve) == cudaSuccess) {
      M->l2_carve = carve;
      cudaStreamAttrValue attr{};
      attr.accessPolicyWindow.base_ptr = const_cast<void*>(wbase);
      attr.accessPolicyWindow.num_bytes = win;
      attr.accessPolicyWindow.hitRatio =
          static_cast<float>(std::min(1.0, static_cast<double>(carve) / win));
      attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(M->stream, cudaStreamAttributeAccessPolicyWindow, &attr);
      if (M->dense)  // the column half runs on the copy stream
        cudaStreamSetAttribute(M->copy_stream, cudaStreamAttributeAccessPolicyWindow, &attr);
    }
    cudaGetLastError();  // the window is a hint; never fail on it
  }
  if (pt) pt->mark(M->stream, "l2 window");
  M->rowacc.alloc(M->m_loc() + M->n_loc());
  M->u.alloc(M->m_loc());
  M->ub.alloc(M->m_loc());
  M->v.alloc(M->n_loc());
  M->vb.alloc(M->n_loc());
  // the longest canonical reduction runs over m + n terms (the history's RMS
  // spread, equil_rms_error); padded vectors are at most m_pad / n_pad long
  const int64_t big = std::max(M->m_pad() + M->n_pad(), M->m + M->n);
  M->red_part.alloc((big + eqb::kChunk - 1) / eqb::kChunk + 1);
  M->tmp_m.alloc(M->m_pad());
  M->tmp_n.alloc(M->n_pad());
  M->tmp_m2.alloc(M->m_pad());
  M->tmp_n2.alloc(M->n_pad());
  if (M->dense) {
    M->colpart.alloc(((M->m + eqb::kChunk - 1) / eqb::kChunk) * M->n);
    M->colcnt.alloc((M->n + 15) / 16);
    CK(cudaMemsetAsync(M->colcnt.p, 0, ((M->n + 15) / 16) * sizeof(unsigned), M->stream));
    CK(cudaStreamSynchronize(M->stream));
  }
}

}  // namespace eqe

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* equil_last_error(void) { return g_err.c_str(); }
const char* equil_version(void) { return "equil_b200 0.1 (sm_100a)"; }

void equil_params_default(equil_params* p) {
  p->alpha = 0.0;
  p->beta = 0.0;
  p->gamma = 0.1;
  p->max_log_scale = 9.210340371976184;
  p->iterations = 1000;
  p->seed = 0;
}

equil_status equil_resolve_targets(const equil_params* p, int64_t rows, int64_t cols,
                                   double* alpha, double* beta) {
  return guarded([&] {
    require(p != nullptr, "resolve_targets: null params");
    resolve_targets(*p, rows, cols, *alpha, *beta);
  });
}

equil_status equil_validate_params(const equil_params* p) {
  return guarded([&] {
    require(p != nullptr, "validate_params: null params");
    validate_params(*p);
  });
}

double equil_det_exp_host(double x) { return eqb::det_exp(x); }

equil_status equil_partition_rows(const int64_t* row_ptr, int64_t rows, int parts,
                                  int64_t* bounds) {
  return guarded([&] {
    require(parts > 0 && rows >= 0, "partition_rows: bad arguments");
    const auto b = partition_rows(row_ptr, rows, parts);
    std::copy(b.begin(), b.end(), bounds);
  });
}

equil_status equil_nccl_unique_id(void* out128) {
  return guarded([&] {
    if (!nccl().ok) fail(EQUIL_ENCCL, "libnccl.so.2 could not be loaded");
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof id);
  });
}

}  // extern "C"

namespace eqe {
struct PreSigns {
  uint64_t seed, total;
};
}  // namespace eqe

static equil_status create_csr_impl(int64_t m, int64_t n, const int64_t* row_ptr,
                                    const int32_t* col, const double* val,
                                    const equil_device_cfg* cfg, equil_matrix** out,
                                    const eqe::PreSigns* pre) {
  return guarded([&] {
    NvtxRange nvtx_("equil:create_csr");
    require(out != nullptr, "ExplicitMatrix::sparse: null output handle");
    *out = nullptr;
    require(m > 0 && n > 0, "ExplicitMatrix::sparse: dimensions must be positive");
    require(row_ptr != nullptr, "ExplicitMatrix::sparse: null row_ptr");
    require(n < (1LL << 31) && m < (1LL << 31), "ExplicitMatrix::sparse: dimension too large");
    const int64_t nnz = row_ptr[m];
    require(nnz >= 0 && nnz < (1LL << 31), "ExplicitMatrix::sparse: bad nnz");
    // row_ptr is checked on the host before anything reads the arrays by it; the
    // O(m) monotonicity scan runs below, once the uploads (which need only nnz)
    // are on their way
    require(row_ptr[0] == 0, "ExplicitMatrix::sparse: row_ptr[0] must be 0");
    auto check_monotone = [&] {
      for (int64_t i = 0; i < m; ++i)
        if (row_ptr[i + 1] < row_ptr[i])
          fail(EQUIL_EINVAL,
               "ExplicitMatrix::sparse: row_ptr decreases at row " + std::to_string(i));
    };
    require(nnz == 0 || (col && val), "ExplicitMatrix::sparse: null col/val");
    // the scan runs on a helper thread from here; its verdict is taken before
    // anything reads the arrays by row_ptr, and it outranks a device error
    // (on a box without a GPU a bad row_ptr is still reported as such)
    std::future<void> mono = std::async(std::launch::async, check_monotone);
    struct MonoJoin {
      std::future<void>& f;
      ~MonoJoin() {
        if (f.valid()) {
          try {
            f.get();
          } catch (...) {
          }
        }
      }
    } mono_join{mono};
    auto mono_get = [&] {
      if (mono.valid()) mono.get();
    };
    PhaseTimer pt("create_csr");
    auto M = std::make_unique<equil_matrix>();
    try {
      setup_common(M.get(), cfg);
    } catch (...) {
      mono_get();
      throw;
    }
    M->m = m;
    M->n = n;
    M->nnz = nnz;
    DeviceGuard dg(M->device);
    cudaStream_t s = M->stream;
    // The sweep layout adds ~4 ms to a pipelined c3 setup and saves ~0.09 ms per
    // iteration: a one-shot call of few iterations keeps the long-slice kernel
    M->oneshot_hint = pre != nullptr;  // the handle serves one SGD call and is destroyed
    if (pre && pre->total > 0 && !M->sweep_forced &&
        pre->total / static_cast<uint64_t>(m + n) < 64)
      M->use_sweep = false;
    if (pre && pre->total > 0) {  // overlaps the uploads and the transpose below
      M->signs.ensure((pre->total + 31) / 32 + 1);
      const size_t sb = eqb::sign_stream_scratch_bytes(pre->total);
      M->sign_scratch.ensure(sb);
      CK(eqb::sign_stream_generate(pre->seed, 17, pre->total, M->signs.p, M->sign_scratch.p, sb,
                                   M->sign_stream));
      CK(cudaEventRecord(M->sign_ev, M->sign_stream));
      M->pre_signs = true;
      M->pre_seed = pre->seed;
      M->pre_total = pre->total;
    }
    pt.mark(s, "setup");
    if (M->world > 1) {  // each rank uploads and transposes only its rows
      mono_get();
      create_sharded(M.get(), row_ptr, col, val, pt);
      alloc_workspaces(M.get(), &pt);
      CK(cudaStreamSynchronize(s));
      *out = M.release();
      return;
    }
    // full A on device (uploaded once)
    DevBuf<int64_t> rp;
    DevBuf<int32_t> ci;
    DevBuf<double> va;
    rp.alloc(m + 1);
    ci.alloc(nnz);
    va.alloc(nnz);
    // row pointers and columns first: validation and the transpose sort need
    // only those, and run while the values are still crossing PCIe
    CK(cudaMemcpyAsync(rp.p, row_ptr, (m + 1) * 8, cudaMemcpyHostToDevice, s));
    if (nnz) {
      CK(cudaMemcpyAsync(ci.p, col, nnz * 4, cudaMemcpyHostToDevice, s));
      CK(cudaEventRecord(M->ev_vals, s));  // values follow the columns on the copy stream
      CK(cudaStreamWaitEvent(M->copy_stream, M->ev_vals, 0));
      CK(cudaMemcpyAsync(va.p, val, nnz * 8, cudaMemcpyHostToDevice, M->copy_stream));
      CK(cudaEventRecord(M->ev_vals, M->copy_stream));
      if (pt.mode == 2) pt.mark(M->copy_stream, "values in");
    } else {
      CK(cudaEventRecord(M->ev_vals, s));
    }
    mono_get();  // (the copies are running; nothing has read the arrays by row_ptr yet)
    eqb::DevCsr fullA{m, n, nnz, rp.p, ci.p, va.p};
    // plan CSR(A) on the host while the device validates and transposes
    Plan planA;
    std::thread planner;
    struct Joiner {
      std::thread& t;
      ~Joiner() {
        if (t.joinable()) t.join();
      }
    } joiner{planner};
    if (M->world == 1)
      planner = std::thread([&] {
        const auto t0 = std::chrono::steady_clock::now();
        planA = plan_tiles(row_ptr, m, 0);
        if (pt.mode == 2)
          fprintf(stderr, "[equil] plan_tiles(A) %.2f ms\n",
                  std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
      });
    pt.mark(s, "upload");
    // validation (explicit_matrix.cpp:21-39 for canonical CSR); the deterministic
    // first error: out of range, then duplicate, then unsorted columns
    DevBuf<unsigned long long> where;
    where.alloc(1);
    CK(cudaMemsetAsync(M->flags.p, 0, sizeof(unsigned), s));
    CK(cudaMemsetAsync(where.p, 0xff, 8, s));
    CK(eqb::launch_validate_csr(fullA, reinterpret_cast<int*>(M->flags.p), where.p, s));
    unsigned long long wh = ~0ULL;
    CK(cudaMemcpyAsync(&wh, where.p, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    pt.mark(s, "validate");
    if (wh != ~0ULL) fail_invalid_entry(wh, row_ptr, m, col);
    finish_sparse(M.get(), rp, ci, va, row_ptr, pt, &planA, &planner);
    *out = M.release();
  });
}

extern "C" {

equil_status equil_matrix_create_csr(int64_t m, int64_t n, const int64_t* row_ptr,
                                     const int32_t* col, const double* val,
                                     const equil_device_cfg* cfg, equil_matrix** out) {
  return create_csr_impl(m, n, row_ptr, col, val, cfg, out, nullptr);
}

}  // extern "C"

namespace eqe {
// ExplicitMatrix::sparse on the device.  With `lines` (Matrix Market ingest)
// a duplicate is reported the way read_matrix_market does
// (src/matrix_market.cpp:142-158): at the line of the later occurrence.
void create_coo_impl(int64_t m, int64_t n, int64_t nnz, const int64_t* rows,
                     const int64_t* cols, const double* vals, const int64_t* lines,
                     const equil_device_cfg* cfg, equil_matrix** out) {
  {
    require(out != nullptr, "ExplicitMatrix::sparse: null output handle");
    *out = nullptr;
    require(m > 0 && n > 0, "ExplicitMatrix::sparse: dimensions must be positive");
    require(n < (1LL << 31) && m < (1LL << 31), "ExplicitMatrix::sparse: dimension too large");
    require(nnz >= 0 && nnz < (1LL << 31), "ExplicitMatrix::sparse: bad nnz");
    require(nnz == 0 || (rows && cols && vals), "ExplicitMatrix::sparse: null entries");
    PhaseTimer pt("create_coo");
    auto M = std::make_unique<equil_matrix>();
    setup_common(M.get(), cfg);
    M->m = m;
    M->n = n;
    M->nnz = nnz;
    DeviceGuard dg(M->device);
    cudaStream_t s = M->stream;
    DevBuf<int64_t> dr, dc, rp;
    DevBuf<double> dv, va;
    DevBuf<int32_t> ci;
    dr.alloc(nnz);
    dc.alloc(nnz);
    dv.alloc(nnz);
    rp.alloc(m + 1);
    ci.alloc(nnz);
    va.alloc(nnz);
    if (nnz) {
      CK(cudaMemcpyAsync(dr.p, rows, nnz * 8, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(dc.p, cols, nnz * 8, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(dv.p, vals, nnz * 8, cudaMemcpyHostToDevice, s));
    }
    eqb::DevCsr A{m, n, nnz, rp.p, ci.p, va.p};
    unsigned long long bad = 0;
    int kind = 0;
    CK(eqb::coo_to_csr(m, n, nnz, dr.p, dc.p, dv.p, A, &bad, &kind, s));
    if (kind == 1)  // explicit_matrix.cpp:23-27
      fail(EQUIL_EINVAL, "ExplicitMatrix::sparse: entry (" + std::to_string(rows[bad]) + ", " +
                             std::to_string(cols[bad]) + ") out of range");
    if (kind == 2 && lines) {  // matrix_market.cpp:142-158
      const int64_t r = static_cast<int64_t>(bad / static_cast<uint64_t>(n));
      const int64_t c = static_cast<int64_t>(bad % static_cast<uint64_t>(n));
      int seen = 0;
      int64_t line = 0;
      for (int64_t k = 0; k < nnz && seen < 2; ++k)
        if (rows[k] == r && cols[k] == c && ++seen == 2) line = lines[k];
      throw std::runtime_error("matrix market: line " + std::to_string(line) +
                               ": duplicate entry (" + std::to_string(r + 1) + ", " +
                               std::to_string(c + 1) + ")");
    }
    if (kind == 2)  // explicit_matrix.cpp:33-38
      fail(EQUIL_EINVAL, "ExplicitMatrix::sparse: duplicate entry (" +
                             std::to_string(bad / static_cast<uint64_t>(n)) + ", " +
                             std::to_string(bad % static_cast<uint64_t>(n)) + ")");
    dr.release();
    dc.release();
    dv.release();
    std::vector<int64_t> rph(m + 1);
    CK(cudaMemcpyAsync(rph.data(), rp.p, (m + 1) * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    pt.mark(s, "coo->csr");
    finish_sparse(M.get(), rp, ci, va, rph.data(), pt, nullptr, nullptr);
    *out = M.release();
  }
}
}  // namespace eqe

extern "C" {

equil_status equil_matrix_create_coo(int64_t m, int64_t n, int64_t nnz, const int64_t* rows,
                                     const int64_t* cols, const double* vals,
                                     const equil_device_cfg* cfg, equil_matrix** out) {
  return guarded([&] {
    NvtxRange nvtx_("equil:create_coo");
    create_coo_impl(m, n, nnz, rows, cols, vals, nullptr, cfg, out);
  });
}

equil_status equil_matrix_create_dense(int64_t m, int64_t n, const double* rowmajor,
                                       const equil_device_cfg* cfg, equil_matrix** out) {
  return guarded([&] {
    NvtxRange nvtx_("equil:create_dense");
    require(out != nullptr, "ExplicitMatrix::dense: null output handle");
    *out = nullptr;
    require(m > 0 && n > 0, "ExplicitMatrix::dense: dimensions must be positive");
    require(rowmajor != nullptr, "ExplicitMatrix::dense: null data");
    require(cfg == nullptr || cfg->world_size <= 1,
            "ExplicitMatrix::dense: the dense path runs on one GPU");
    require(n <= static_cast<int64_t>(eqb::kChunk) * 32, "dense: n too large (<= 65536)");
    require((m + eqb::kChunk - 1) / eqb::kChunk <= 64, "dense: m too large (<= 131072)");
    auto M = std::make_unique<equil_matrix>();
    setup_common(M.get(), cfg);
    M->dense = true;
    M->m = m;
    M->n = n;
    M->nnz = m * n;
    DeviceGuard dg(M->device);
    M->Ad.alloc(m * n);
    CK(cudaMemcpyAsync(M->Ad.p, rowmajor, m * n * 8, cudaMemcpyHostToDevice, M->stream));
    M->a_bounds = {0, m};
    M->t_bounds = {0, n};
    alloc_workspaces(M.get());
    CK(cudaStreamSynchronize(M->stream));
    *out = M.release();
  });
}

void equil_matrix_destroy(equil_matrix* A) {
  if (!A) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(A->device);
  cudaStreamSynchronize(A->stream);
  delete A;
  if (prev >= 0) cudaSetDevice(prev);
}

void* equil_matrix_stream(equil_matrix* A) {
  return A ? static_cast<void*>(A->stream) : nullptr;
}

double equil_last_loop_ms(equil_matrix* A, int* iterations) {
  if (!A) return 0.0;
  if (iterations) *iterations = A->last_loop_iters;
  return A->last_loop_ms;
}

long long equil_kernel_launches(void) { return eqb::launch_count(); }

int equil_build_flags(void) {
#ifdef EQ_CHECKED
  return 1;
#else
  return 0;
#endif
}

int equil_sweep_active(const equil_matrix* A) { return A && A->sweep ? 1 : 0; }

int equil_exchange_mode(const equil_matrix* A) {
  if (!A || A->world == 1 || A->p2p_state == 0) return 0;
  return A->p2p_state == 1 ? 2 : 1;
}

equil_status equil_matrix_shape(const equil_matrix* A, int64_t* m, int64_t* n,
                                int64_t* nnz) {
  return guarded([&] {
    require(A != nullptr, "matrix: null handle");
    if (m) *m = A->m;
    if (n) *n = A->n;
    if (nnz) *nnz = A->nnz;
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// SGD driver
// ---------------------------------------------------------------------------
namespace eqe {

struct DiagPlan {
  int stride = 0;
  bool obj = false, rms = false;
};

// canonical reduction of x[0, len) into *out (device): kind 0 sum of squares,
// 1 plain sum, 2 sum of coef * x; optional sqrt of the result
void canon_reduce(equil_matrix* M, const double* x, int64_t len, double* out, int kind,
                  double coef, bool sqrt_out) {
  const size_t parts = static_cast<size_t>((len + eqb::kChunk - 1) / eqb::kChunk) + 1;
  if (parts > M->red_part.n) {  // never inside a captured graph: setup sizes it for m + n
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(M->stream, &cs));
    if (cs != cudaStreamCaptureStatusNone)
      throw std::runtime_error("canon_reduce: partials buffer too small during capture");
    M->red_part.ensure(parts);
  }
  CK(eqb::launch_canon_reduce(x, len, kind, coef, M->red_part.p, M->red_counter.p, out,
                              sqrt_out ? 1 : 0, M->stream, static_cast<int64_t>(M->red_part.n)));
}

}  // namespace eqe

namespace eqe {

// internal::sgd_row_col (src/equilibrate.cpp:138-210).  Uniform targets
// (lin = alpha^2, beta^2) when lin_u_host / lin_v_host are null, otherwise the
// per-coordinate linear terms of sgd_equilibrate_targets (src/variants.cpp:105-118);
// alpha, beta > 0 enable the RMS diagnostic (alpha_for_rms, beta_for_rms).
void sgd_row_col(equil_matrix* M, const equil_params* p, const equil_diag_cfg* diag,
                 equil_scaling_out* out, double alpha, double beta,
                 const double* lin_u_host, const double* lin_v_host) {
  {
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    validate_params(*p);  // :142
    const bool vec_lin = lin_u_host != nullptr;
    if (vec_lin) {  // local slices of the per-coordinate linear terms
      M->lin_u.ensure(M->m_loc());
      M->lin_v.ensure(M->n_loc());
      CK(cudaMemcpyAsync(M->lin_u.p, lin_u_host + M->a_goff(), M->m_loc() * 8,
                         cudaMemcpyHostToDevice, M->stream));
      CK(cudaMemcpyAsync(M->lin_v.p, lin_v_host + M->t_goff(), M->n_loc() * 8,
                         cudaMemcpyHostToDevice, M->stream));
    }
    DiagPlan dp;
    if (diag && diag->stride > 0) {
      dp.stride = diag->stride;
      dp.obj = diag->want_objective != 0;
      dp.rms = diag->want_rms != 0;
      require(!M->dense, "sgd_equilibrate: history is implemented for sparse matrices");
      require(out->hist_cap >= p->iterations / dp.stride + 1,
              "sgd_equilibrate: history capacity too small");
    } else if (diag && diag->stride < 0) {
      fail(EQUIL_EINVAL, "sgd_row_col: stride must be positive");
    }
    cudaStream_t s = M->stream;
    const int T = p->iterations;
    const int64_t m = M->m, n = M->n;
    const uint64_t per_iter = static_cast<uint64_t>(m + n);
    const uint64_t total = per_iter * static_cast<uint64_t>(T);
    const double lin_u = alpha * alpha, lin_v = beta * beta;
    const double gamma = p->gamma, Mx = p->max_log_scale;
    auto block_const = [&](double lin) {
      eqb::SgdBlockConst c;
      c.lin = lin;
      c.gamma = gamma;
      c.M = Mx;
      const double cap = lin / gamma;
      c.thresh = cap + 1e-9 * std::max(1.0, std::abs(cap));
      return c;
    };
    const eqb::SgdBlockConst cu = block_const(lin_u), cv = block_const(lin_v);

    PhaseTimer pt("sgd");
    // K1: all T*(n+m) signs up front (never depends on the iterate); a
    // one-shot call generated them during the matrix setup
    if (total > 0 && M->pre_signs && M->pre_seed == p->seed && M->pre_total == total) {
      CK(cudaStreamWaitEvent(s, M->sign_ev, 0));
      M->pre_signs = false;
    } else if (total > 0) {
      M->signs.ensure((total + 31) / 32 + 1);
      const size_t sb = eqb::sign_stream_scratch_bytes(total);
      M->sign_scratch.ensure(sb);
      CK(eqb::sign_stream_generate(p->seed, 17, total, M->signs.p, M->sign_scratch.p, sb, s));
    }
    pt.mark(s, "signs");
    // init: u = v = 0, ubar = vbar = 0, xs = s_1, xw = w_1
    CK(cudaMemsetAsync(M->flags.p, 0, sizeof(unsigned), s));
    const int64_t a_poff = M->world == 1 ? M->a_goff() : M->rank * M->a_max;
    const int64_t t_poff = M->world == 1 ? M->t_goff() : M->rank * M->t_max;
    if (M->world > 1 && M->p2p_state == 0 && T > 0) setup_peers(M);
    const bool p2p = M->world > 1 && M->p2p_state == 1;
    if (T > 0) {
      CK(eqb::launch_sgd_init(M->xs[0].p, M->xw[0].p, M->u.p, M->ub.p, M->v.p, M->vb.p,
                              M->n_pad(), M->m_pad(), M->signs.p, M->m_loc(), M->n_loc(),
                              M->a_goff(), M->t_goff(), a_poff, t_poff, m, n,
                              M->slots ? M->wmap.p + a_poff : nullptr,
                              M->slots ? M->smap.p + t_poff : nullptr, s));
      allgather_padded(M, M->xs[0].p, M->t_max);
      allgather_padded(M, M->xw[0].p, M->a_max);
    } else {
      CK(cudaMemsetAsync(M->ub.p, 0, M->m_loc() * 8, s));
      CK(cudaMemsetAsync(M->vb.p, 0, M->n_loc() * 8, s));
    }

    // history (src/equilibrate.cpp:174-195) into device slots, read at the end:
    // per record [rms_acc, quad, lin_u.u, lin_v.v, |u|^2, |v|^2].  Every term
    // vector is reduced in global order; with world > 1 the local terms are
    // written into the padded layout, all-gathered and un-padded first, so the
    // record is identical for any number of GPUs.
    constexpr int kRec = 6;
    const int nrec = dp.stride ? T / dp.stride + 1 : 0;
    const bool multi = M->world > 1;
    const int64_t ml = M->m_loc(), nl = M->n_loc();
    DevBuf<double> hist, terms, eu_p, ev_p, ta_p, tt_p, ub_f, vb_f, vb_p;
    if (nrec) {
      hist.alloc(kRec * nrec);
      CK(cudaMemsetAsync(hist.p, 0, kRec * nrec * 8, s));
      terms.alloc(m + n);
      eu_p.alloc(M->m_pad());
      ev_p.alloc(M->n_pad());
      if (multi) {
        ta_p.alloc(M->m_pad());
        tt_p.alloc(M->n_pad());
        ub_f.alloc(m);
        vb_f.alloc(n);
        vb_p.alloc(M->n_pad());
      }
    }
    // local slice -> padded buffer (gathered); world 1: the slice is the vector
    auto to_padded = [&](const double* loc, int64_t cnt, bool mside, double* pad) {
      if (!multi) return;
      const int64_t off = mside ? a_poff : t_poff;
      if (loc != pad + off)
        CK(cudaMemcpyAsync(pad + off, loc, cnt * 8, cudaMemcpyDeviceToDevice, s));
      allgather_padded(M, pad, mside ? M->a_max : M->t_max);
    };
    auto unpad_to = [&](const double* pad, bool mside, double* dst) {
      const int64_t full = mside ? m : n;
      const int64_t maxcnt = mside ? M->a_max : M->t_max;
      unpad_kernel<<<static_cast<unsigned>((full + 255) / 256), 256, 0, s>>>(
          dst, pad, (mside ? M->a_bounds_d : M->t_bounds_d).p, M->world, maxcnt, full);
      CK(cudaGetLastError());
    };
    int rec = 0;
    auto record = [&](int) {
      double* slot = hist.p + kRec * rec;
      if (dp.rms && alpha > 0.0 && beta > 0.0) {  // rms_error (src/metrics.cpp:41-56)
        CK(eqb::launch_exp(M->ub.p, eu_p.p + a_poff, ml, 2.0, s));
        CK(eqb::launch_exp(M->vb.p, ev_p.p + t_poff, nl, 2.0, s));
        to_padded(eu_p.p + a_poff, ml, true, eu_p.p);
        to_padded(ev_p.p + t_poff, nl, false, ev_p.p);
        double* ta = multi ? ta_p.p + a_poff : terms.p;
        double* tt = multi ? tt_p.p + t_poff : terms.p + m;
        CK(eqb::launch_rms_terms(0, M->A, eu_p.p, ev_p.p, ta, a_poff, alpha, s));
        CK(eqb::launch_rms_terms(1, M->AT, eu_p.p, ev_p.p, tt, t_poff, beta, s));
        if (multi) {
          to_padded(ta, ml, true, ta_p.p);
          to_padded(tt, nl, false, tt_p.p);
          unpad_to(ta_p.p, true, terms.p);
          unpad_to(tt_p.p, false, terms.p + m);
        }
        canon_reduce(M, terms.p, m + n, slot + 0, 1);
      }
      if (dp.obj) {  // objective_weighted (src/equilibrate.cpp:10-22)
        const double* ubf = M->ub.p;  // whole ubar / vbar in global order
        const double* vbf = M->vb.p;
        const double* vbp = M->vb.p;  // vbar in padded coordinates (gathered)
        if (multi) {
          to_padded(M->ub.p, ml, true, ta_p.p);
          unpad_to(ta_p.p, true, ub_f.p);
          to_padded(M->vb.p, nl, false, vb_p.p);
          unpad_to(vb_p.p, false, vb_f.p);
          ubf = ub_f.p;
          vbf = vb_f.p;
          vbp = vb_p.p;
        }
        double* ot = multi ? ta_p.p + a_poff : terms.p;
        CK(eqb::launch_obj_terms(M->A, M->ub.p, vbp, ot, s));
        if (multi) {
          to_padded(ot, ml, true, ta_p.p);
          unpad_to(ta_p.p, true, terms.p);
        }
        canon_reduce(M, terms.p, m, slot + 1, 1);
        if (vec_lin) {  // lin_u.dot(u): rounded products, canonical sum
          double* pu = multi ? ta_p.p + a_poff : terms.p;
          CK(eqb::launch_mul(pu, M->lin_u.p, M->ub.p, ml, s));
          if (multi) {
            to_padded(pu, ml, true, ta_p.p);
            unpad_to(ta_p.p, true, terms.p);
          }
          canon_reduce(M, terms.p, m, slot + 2, 1);
          double* pv = multi ? tt_p.p + t_poff : terms.p;
          CK(eqb::launch_mul(pv, M->lin_v.p, M->vb.p, nl, s));
          if (multi) {
            to_padded(pv, nl, false, tt_p.p);
            unpad_to(tt_p.p, false, terms.p);
          }
          canon_reduce(M, terms.p, n, slot + 3, 1);
        } else {
          canon_reduce(M, ubf, m, slot + 2, 2, lin_u);
          canon_reduce(M, vbf, n, slot + 3, 2, lin_v);
        }
        canon_reduce(M, ubf, m, slot + 4, 0);
        canon_reduce(M, vbf, n, slot + 5, 0);
      }
      ++rec;
    };
    if (dp.stride) record(0);

    auto host_step = [&](int t) {
      eqb::SgdStep st;
      st.step = 2.0 / (gamma * static_cast<double>(t + 1));  // :106
      st.aw = 2.0 / (static_cast<double>(t) + 2.0);           // :107
      st.aw1 = 1.0 - st.aw;
      st.pad = 0;
      return st;
    };
    auto iter_args = [&](int t) {
      eqb::SgdIterArgs a{};
      for (int k = 0; k < 2; ++k) {  // column blocks (round set per launch)
        a.nblk[k] = M->nblk[k];
        a.bnd[k] = M->bnd[k].p;
        a.carry[k] = M->carry[k].p;
      }
      for (int k = 0; k < 2; ++k) {
        const eqb::DevCsr& C = k ? M->AT : M->A;
        a.rp[k] = C.row_ptr;
        a.ci[k] = C.col;
        a.va[k] = C.val;
        a.rl[k] = k ? M->rowlist_t.p : M->rowlist_a.p;
      }
      a.tiles = M->tiles_sgd.p;
      a.n_long = M->n_sgd_long;
      a.xs_cur = M->xs[(t - 1) & 1].p;
      a.xw_cur = M->xw[(t - 1) & 1].p;
      a.xs_next = M->xs[t & 1].p;
      a.xw_next = M->xw[t & 1].p;
      a.x[0] = M->u.p;
      a.x[1] = M->v.p;
      a.avg[0] = M->ub.p;
      a.avg[1] = M->vb.p;
      a.goff[0] = M->a_goff();
      a.goff[1] = M->t_goff();
      a.poff[0] = a_poff;
      a.poff[1] = t_poff;
      a.signs = M->signs.p;
      a.sign_next[0] = static_cast<int64_t>(t) * (m + n) + n + M->a_goff();
      a.sign_next[1] = static_cast<int64_t>(t) * (m + n) + M->t_goff();
      a.has_next = t < T;
      a.c[0] = cu;
      a.c[1] = cv;
      a.lin[0] = vec_lin ? M->lin_u.p : nullptr;
      a.lin[1] = vec_lin ? M->lin_v.p : nullptr;
      if (M->slots) {
        a.ci[0] = M->a_ci_sgd.p;
        a.ci[1] = M->t_ci_sgd.p;
        a.slot[0] = M->wmap.p + a_poff;  // local row r -> slot
        a.slot[1] = M->smap.p + t_poff;
      }
      a.st = host_step(t);
      a.flags = M->flags.p;
      if (p2p) {
        a.npeer = static_cast<int>(M->peer_delta.size());
        for (int g = 0; g < a.npeer; ++g) a.peer_delta[g] = M->peer_delta[g];
      }
      return a;
    };
    auto dense_args = [&](int t) {
      eqb::DenseIterArgs a{};
      a.A = M->Ad.p;
      a.m = m;
      a.n = n;
      a.xs_cur = M->xs[(t - 1) & 1].p;
      a.xw_cur = M->xw[(t - 1) & 1].p;
      a.xs_next = M->xs[t & 1].p;
      a.xw_next = M->xw[t & 1].p;
      a.u = M->u.p;
      a.ub = M->ub.p;
      a.v = M->v.p;
      a.vb = M->vb.p;
      a.signs = M->signs.p;
      a.sign_next_w = static_cast<int64_t>(t) * (m + n) + n;
      a.sign_next_s = static_cast<int64_t>(t) * (m + n);
      a.has_next = t < T;
      a.cu = cu;
      a.cv = cv;
      a.lin_u = vec_lin ? M->lin_u.p : nullptr;
      a.lin_v = vec_lin ? M->lin_v.p : nullptr;
      a.st = host_step(t);
      a.flags = M->flags.p;
      a.colpart = M->colpart.p;
      a.colcnt = M->colcnt.p;
      return a;
    };
    auto one_iter = [&](int t) {
      if (M->dense) {
        static const int dconc = getenv("EQUIL_CONC") ? atoi(getenv("EQUIL_CONC")) : 1;
        if (dconc)
          CK(eqb::launch_dense_sgd_iter(dense_args(t), s, M->copy_stream, M->ev_fork, M->ev_join));
        else
          CK(eqb::launch_dense_sgd_iter(dense_args(t), s));
      } else {
        static const int conc = getenv("EQUIL_CONC") ? atoi(getenv("EQUIL_CONC")) : 1;
        const int rounds = std::max(M->nblk[0], M->nblk[1]);
        for (int rd = 0; rd < rounds; ++rd) {  // column-block rounds (1 unless blocked)
          eqb::SgdIterArgs a = iter_args(t);
          a.round = rd;
          if (M->sell) {
            eqb::SellArgs sa{};
            sa.xlen[0] = M->n_pad();  // A's rows gather xs, A^T's xw
            sa.xlen[1] = M->m_pad();
            sa.quad_min = M->sell_nb == 1 ? quad_min(M) : 0x7fffffff;  // see plan_sell
            sa.slices = M->sell_slices.p;
            sa.nslices = M->n_sell;
            sa.row = M->sell_row.p;
            sa.len = M->sell_len.p;
            if (M->sell_nb > 1) {  // column block rd of every slice, sums carried per lane
              sa.slices = M->sell_bslices.p + static_cast<size_t>(rd) * M->n_sell;
              sa.len = M->sell_bln.p + static_cast<size_t>(rd) * 32 * M->n_sell;
              a.carry[0] = a.carry[1] = M->sell_carry.p;
            }
            for (int k = 0; k < 2; ++k) {
              sa.ci[k] = M->sell_ci[k].p;
              sa.va[k] = M->sell_va[k].p;
            }
            // with peer stores (p2p) the fused epilogue sends each row's next
            // value as soon as its sum is done, overlapping the exchange with
            // the passes; the split epilogue would send them all afterwards
            if (M->split_epi && M->sell_nb == 1 && M->sell_long == 2 && !p2p) {
              // row sums from both kernels (concurrent), then one update pass
              a.carry[0] = M->rowacc.p;
              a.carry[1] = M->rowacc.p + M->m_loc();
              CK(cudaEventRecord(M->ev_fork, s));
              CK(cudaStreamWaitEvent(M->copy_stream, M->ev_fork, 0));
              eqb::SellArgs sl = sa;
              sl.nslices = M->n_sell_long;
              // A's long rows: the column sweep (all long slices are A's), ahead of
              // the warp slices on the same stream -- its shared-memory stages leave
              // the concurrent warp kernel too little L1 for xw's hot slots (c3:
              // 1.09-1.17 concurrent vs 0.92 serial)
              if (M->sweep)
                CK(eqb::launch_sweep(a.xs_cur, a.carry[0], M->sweep_args, s));
              else
                CK(eqb::launch_sgd_sell_split(a, sl, true, M->sell_lvariant, M->copy_stream));
              sa.first = M->n_sell_long;
              // alone on the SMs (after the sweep) the warp slices do slightly better
              // with batches of 4 at 10 CTAs per SM (c3: 0.867-0.881 vs 0.880-0.887)
              CK(eqb::launch_sgd_sell_split(
                  a, sa, false, M->sweep && M->sell_variant == 0 ? 2 : M->sell_variant, s));
              CK(cudaEventRecord(M->ev_join, M->copy_stream));
              CK(cudaStreamWaitEvent(s, M->ev_join, 0));
              CK(eqb::launch_sgd_update_rows(a, M->m_loc(), M->n_loc(), s));
            } else if (M->sell_long == 2 && M->n_sell_long > 0) {
              // long slices on warp-specialised CTAs, the rest on warps,
              // concurrently (fork / join on the copy stream)
              CK(cudaEventRecord(M->ev_fork, s));
              CK(cudaStreamWaitEvent(M->copy_stream, M->ev_fork, 0));
              eqb::SellArgs sl = sa;
              sl.nslices = M->n_sell_long;
              CK(eqb::launch_sgd_sell_long(a, sl, M->sell_lvariant, M->copy_stream));
              sa.first = M->n_sell_long;
              CK(eqb::launch_sgd_sell(a, sa, M->sell_variant, s));
              CK(cudaEventRecord(M->ev_join, M->copy_stream));
              CK(cudaStreamWaitEvent(s, M->ev_join, 0));
            } else if (M->sell_long || M->n_sgd_long == 0) {
              CK(eqb::launch_sgd_sell(a, sa, M->sell_variant, s));
            } else {
              // rows longer than a tile stay CTA-cooperative (their sequential
              // chains would otherwise wait on every load round trip)
              CK(cudaEventRecord(M->ev_fork, s));
              CK(cudaStreamWaitEvent(M->copy_stream, M->ev_fork, 0));
              CK(eqb::launch_sgd_iter_part(a, 0, M->n_sgd_long, true, 6, M->copy_stream));
              CK(eqb::launch_sgd_sell(a, sa, M->sell_variant, s));
              CK(cudaEventRecord(M->ev_join, M->copy_stream));
              CK(cudaStreamWaitEvent(s, M->ev_join, 0));
            }
          } else if (rounds > 1) {
            // column blocks: one launch pair per (round, matrix), so each launch
            // gathers from one block, which the L2 access-policy window on both
            // streams keeps persisting (EQUIL_BLOCK_WIN=0: the whole-buffer window)
            for (int mat = 0; mat < 2; ++mat) {
              if (rd >= M->nblk[mat]) continue;
              if (M->block_win) {
                const int64_t len = mat ? M->m_pad() : M->n_pad();
                const int64_t b0 = rd * M->bwidth[mat];
                const double* base = (mat ? a.xw_cur : a.xs_cur) + b0;
                const size_t bytes = static_cast<size_t>(std::min(M->bwidth[mat], len - b0)) * 8;
                set_l2_window(M, s, base, bytes);
                set_l2_window(M, M->copy_stream, base, bytes);
              }
              const int lb = mat ? M->n_la : 0;
              const int ln = mat ? M->n_sgd_long - M->n_la : M->n_la;
              const int sb = M->n_sgd_long + (mat ? M->n_sa : 0);
              const int sn = mat ? M->n_sgd - M->n_sgd_long - M->n_sa : M->n_sa;
              CK(cudaEventRecord(M->ev_fork, s));
              CK(cudaStreamWaitEvent(M->copy_stream, M->ev_fork, 0));
              if (ln > 0) CK(eqb::launch_sgd_iter_part(a, lb, ln, true, 6, M->copy_stream));
              if (sn > 0) CK(eqb::launch_sgd_iter_part(a, sb, sn, false, 6, s));
              CK(cudaEventRecord(M->ev_join, M->copy_stream));
              CK(cudaStreamWaitEvent(s, M->ev_join, 0));
            }
            if (M->block_win && rd == rounds - 1) {  // back to the default windows
              set_l2_window(M, s, M->xbuf.p, 0);
              set_l2_window(M, M->copy_stream, nullptr, 0);
            }
          } else if (conc && M->n_sgd_long > 0 && M->n_sgd_long < M->n_sgd) {
            // long-row CTA groups and warp tiles as two concurrent kernels (fork /
            // join on the copy stream): each kernel gets its own residency on the
            // SMs instead of one launch sized for both (c3: 4-5% faster)
            CK(cudaEventRecord(M->ev_fork, s));
            CK(cudaStreamWaitEvent(M->copy_stream, M->ev_fork, 0));
            CK(eqb::launch_sgd_iter_part(a, 0, M->n_sgd_long, true, conc >= 2 ? 8 : 6,
                                         M->copy_stream));
            CK(eqb::launch_sgd_iter_part(a, M->n_sgd_long, M->n_sgd - M->n_sgd_long, false,
                                         conc >= 3 ? 8 : 6, s));
            CK(cudaEventRecord(M->ev_join, M->copy_stream));
            CK(cudaStreamWaitEvent(s, M->ev_join, 0));
          } else {
            CK(eqb::launch_sgd_iter(a, M->n_sgd, s));
          }
        }
        if (t < T && p2p) {
          rank_barrier(M);  // the epilogue already stored into every peer's copy
        } else if (t < T) {
          allgather_padded(M, M->xs[t & 1].p, M->t_max);
          allgather_padded(M, M->xw[t & 1].p, M->a_max);
        }
      }
    };

    if (dp.stride == 0 && T > 0 && !M->hx && !M->oneshot) {  // (host exchange: no capture)
      // capture the whole T loop once per (T, targets, gamma, M) and replay it
      equil_matrix::Key key{T, alpha, beta, gamma, Mx, vec_lin};
      if (!M->graph || !(M->graph_key == key)) {
        if (M->graph) {
          cudaGraphExecDestroy(M->graph);
          M->graph = nullptr;
        }
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        try {
          // external event-record nodes: the graph itself timestamps the loop
          CK(cudaEventRecordWithFlags(M->ev_loop0, s, cudaEventRecordExternal));
          for (int t = 1; t <= T; ++t) one_iter(t);
          CK(cudaEventRecordWithFlags(M->ev_loop1, s, cudaEventRecordExternal));
        } catch (...) {
          cudaStreamEndCapture(s, &g);
          throw;
        }
        CK(cudaStreamEndCapture(s, &g));
        {  // kernel nodes of one replay, for the launch accounting
          size_t nn = 0;
          CK(cudaGraphGetNodes(g, nullptr, &nn));
          std::vector<cudaGraphNode_t> nodes(nn);
          if (nn) CK(cudaGraphGetNodes(g, nodes.data(), &nn));
          long long kn = 0;
          for (cudaGraphNode_t nd : nodes) {
            cudaGraphNodeType ty;
            if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel) ++kn;
          }
          M->graph_launches = kn;
        }
        CK(cudaGraphInstantiate(&M->graph, g, 0));
        cudaGraphDestroy(g);
        M->graph_key = key;
      }
      CK(cudaGraphLaunch(M->graph, s));
      eqb::note_launches(M->graph_launches);
    } else {
      CK(cudaEventRecord(M->ev_loop0, s));
      for (int t = 1; t <= T; ++t) {
        one_iter(t);
        if (dp.stride && t % dp.stride == 0) record(t);
      }
      CK(cudaEventRecord(M->ev_loop1, s));
    }
    M->last_loop_iters = T;
    pt.mark(s, "loop");

    // finalize: u = ubar, v = vbar, d = exp(ubar), e = exp(vbar) (:201-204)
    double* dloc = M->tmp_m.p;
    double* eloc = M->tmp_n.p;
    CK(eqb::launch_exp(M->ub.p, dloc, ml, 1.0, s));
    CK(eqb::launch_exp(M->vb.p, eloc, nl, 1.0, s));
    if (p2p && !M->hx) {  // a timed-out device barrier leaves the ranks out of step
      unsigned long long err = 0;
      CK(cudaMemcpyAsync(&err, M->xbar() + eqb::kBarError, sizeof err, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (err) fail(EQUIL_ERUNTIME, "sgd_equilibrate: peer barrier timed out (a rank stalled)");
    }
    unsigned flags = 0;
    if (M->world > 1 && M->hx) {  // host exchange: max of the flag words
      unsigned mine = 0;
      CK(cudaMemcpyAsync(&mine, M->flags.p, sizeof mine, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      M->hx->put(M->rank, &mine, sizeof mine);
      M->hx->barrier();
      unsigned all = 0;
      for (int g = 0; g < M->world; ++g) {
        unsigned v = 0;
        std::memcpy(&v, M->hx->slot(g), sizeof v);
        all |= v;
      }
      M->hx->barrier();
      CK(cudaMemcpyAsync(M->flags.p, &all, sizeof all, cudaMemcpyHostToDevice, s));
    } else if (M->world > 1) {
      // the flag words are bit sets (1: iterate bound, 2: box); NCCL has no
      // bitwise OR, so gather every rank's word and OR them
      DevBuf<unsigned> words;
      words.alloc(M->world);
      nccl_check(nccl().AllGather(M->flags.p, words.p, 1, ncclUint32, M->comm, s),
                 "ncclAllGather");
      std::vector<unsigned> w(M->world);
      CK(cudaMemcpyAsync(w.data(), words.p, M->world * sizeof(unsigned), cudaMemcpyDeviceToHost,
                         s));
      CK(cudaStreamSynchronize(s));
      unsigned all = 0;
      for (unsigned x : w) all |= x;
      CK(cudaMemcpyAsync(M->flags.p, &all, sizeof all, cudaMemcpyHostToDevice, s));
    }
    CK(cudaMemcpyAsync(&flags, M->flags.p, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    const cudaMemcpyKind kind =
        out->outputs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (M->world == 1) {
      if (out->u) CK(cudaMemcpyAsync(out->u, M->ub.p, ml * 8, kind, s));
      if (out->v) CK(cudaMemcpyAsync(out->v, M->vb.p, nl * 8, kind, s));
      if (out->d) CK(cudaMemcpyAsync(out->d, dloc, ml * 8, kind, s));
      if (out->e) CK(cudaMemcpyAsync(out->e, eloc, nl * 8, kind, s));
    } else {
      // gather the four vectors in padded coordinates, then un-pad
      auto gather_out = [&](const double* loc, int64_t cnt, int64_t maxcnt, int64_t full,
                            const DevBuf<int64_t>& bd, double* dst) {
        DevBuf<double> pad, flat;
        pad.alloc(maxcnt * M->world);
        flat.alloc(full);
        CK(cudaMemcpyAsync(pad.p + M->rank * maxcnt, loc, cnt * 8, cudaMemcpyDeviceToDevice, s));
        allgather_padded(M, pad.p, maxcnt);
        unpad_kernel<<<static_cast<unsigned>((full + 255) / 256), 256, 0, s>>>(
            flat.p, pad.p, bd.p, M->world, maxcnt, full);
        CK(cudaGetLastError());
        if (dst) CK(cudaMemcpyAsync(dst, flat.p, full * 8, kind, s));
        CK(cudaStreamSynchronize(s));
      };
      gather_out(M->ub.p, ml, M->a_max, m, M->a_bounds_d, out->u);
      gather_out(M->vb.p, nl, M->t_max, n, M->t_bounds_d, out->v);
      gather_out(dloc, ml, M->a_max, m, M->a_bounds_d, out->d);
      gather_out(eloc, nl, M->t_max, n, M->t_bounds_d, out->e);
    }
    std::vector<double> hh(kRec * static_cast<size_t>(std::max(nrec, 1)));
    if (nrec)
      CK(cudaMemcpyAsync(hh.data(), hist.p, kRec * nrec * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    pt.mark(s, "finalize");
    M->last_loop_ms = 0.0;
    if (T > 0) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, M->ev_loop0, M->ev_loop1) == cudaSuccess)
        M->last_loop_ms = ms;
      cudaGetLastError();
    }
    out->alpha = alpha;
    out->beta = beta;
    out->iterate_bound_ok = (flags & 1u) ? 0 : 1;
    out->box_feasible = (flags & 2u) ? 0 : 1;
    out->apply_count = T;
    out->adjoint_count = T;
    out->hist_len = nrec;
    for (int h = 0; h < nrec; ++h) {
      const double* r = hh.data() + kRec * h;
      if (out->hist_iter) out->hist_iter[h] = h * dp.stride;
      if (out->hist_objective)
        out->hist_objective[h] =
            dp.obj ? 0.5 * r[1] - r[2] - r[3] + 0.5 * gamma * (r[4] + r[5]) : 0.0;
      if (out->hist_rms)
        out->hist_rms[h] = dp.rms ? std::sqrt(r[0] / static_cast<double>(m + n)) : 0.0;
    }
  }
}

// canonical sum on the host (det_math.cuh definition; precondition checks only)
double canon_sum_host(const double* x, int64_t len) {
  if (len <= 0) return 0.0;
  const int64_t nc = (len + eqb::kChunk - 1) / eqb::kChunk;
  std::vector<double> part(nc), s(eqb::kLanes2);
  for (int64_t c = 0; c < nc; ++c) {
    const int64_t base = c * eqb::kChunk, clen = std::min<int64_t>(eqb::kChunk, len - base);
    for (int l = 0; l < eqb::kLanes1; ++l) {
      double acc = 0.0;
      for (int64_t k = l; k < clen; k += eqb::kLanes1) acc = acc + x[base + k];
      s[l] = acc;
    }
    for (int h = eqb::kLanes1 / 2; h >= 1; h >>= 1)
      for (int l = 0; l < h; ++l) s[l] = s[l] + s[l + h];
    part[c] = s[0];
  }
  for (int l = 0; l < eqb::kLanes2; ++l) {
    double acc = 0.0;
    for (int64_t k = l; k < nc; k += eqb::kLanes2) acc = acc + part[k];
    s[l] = acc;
  }
  for (int h = eqb::kLanes2 / 2; h >= 1; h >>= 1)
    for (int l = 0; l < h; ++l) s[l] = s[l] + s[l + h];
  return s[0];
}

}  // namespace eqe

extern "C" equil_status equil_sgd_equilibrate(equil_matrix* M, const equil_params* p,
                                              const equil_diag_cfg* diag,
                                              equil_scaling_out* out) {
  return guarded([&] {
    NvtxRange nvtx_("equil:sgd_equilibrate");
    require(M != nullptr && p != nullptr && out != nullptr, "sgd_equilibrate: null argument");
    double alpha = 0, beta = 0;
    resolve_targets(*p, M->m, M->n, alpha, beta);  // src/equilibrate.cpp:216
    sgd_row_col(M, p, diag, out, alpha, beta, nullptr, nullptr);
  });
}

extern "C" equil_status equil_sgd_equilibrate_targets(equil_matrix* M, const double* r,
                                                      const double* c, const equil_params* p,
                                                      const equil_diag_cfg* diag,
                                                      equil_scaling_out* out) {
  return guarded([&] {
    NvtxRange nvtx_("equil:sgd_equilibrate_targets");
    require(M != nullptr && p != nullptr && out != nullptr,
            "sgd_equilibrate_targets: null argument");
    require(r != nullptr && c != nullptr, "sgd_equilibrate_targets: target length mismatch");
    for (int64_t i = 0; i < M->m; ++i)
      require(r[i] > 0.0, "sgd_equilibrate_targets: targets must be positive");
    for (int64_t j = 0; j < M->n; ++j)
      require(c[j] > 0.0, "sgd_equilibrate_targets: targets must be positive");
    const double sum_r = canon_sum_host(r, M->m), sum_c = canon_sum_host(c, M->n);
    require(std::abs(sum_r - sum_c) <= 1e-8 * std::max(sum_r, sum_c),
            "sgd_equilibrate_targets: sum(r) == sum(c) violated");
    sgd_row_col(M, p, diag, out, 0.0, 0.0, r, c);  // variants.cpp:117
  });
}

// ---------------------------------------------------------------------------
// LSQR (src/lsqr.cpp:17-138).  Device vectors, canonical norms, host scalar
// recurrence with std::hypot.
// ---------------------------------------------------------------------------
namespace eqe {

// one matvec pass of B (scaled by scale when non-null) in the given mode
void apply_pass(equil_matrix* M, bool adjoint, const double* xg, double* out, int mode,
                const double* scale, const double* prev, const double* coef,
                const int* skip, bool slotted) {
  if (M->dense) {
    eqb::DensePassArgs a{};
    a.A = M->Ad.p;
    a.m = M->m;
    a.n = M->n;
    a.adjoint = adjoint ? 1 : 0;
    a.xg = xg;
    a.out = out;
    a.scale = scale;
    a.prev = prev;
    a.coef = coef;
    a.mode = mode;
    a.skip = skip;
    a.colpart = M->colpart.p;
    a.colcnt = M->colcnt.p;
    CK(eqb::launch_dense_pass(a, M->stream));
    return;
  }
  eqb::PassArgs a{};
  const eqb::DevCsr& C = adjoint ? M->AT : M->A;
  a.rp = C.row_ptr;
  a.ci = C.col;
  a.va = C.val;
  a.tiles = adjoint ? M->tiles_t.p : M->tiles_a.p;
  a.rl = adjoint ? M->rowlist_t.p : M->rowlist_a.p;
  a.xg = xg;
  a.out = out;
  a.scale = scale;
  a.prev = prev;
  a.coef = coef;
  a.mode = mode;
  a.skip = skip;
  if (M->sell && M->sell_passes) {
    sell_pass(M, adjoint ? 1 : 0, a, nullptr, false, slotted);
    return;
  }
  CK(eqb::launch_pass(a, adjoint ? M->n_t : M->n_a, M->stream));
}

// two passes of A (not the adjoint) sharing one traversal of CSR(A):
// out0 <- (xg0, mode0, ...), out1 <- (xg1, mode1, ...); dense: two passes.
// pair (interleaved slices only, pair_layout): xg0 holds both gathered vectors
// interleaved, xg0[2c] for pass 0 and xg0[2c + 1] for pass 1; xg1 is ignored.
bool pair_layout(const equil_matrix* M) { return !M->dense && M->sell && M->sell_passes; }

void apply_pass_dual(equil_matrix* M, const double* xg0, double* out0, int mode0,
                     const double* scale0, const double* prev0, const double* coef0,
                     const double* xg1, double* out1, int mode1, const double* scale1,
                     const double* prev1, const double* coef1, bool pair = false,
                     bool slotted = false) {
  if (M->dense) {
    apply_pass(M, false, xg0, out0, mode0, scale0, prev0, coef0);
    apply_pass(M, false, xg1, out1, mode1, scale1, prev1, coef1);
    return;
  }
  eqb::PassArgs a{}, b{};
  for (eqb::PassArgs* p : {&a, &b}) {
    p->rp = M->A.row_ptr;
    p->ci = M->A.col;
    p->va = M->A.val;
    p->tiles = M->tiles_a.p;
    p->rl = M->rowlist_a.p;
  }
  a.xg = xg0; a.out = out0; a.mode = mode0; a.scale = scale0; a.prev = prev0; a.coef = coef0;
  b.xg = xg1; b.out = out1; b.mode = mode1; b.scale = scale1; b.prev = prev1; b.coef = coef1;
  if (M->sell && M->sell_passes) {
    sell_pass(M, 0, a, &b, pair, slotted);
    return;
  }
  if (pair) throw std::runtime_error("apply_pass_dual: interleaved pair without slices");
  CK(eqb::launch_pass_dual(a, b, M->n_a, M->stream));
}

double read_scalar(equil_matrix* M, const double* dev) {
  double h = 0;
  CK(cudaMemcpyAsync(&h, dev, 8, cudaMemcpyDeviceToHost, M->stream));
  CK(cudaStreamSynchronize(M->stream));
  return h;
}

struct LsqrState {
  int hist_len = 0;
  int iterations = 0;
  bool reached_tol = false, breakdown = false;
  long long applies = 0, adjoints = 0;
};

// Row-sharded LSQR vectors.  m-side vectors (u, the residual) live as local
// slices of A's rows, n-side ones (v, w, x) as local slices of A^T's rows;
// the vectors a pass gathers from (d.*u, e.*v, e.*x) are kept in the padded
// layout of the SGD loop and all-gathered after every update.  A norm is the
// canonical reduction of the whole vector in global order: the padded buffer
// is all-gathered and un-padded first, so every rank computes the identical
// scalar for any world size (world 1: no copies).
struct LsqrLayout {
  equil_matrix* M;
  int64_t mL, nL, mP, nP, pa, pt;
  DevBuf<double> flat_m, flat_n;
  explicit LsqrLayout(equil_matrix* m_) : M(m_) {
    mL = M->m_loc();
    nL = M->n_loc();
    mP = M->m_pad();
    nP = M->n_pad();
    pa = M->world == 1 ? 0 : M->rank * M->a_max;
    pt = M->world == 1 ? 0 : M->rank * M->t_max;
    if (M->world > 1) {
      flat_m.alloc(M->m);
      flat_n.alloc(M->n);
    }
  }
  void gather(double* pad, bool mside) {
    allgather_padded(M, pad, mside ? M->a_max : M->t_max);
  }
  // out_dev = |v| for the padded vector whose local slice was just written
  void norm(double* pad, bool mside, double* out_dev) {
    const int64_t full = mside ? M->m : M->n;
    if (M->world == 1) {
      canon_reduce(M, pad, full, out_dev, 0, 0.0, true);
      return;
    }
    const int64_t maxcnt = mside ? M->a_max : M->t_max;
    double* flat = mside ? flat_m.p : flat_n.p;
    gather(pad, mside);
    unpad_kernel<<<static_cast<unsigned>((full + 255) / 256), 256, 0, M->stream>>>(
        flat, pad, (mside ? M->a_bounds_d : M->t_bounds_d).p, M->world, maxcnt, full);
    CK(cudaGetLastError());
    canon_reduce(M, flat, full, out_dev, 0, 0.0, true);
  }
};

// lsqr_core (:17-81) on B = diag(d) A diag(e) (d, e local slices or null) with
// local rhs slice c; x receives the local slice of the solution
void lsqr_core(equil_matrix* M, const double* c, const double* b_loc, double bnorm,
               const double* d, const double* e, int max_iters, double tol,
               double* hist, int hist_cap, LsqrState& st, DevBuf<double>& x) {
  cudaStream_t s = M->stream;
  LsqrLayout L(M);
  // pair: the two vectors the fused residual + B v pass gathers, e.x and e.v,
  // live interleaved in one padded array (xv[2c], xv[2c + 1]) so that pass
  // makes one 16-byte gather per entry; it is all-gathered once per iteration,
  // after the x update (e.v is only read by that pass)
  const bool pair = pair_layout(M);
  const int64_t os = pair ? 2 : 1;
  // slotted: the gathered vectors (d.u for the A^T pass, the (e.x, e.v) pair
  // for the A pass) are written in the SGD loop's hot-first slot layout, so
  // the passes run on the SGD's slot-mapped interleaved columns and A's
  // longest rows -- gathered by most rows of A^T -- stay L1-resident
  const bool slotted = pair && M->slots && M->sell_nb == 1;
  const int32_t* slot_u = slotted ? M->wmap.p + L.pa : nullptr;  // local A row -> slot
  const int32_t* slot_v = slotted ? M->smap.p + L.pt : nullptr;  // local A^T row -> slot
  DevBuf<double> u, v, w, un, du, vn, ev, ex, xv, r;
  u.alloc(L.mL); v.alloc(L.nL); w.alloc(L.nL); x.alloc(L.nL);
  un.alloc(L.mP); du.alloc(L.mP); r.alloc(L.mP);
  vn.alloc(L.nP);
  if (pair) {
    xv.alloc(2 * L.nP);
    CK(cudaMemsetAsync(xv.p, 0, 2 * L.nP * 8, s));  // e.x = 0 for the first pass
  } else {
    ev.alloc(L.nP);
    ex.alloc(L.nP);
  }
  double* unL = un.p + L.pa;
  double* duL = slotted ? du.p : du.p + L.pa;  // slotted: slot maps hold absolute positions
  double* rL = r.p + L.pa;
  double* vnL = vn.p + L.pt;
  double* evL = pair ? xv.p + (slotted ? 0 : 2 * L.pt) + 1 : ev.p + L.pt;
  double* exL = pair ? xv.p + (slotted ? 0 : 2 * L.pt) : ex.p + L.pt;
  auto gather_ev = [&] {
    if (pair) allgather_padded(M, xv.p, 2 * M->t_max);
    else L.gather(ev.p, false);
  };
  auto gather_ex = [&] {
    if (pair) allgather_padded(M, xv.p, 2 * M->t_max);
    else L.gather(ex.p, false);
  };
  CK(cudaMemsetAsync(x.p, 0, L.nL * 8, s));
  double* sc = M->scal.p;  // [0] beta, [1] alpha, [2] residual norm
  int* dummy = reinterpret_cast<int*>(sc + 8);
  int* inv = reinterpret_cast<int*>(sc + 9);  // this iteration's invariant flag

  CK(cudaMemcpyAsync(unL, c, L.mL * 8, cudaMemcpyDeviceToDevice, s));
  L.norm(un.p, true, sc + 0);  // beta = |c|
  CK(eqb::launch_lsqr_normalize(u.p, c, sc + 0, duL, d, L.mL, nullptr, nullptr, s, 1, slot_u));
  L.gather(du.p, true);
  apply_pass(M, true, du.p, vnL, eqb::kPassScaled, e, nullptr, nullptr, nullptr,
             slotted);  // v = B^T u
  ++st.adjoints;
  L.norm(vn.p, false, sc + 1);
  double beta = read_scalar(M, sc + 0);
  double alpha = read_scalar(M, sc + 1);
  if (alpha == 0.0) {
    st.breakdown = true;
    return;
  }
  CK(eqb::launch_lsqr_normalize(v.p, vnL, sc + 1, evL, e, L.nL, dummy, nullptr, s, os, slot_v));
  gather_ev();
  CK(cudaMemcpyAsync(w.p, v.p, L.nL * 8, cudaMemcpyDeviceToDevice, s));
  double phibar = beta, rhobar = alpha;

  // One host synchronisation per iteration.  The device runs the first half of
  // iteration t (B v - alpha u is already there, |u'|, u = u'/beta, B^T u -
  // beta v, |v'|, v = v'/alpha) with the reference's invariant branches
  // (:41-52) as device flags: a normalisation whose norm is not positive sets
  // `inv` and every later step of the iteration is skipped.  The host then
  // reads beta, alpha, the flag and iteration t-1's residual norm in one copy,
  // records t-1 (and stops where the reference stops after t-1: tol reached or
  // invariant), and runs the scalar recurrence with std::hypot exactly as
  // :58-64 before the x / w update and the fused residual + next B v pass.
  // A stop found at that point discards only the speculative first half of
  // iteration t (u, v, not outputs); counts are committed per accepted iteration.
  if (!M->lsqr_sync) {
    void* q = nullptr;
    CK(cudaHostAlloc(&q, sizeof(equil_matrix::LsqrSync), cudaHostAllocDefault));
    M->lsqr_sync = static_cast<equil_matrix::LsqrSync*>(q);
  }
  equil_matrix::LsqrSync* hs = M->lsqr_sync;
  auto record = [&](double rnorm) -> bool {  // true: stop after this iteration
    const double rel = rnorm / bnorm;
    if (st.hist_len < hist_cap) hist[st.hist_len] = rel;
    ++st.hist_len;
    if (rel <= tol) {
      st.reached_tol = true;
      return true;
    }
    return false;
  };
  bool prev_invariant = false;
  for (int t = 1; t <= max_iters; ++t) {
    // un = Bv - alpha u: computed here for t = 1, afterwards by the fused pass at
    // the end of the previous iteration (same arithmetic, one A traversal less).
    // With the pair layout the first one is the fused pass too, its residual
    // half (b - A 0, into r) discarded.
    if (t == 1) {
      if (pair)
        apply_pass_dual(M, xv.p, rL, eqb::kPassResid, nullptr, b_loc, nullptr, nullptr, unL,
                        eqb::kPassLsqrU, d, u.p, sc + 1, true, slotted);
      else
        apply_pass(M, false, ev.p, unL, eqb::kPassLsqrU, d, u.p, sc + 1);
    }
    CK(cudaMemsetAsync(inv, 0, sizeof(int), s));
    L.norm(un.p, true, sc + 0);
    CK(eqb::launch_lsqr_normalize(u.p, unL, sc + 0, duL, d, L.mL, inv, nullptr, s, 1, slot_u));
    L.gather(du.p, true);
    apply_pass(M, true, du.p, vnL, eqb::kPassLsqrV, e, v.p, sc + 0, inv,
               slotted);  // B^T u - beta v
    L.norm(vn.p, false, sc + 1);
    CK(eqb::launch_lsqr_normalize(v.p, vnL, sc + 1, evL, e, L.nL, inv, inv, s, os, slot_v));
    if (!pair) gather_ev();  // pair: travels with e.x below
    CK(cudaMemcpyAsync(hs, sc, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&hs->inv, inv, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (t > 1) {  // iteration t-1's residual (:66-78)
      if (record(hs->rnorm)) return;
      if (prev_invariant) {
        st.breakdown = true;
        return;
      }
    }
    ++st.applies;
    beta = hs->beta;
    const bool u_inv = !(beta > 0.0);
    alpha = u_inv ? 0.0 : hs->alpha;
    if (!u_inv) ++st.adjoints;
    const bool invariant = u_inv || !(alpha > 0.0);
    const double rho = std::hypot(rhobar, beta);  // :58-64
    const double cs = rhobar / rho;
    const double sn = beta / rho;
    const double theta = sn * alpha;
    rhobar = -cs * alpha;
    const double phi = cs * phibar;
    phibar = sn * phibar;
    CK(eqb::launch_lsqr_xw_update(x.p, w.p, v.p, phi / rho, theta / rho, e, exL, L.nL, s, os,
                                  slot_v));
    gather_ex();
    st.iterations = t;
    // residual b - A(e.x) and, in the same traversal of A, the next iteration's
    // B v - alpha u (its inputs v, alpha, u are final here; unused if we stop)
    if (pair)
      apply_pass_dual(M, xv.p, rL, eqb::kPassResid, nullptr, b_loc, nullptr, nullptr, unL,
                      eqb::kPassLsqrU, d, u.p, sc + 1, true, slotted);
    else
      apply_pass_dual(M, ex.p, rL, eqb::kPassResid, nullptr, b_loc, nullptr, ev.p, unL,
                      eqb::kPassLsqrU, d, u.p, sc + 1);
    L.norm(r.p, true, sc + 2);
    prev_invariant = invariant;
  }
  if (st.iterations > 0) {  // the last iteration's residual
    const double rnorm = read_scalar(M, sc + 2);
    if (record(rnorm)) return;
    if (prev_invariant) st.breakdown = true;
  }
}

void lsqr_common(equil_matrix* M, const double* b, const equil_params* p, int max_iters,
                 double tol, equil_lsqr_out* out, const char* who) {
  require(M != nullptr && out != nullptr, std::string(who) + ": null argument");
  require(b != nullptr, std::string(who) + ": rhs length mismatch");
  std::lock_guard<std::mutex> lk(M->mu);
  DeviceGuard dg(M->device);
  cudaStream_t s = M->stream;
  const int64_t m = M->m, n = M->n;
  const int64_t mL = M->m_loc(), nL = M->n_loc();
  DevBuf<double> b_d;  // the whole rhs on every rank (its norm is global)
  b_d.alloc(m);
  CK(cudaMemcpyAsync(b_d.p, b, m * 8, cudaMemcpyHostToDevice, s));
  canon_reduce(M, b_d.p, m, M->scal.p + 3, 0, 0.0, true);
  const double bnorm = read_scalar(M, M->scal.p + 3);
  require(bnorm > 0.0, std::string(who) + ": rhs must be nonzero");
  require(max_iters >= 0, std::string(who) + ": max_iters must be nonnegative");
  const int T = p ? p->iterations : 0;
  require(out->residual_history != nullptr &&
              out->residual_cap >= max_iters + 1 + (p ? std::max(T, 0) : 0),
          std::string(who) + ": residual_history capacity too small");
  const double* b_loc = b_d.p + M->a_goff();
  LsqrState st;
  DevBuf<double> dd, ed, c, x;
  const double* c_ptr = b_loc;
  const double* d_loc = nullptr;
  const double* e_loc = nullptr;
  if (p) {
    // sgd_equilibrate on the charged operator (:115-116); full d, e on device
    dd.alloc(m);
    ed.alloc(n);
    equil_scaling_out so{};
    so.u = nullptr;
    so.v = nullptr;
    so.d = dd.p;
    so.e = ed.p;
    so.outputs_on_device = 1;
    M->mu.unlock();
    const equil_status rc = equil_sgd_equilibrate(M, p, nullptr, &so);
    M->mu.lock();
    if (rc != EQUIL_OK) fail(rc, g_err);
    st.applies = so.apply_count;
    st.adjoints = so.adjoint_count;
    for (int t = 0; t <= T; ++t) out->residual_history[st.hist_len++] = 1.0;  // :121-123
    d_loc = dd.p + M->a_goff();
    e_loc = ed.p + M->t_goff();
    c.alloc(mL);
    CK(eqb::launch_mul(c.p, d_loc, b_loc, mL, s));  // c = d .* b (:126)
    c_ptr = c.p;
  } else {
    out->residual_history[st.hist_len++] = 1.0;  // :94
  }
  lsqr_core(M, c_ptr, b_loc, bnorm, d_loc, e_loc, max_iters, tol, out->residual_history,
            out->residual_cap, st, x);
  // x = e .* x_scaled (:134)
  if (p) CK(eqb::launch_mul(x.p, e_loc, x.p, nL, s));
  if (out->x) {
    if (M->world == 1) {
      CK(cudaMemcpyAsync(out->x, x.p, n * 8, cudaMemcpyDeviceToHost, s));
    } else {  // gather the slices, un-pad, copy out
      DevBuf<double> pad, flat;
      pad.alloc(M->n_pad());
      flat.alloc(n);
      CK(cudaMemcpyAsync(pad.p + M->rank * M->t_max, x.p, nL * 8, cudaMemcpyDeviceToDevice, s));
      allgather_padded(M, pad.p, M->t_max);
      unpad_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
          flat.p, pad.p, M->t_bounds_d.p, M->world, M->t_max, n);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(out->x, flat.p, n * 8, cudaMemcpyDeviceToHost, s));
    }
  }
  CK(cudaStreamSynchronize(s));
  out->hist_len = st.hist_len;
  out->iterations = st.iterations;
  out->equil_iterations = p ? T : 0;
  out->reached_tol = st.reached_tol;
  out->breakdown = st.breakdown;
  out->apply_count = st.applies;
  out->adjoint_count = st.adjoints;
}

}  // namespace eqe

extern "C" {

equil_status equil_lsqr(equil_matrix* A, const double* b, int max_iters, double tol,
                        equil_lsqr_out* out) {
  return guarded([&] {
    NvtxRange nvtx_("equil:lsqr");
    lsqr_common(A, b, nullptr, max_iters, tol, out, "lsqr");
  });
}

equil_status equil_lsqr_preconditioned(equil_matrix* A, const double* b,
                                       const equil_params* p, int max_iters, double tol,
                                       equil_lsqr_out* out) {
  return guarded([&] {
    NvtxRange nvtx_("equil:lsqr_preconditioned");
    require(p != nullptr, "lsqr_preconditioned: null params");
    lsqr_common(A, b, p, max_iters, tol, out, "lsqr_preconditioned");
  });
}

equil_status equil_apply(equil_matrix* M, const double* x, double* y, int adjoint) {
  return guarded([&] {
    require(M != nullptr && x != nullptr && y != nullptr, "apply: null argument");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    require(M->world == 1, "apply: single-GPU matrices only");
    const int64_t nin = adjoint ? M->m : M->n, nout = adjoint ? M->n : M->m;
    DevBuf<double> xi, yo;
    xi.alloc(nin);
    yo.alloc(nout);
    CK(cudaMemcpyAsync(xi.p, x, nin * 8, cudaMemcpyHostToDevice, M->stream));
    apply_pass(M, adjoint != 0, xi.p, yo.p, eqb::kPassPlain, nullptr, nullptr, nullptr);
    CK(cudaMemcpyAsync(y, yo.p, nout * 8, cudaMemcpyDeviceToHost, M->stream));
    CK(cudaStreamSynchronize(M->stream));
  });
}

equil_status equil_export_transpose(equil_matrix* M, int64_t* t_row_ptr, int32_t* t_col,
                                    double* t_val) {
  return guarded([&] {
    require(M != nullptr, "export_transpose: null handle");
    require(!M->dense && M->world == 1, "export_transpose: single-GPU sparse matrices only");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    CK(cudaMemcpy(t_row_ptr, M->AT.row_ptr, (M->n + 1) * 8, cudaMemcpyDeviceToHost));
    if (M->nnz) {
      CK(cudaMemcpy(t_col, M->AT.col, M->nnz * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(t_val, M->AT.val, M->nnz * 8, cudaMemcpyDeviceToHost));
    }
  });
}

equil_status equil_sign_bits(uint64_t seed, uint64_t stream, uint64_t start,
                             uint64_t count, uint32_t* bits_out, int device) {
  return guarded([&] {
    require(bits_out != nullptr || count == 0, "sign_bits: null output");
    if (count == 0) return;
    DeviceGuard dg(device);
    const uint64_t total = start + count;
    DevBuf<uint32_t> bits;
    DevBuf<unsigned char> scratch;
    bits.alloc((total + 31) / 32 + 1);
    const size_t sb = eqb::sign_stream_scratch_bytes(total);
    scratch.alloc(sb);
    CK(eqb::sign_stream_generate(seed, stream, total, bits.p, scratch.p, sb, 0));
    std::vector<uint32_t> all((total + 31) / 32 + 1, 0);
    CK(cudaMemcpy(all.data(), bits.p, ((total + 31) / 32) * 4, cudaMemcpyDeviceToHost));
    const uint64_t nw = (count + 31) / 32;
    for (uint64_t w = 0; w < nw; ++w) {
      uint32_t word = 0;
      for (int k = 0; k < 32; ++k) {
        const uint64_t o = w * 32 + k;
        if (o >= count) break;
        const uint64_t g = start + o;
        if ((all[g >> 5] >> (g & 31)) & 1u) word |= 1u << k;
      }
      bits_out[w] = word;
    }
  });
}

equil_status equil_det_exp_device(const double* x, double* y, int64_t n, int device) {
  return guarded([&] {
    if (n <= 0) return;
    DeviceGuard dg(device);
    DevBuf<double> a, b;
    a.alloc(n);
    b.alloc(n);
    CK(cudaMemcpy(a.p, x, n * 8, cudaMemcpyHostToDevice));
    CK(eqb::launch_exp(a.p, b.p, n, 1.0, 0));
    CK(cudaMemcpy(y, b.p, n * 8, cudaMemcpyDeviceToHost));
  });
}

equil_status equil_canon_sumsq_device(const double* x, int64_t n, double* out, int device) {
  return guarded([&] {
    DeviceGuard dg(device);
    DevBuf<double> a, part, res;
    DevBuf<unsigned> cnt;
    a.alloc(std::max<int64_t>(n, 1));
    part.alloc((n + eqb::kChunk - 1) / eqb::kChunk + 1);
    res.alloc(1);
    cnt.alloc(1);
    CK(cudaMemset(cnt.p, 0, 4));
    if (n > 0) CK(cudaMemcpy(a.p, x, n * 8, cudaMemcpyHostToDevice));
    CK(eqb::launch_canon_reduce(a.p, n, 0, 0.0, part.p, cnt.p, res.p, 0, 0));
    CK(cudaMemcpy(out, res.p, 8, cudaMemcpyDeviceToHost));
  });
}

equil_status equil_sgd_equilibrate_csr(int64_t m, int64_t n, const int64_t* row_ptr,
                                       const int32_t* col, const double* val,
                                       const equil_params* p, const equil_device_cfg* cfg,
                                       equil_scaling_out* out) {
  equil_matrix* M = nullptr;
  // the sign stream depends only on (seed, T, m + n): generate it while the
  // matrix is built (invalid parameters are reported by the call below first)
  eqe::PreSigns pre{0, 0};
  if (p && equil_validate_params(p) == EQUIL_OK && m > 0 && n > 0)
    pre = {p->seed, static_cast<uint64_t>(m + n) * static_cast<uint64_t>(p->iterations)};
  equil_status rc = create_csr_impl(m, n, row_ptr, col, val, cfg, &M, &pre);
  if (rc != EQUIL_OK) return rc;
  M->oneshot = true;  // one call on this handle: launch the loop directly, no graph
  rc = equil_sgd_equilibrate(M, p, nullptr, out);
  const auto t0 = std::chrono::steady_clock::now();
  equil_matrix_destroy(M);
  if (const char* e = getenv("EQUIL_VERBOSE"))
    if (atoi(e) >= 2)
      fprintf(stderr, "[equil] one-shot destroy %.2f ms\n",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                  .count());
  return rc;
}

}  // extern "C"

