// engine_internal.h -- shared internals of the host engine (engine.cu,
// engine_ext.cu): error plumbing of the C ABI, pooled device buffers, the
// parameter rules of src/params.cpp, the traversal plan types and the
// equil_matrix handle itself.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <map>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <future>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/equil_b200.h"
#include "internal.h"
#include "mmio.h"
#include "mt64_host.h"

// ---------------------------------------------------------------------------
// NCCL, resolved at run time (the process that drives us -- e.g. torch -- has
// usually loaded libnccl.so.2 already; dlopen then returns that copy).
// ---------------------------------------------------------------------------
namespace eqe {
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
constexpr int ncclUint8 = 1, ncclInt32 = 2, ncclUint32 = 3, ncclInt64 = 4, ncclFloat64 = 8;
constexpr int ncclSum = 0, ncclMax = 2, ncclMin = 3;

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

inline NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(api.h, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(api.h, "ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(api.h, "ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(api.h, "ncclAllGather"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(api.h, "ncclAllReduce"));
    api.Send = reinterpret_cast<decltype(api.Send)>(dlsym(api.h, "ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(dlsym(api.h, "ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(api.h, "ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(api.h, "ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(api.h, "ncclGetErrorString"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather &&
             api.AllReduce && api.Send && api.Recv && api.GroupStart && api.GroupEnd;
  });
  return api;
}

inline thread_local std::string g_err;

struct Fail {
  equil_status code;
  std::string msg;
};

[[noreturn]] inline void fail(equil_status c, const std::string& m) { throw Fail{c, m}; }
inline void require(bool c, const std::string& m) {
  if (!c) fail(EQUIL_EINVAL, m);
}
inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(e == cudaErrorMemoryAllocation ? EQUIL_ENOMEM : EQUIL_ECUDA,
         std::string(what) + ": " + cudaGetErrorString(e));
  }
}
#define CK(x) cuda_check((x), #x)
// Host -> device copy ordered on stream s and complete on return.  A plain
// cudaMemcpy from pageable memory may return before its DMA has landed, and it
// runs on the legacy stream, which our non-blocking streams do not wait for.
inline void h2d_sync(cudaStream_t s, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return;
  cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s), "cudaMemcpyAsync");
  cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
}
inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != 0) {
    const char* s = nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error";
    fail(EQUIL_ENCCL, std::string(what) + ": " + s);
  }
}

template <class F>
equil_status guarded(F&& f) {
  try {
    f();
    return EQUIL_OK;
  } catch (const Fail& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return EQUIL_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return EQUIL_ERUNTIME;
  }
}

// NVTX range for profilers (nsys / ncu --nvtx): one per C ABI call and phase
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// EQUIL_VERBOSE=1: per-phase wall times of setup calls (synchronizing; debug
// only).  EQUIL_VERBOSE=2: a non-synchronizing timeline instead -- each mark
// records the host time and an event on the given stream; at the end every
// mark prints both, relative to the first (the device times need the events
// to have completed, so they are printed when the timer goes out of scope).
struct PhaseTimer {
  const char* what;
  int mode;
  std::chrono::steady_clock::time_point t, t0;
  struct Rec {
    const char* phase;
    double host_ms;
    cudaEvent_t ev;
  };
  std::vector<Rec> recs;
  cudaEvent_t e0 = nullptr;
  explicit PhaseTimer(const char* w)
      : what(w), mode(getenv("EQUIL_VERBOSE") ? atoi(getenv("EQUIL_VERBOSE")) : 0),
        t(std::chrono::steady_clock::now()), t0(t) {
    if (getenv("EQUIL_VERBOSE") && mode == 0) mode = 1;
  }
  void mark(cudaStream_t s, const char* phase) {
    nvtxMarkA(phase);
    if (mode == 0) return;
    const auto now = std::chrono::steady_clock::now();
    if (mode == 2) {
      cudaEvent_t e = nullptr;
      if (!e0) {
        cudaEventCreate(&e0);
        cudaEventRecord(e0, s);
      }
      cudaEventCreate(&e);
      cudaEventRecord(e, s);
      recs.push_back({phase, std::chrono::duration<double, std::milli>(now - t0).count(), e});
      return;
    }
    cudaStreamSynchronize(s);
    const auto after = std::chrono::steady_clock::now();
    fprintf(stderr, "[equil] %s %-14s %8.2f ms\n", what, phase,
            std::chrono::duration<double, std::milli>(after - t).count());
    t = after;
  }
  ~PhaseTimer() {
    if (mode != 2) return;
    for (const Rec& r : recs) {
      float ms = -1.0f;
      if (cudaEventSynchronize(r.ev) == cudaSuccess) cudaEventElapsedTime(&ms, e0, r.ev);
      fprintf(stderr, "[equil] %s %-14s host %8.2f ms  device %8.2f ms\n", what, r.phase,
              r.host_ms, static_cast<double>(ms));
      cudaEventDestroy(r.ev);
    }
    if (e0) cudaEventDestroy(e0);
    cudaGetLastError();
  }
};

// Device buffers come from the device's stream-ordered memory pool (release
// threshold kept at max), allocated on a private per-device stream and made
// visible before use, so repeated matrix setups reuse already-mapped memory
// instead of paying cudaMalloc / cudaFree page mapping every time.  Release
// keeps cudaFree's semantics: the device is synchronised before the memory goes
// back to the pool.
inline cudaStream_t alloc_stream(int dev) {
  static std::mutex mu;
  static cudaStream_t streams[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!streams[dev]) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      // an allocation must never wait on another stream's pending frees (setup
      // allocates on alloc_stream while the matrix stream is busy)
      int no = 0;
      cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
    }
    cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking);
    cudaGetLastError();
  }
  return streams[dev];
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  int dev = -1;         // >= 0: pool allocation on alloc_stream(dev)
  cudaStream_t own = nullptr;  // alloc_on: stream-ordered on this stream
  // a temporary used only on stream s (setup): stream-ordered allocation and
  // free, no synchronisation on either side; s must outlive the buffer
  void alloc_on(size_t count, cudaStream_t s) {
    release();
    if (count == 0) count = 1;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s));
    own = s;
    n = count;
  }
  void alloc(size_t count) {
    release();
    if (count == 0) count = 1;
    int d = 0;
    CK(cudaGetDevice(&d));
    cudaStream_t s = alloc_stream(d);
    CK(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s));
    CK(cudaStreamSynchronize(s));
    dev = d;
    n = count;
  }
  // A persistent buffer first used on stream s (setup): the allocation is
  // ordered on s, so it reuses memory that earlier temporaries of s freed and
  // the host does not wait; other streams must be ordered after this point of
  // s before they touch it.  Freed like alloc()'s buffers (device sync first).
  void alloc_async(size_t count, cudaStream_t s) {
    release();
    if (count == 0) count = 1;
    int d = 0;
    CK(cudaGetDevice(&d));
    CK(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s));
    dev = d;
    n = count;
  }
  // free in the order of stream s (every use of the buffer was on s): no device sync
  void release_on(cudaStream_t s) {
    if (p && !own && dev >= 0) {
      cudaFreeAsync(p, s);
      p = nullptr;
      n = 0;
      dev = -1;
      return;
    }
    release();
  }
  void adopt(T* q, size_t count) {  // take ownership of a cudaMalloc'ed array
    release();
    p = q;
    n = count;
    dev = -1;
  }
  void ensure(size_t count) {
    if (count > n || !p) alloc(count);
  }
  void release() {
    if (p && own) {
      cudaFreeAsync(p, own);
      p = nullptr;
      own = nullptr;
      n = 0;
      return;
    }
    if (p) {
      if (dev >= 0) {
        int cur = 0;
        cudaGetDevice(&cur);
        if (cur != dev) cudaSetDevice(dev);
        cudaDeviceSynchronize();  // like cudaFree: nothing may still use p
        cudaFreeAsync(p, alloc_stream(dev));
        if (cur != dev) cudaSetDevice(cur);
      } else {
        cudaFree(p);
      }
    }
    p = nullptr;
    n = 0;
    dev = -1;
  }
  void swap(DevBuf& o) {
    std::swap(p, o.p);
    std::swap(n, o.n);
    std::swap(dev, o.dev);
    std::swap(own, o.own);
  }
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) CK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// ---- params (src/params.cpp:7-44) -----------------------------------------
inline void resolve_targets(const equil_params& p, int64_t rows, int64_t cols,
                     double& alpha, double& beta) {
  require(rows > 0 && cols > 0, "resolve_targets: dimensions must be positive");
  require(p.alpha >= 0.0 && p.beta >= 0.0,
          "resolve_targets: targets must be positive (or 0 for auto)");
  const double m = static_cast<double>(rows);
  const double n = static_cast<double>(cols);
  alpha = p.alpha;
  beta = p.beta;
  if (alpha == 0.0 && beta == 0.0) {
    alpha = std::pow(n / m, 0.25);
    beta = std::pow(m / n, 0.25);
  } else if (beta == 0.0) {
    beta = alpha * std::sqrt(m / n);
  } else if (alpha == 0.0) {
    alpha = beta * std::sqrt(n / m);
  } else {
    const double lhs = m * alpha * alpha;
    const double rhs = n * beta * beta;
    require(std::abs(lhs - rhs) <= 1e-8 * std::max(lhs, rhs),
            "resolve_targets: m*alpha^2 == n*beta^2 violated");
  }
}

inline void validate_params(const equil_params& p) {
  require(p.gamma > 0.0, "params: gamma must be positive");
  require(p.max_log_scale > 0.0, "params: max_log_scale must be positive");
  require(p.iterations >= 0, "params: iterations must be nonnegative");
  require(std::isfinite(p.gamma) && std::isfinite(p.max_log_scale),
          "params: gamma and max_log_scale must be finite");
}

// ---- traversal plan ---------------------------------------------------------
// Rows longer than kTileNnz become kind-3 long slices (32 length-sorted rows
// per CTA); all other rows are grouped into kind-2 slices: within windows of
// kSliceWindow consecutive rows, rows are sorted by length (longest first) and
// cut into groups of 32, so the lanes of a slice have similar chain lengths and
// the epilogue's scattered writes stay inside one window.  The row order never
// affects results: each row is an independent sequential sum.  Windows are
// planned in parallel host threads; the result does not depend on the thread
// count (parts are concatenated in window order, ties keep row order).
// The interleaved-slice plan (sell.cu) reuses the same row groups: every
// kind-3 group and every kind-2 slice becomes one slice (plan_sell orders them).
struct SellEnt {
  int32_t maxlen;  // entries of the group's longest row
  int16_t cnt;     // rows
  int16_t lng;     // a kind-3 group (rows longer than kTileNnz)
  int32_t r0;      // first row in rowlist
};
struct Plan {
  int64_t long_nnz = 0;  // entries of the rows longer than kTileNnz
  std::vector<eqb::Tile> lng, slices;
  std::vector<int32_t> rowlist;
  std::vector<SellEnt> sell;
};

Plan plan_tiles(const int64_t* rp, int64_t rows, int mat);
std::vector<int64_t> partition_rows(const int64_t* rp, int64_t rows, int parts);

}  // namespace eqe

namespace eqe {
// In-process rank exchange used instead of NCCL when EQUIL_HOST_EXCHANGE=1:
// several rank handles of one sharded matrix live in one process (one thread
// each, e.g. all on one GPU in a test) and meet on the host -- a barrier on a
// condition variable, slices passed through host buffers.  No kernel ever
// waits on another rank; the sharded engine's index arithmetic, padding and
// reductions run exactly as with NCCL.
// Host-side exchange among the ranks of a sharded matrix for tests and
// single-GPU runs of the sharded engine (no NCCL): put() publishes this rank's
// bytes, barrier(), then slot(g) reads rank g's.  ThreadExchange: ranks are
// threads of one process (EQUIL_HOST_EXCHANGE=1).  ShmExchange: ranks are
// processes (EQUIL_HOST_EXCHANGE=2), POSIX shared memory + a process-shared
// barrier; peers' gathered-vector buffers are then mapped over CUDA IPC, as
// they are with NCCL.
struct HostExchange {
  int world = 0;
  virtual ~HostExchange() = default;
  virtual void barrier() = 0;
  virtual void put(int rank, const void* data, size_t bytes) = 0;
  virtual const char* slot(int g) = 0;
  virtual bool in_process() const = 0;
  virtual size_t capacity() const = 0;  // bytes one put may carry
};
struct ThreadExchange : HostExchange {
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<std::vector<char>> slots;
  void barrier() override {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
  void put(int rank, const void* data, size_t bytes) override {
    slots[rank].assign(static_cast<const char*>(data), static_cast<const char*>(data) + bytes);
  }
  const char* slot(int g) override { return slots[g].data(); }
  bool in_process() const override { return true; }
  size_t capacity() const override { return SIZE_MAX; }
};
std::shared_ptr<HostExchange> shm_exchange(const void* id128, int world, int rank);
inline std::shared_ptr<HostExchange> host_exchange(const void* id128, int world) {
  static std::mutex mu;
  static std::map<std::string, std::weak_ptr<HostExchange>> reg;
  std::lock_guard<std::mutex> lk(mu);
  const std::string key(static_cast<const char*>(id128), 128);
  auto hx = reg[key].lock();
  if (!hx) {
    auto t = std::make_shared<ThreadExchange>();
    t->world = world;
    t->slots.resize(world);
    hx = t;
    reg[key] = hx;
  }
  return hx;
}
}  // namespace eqe

// The device-resident matrix behind the opaque handle of include/equil_b200.h.
using namespace eqe;
// ---------------------------------------------------------------------------
struct equil_matrix {
  int device = 0, rank = 0, world = 1;
  bool dense = false;
  int64_t m = 0, n = 0, nnz = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // uploads that overlap work on `stream`
  cudaEvent_t ev_vals = nullptr;       // values of A on the device
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // one-shot calls (equil_sgd_equilibrate_csr) know the seed and T before the
  // matrix is built: the sign stream is generated on a high-priority side
  // stream while the matrix uploads and transposes; sgd_row_col then only
  // waits on sign_ev (pre_* describe what was generated)
  cudaStream_t sign_stream = nullptr;
  cudaEvent_t sign_ev = nullptr;
  bool pre_signs = false;
  uint64_t pre_seed = 0, pre_total = 0;
  std::mutex mu;
  ncclComm_t comm = nullptr;
  std::shared_ptr<eqe::HostExchange> hx;  // EQUIL_HOST_EXCHANGE=1 instead of comm

  // sparse shards (local rows, columns in padded coordinates)
  eqb::DevCsr A, AT;
  DevBuf<int64_t> a_rp, t_rp;
  DevBuf<int32_t> a_ci, t_ci;
  DevBuf<double> a_va, t_va;
  std::vector<int64_t> a_bounds, t_bounds;  // partitions of rows / columns
  int64_t a_max = 0, t_max = 0;             // padded slice sizes
  DevBuf<int64_t> a_bounds_d, t_bounds_d;
  DevBuf<eqb::Tile> tiles_sgd, tiles_a, tiles_t;
  DevBuf<int32_t> rowlist_a, rowlist_t;
  int n_sgd = 0, n_a = 0, n_t = 0;
  int n_sgd_long = 0;  // leading kind-3 entries of tiles_sgd
  int n_la = 0, n_sa = 0;  // A's kind-3 entries / A's warp slices in tiles_sgd
  // L2 persisting window of the gathered vectors (alloc_workspaces): carve-out,
  // device maximum window, default window bytes (xbuf); with column blocks each
  // launch's window is its block (EQUIL_BLOCK_WIN)
  size_t l2_carve = 0, l2_max_window = 0, l2_default_bytes = 0;
  bool block_win = true;
  // hot-first slot layout of the gathered vectors (build_slot_layout): the SGD
  // passes read CSR copies whose column indices point at slots, and the
  // epilogues write each row's next value at its slot
  bool use_slots = true;
  bool slots = false;
  DevBuf<int32_t> a_ci_sgd, t_ci_sgd, wmap, smap;
  // interleaved row slices of the SGD passes (sell.cu, build_sell_layout):
  // the default traversal when the slot layout is on and nothing is blocked;
  // EQUIL_SELL=0 keeps the staged warp tiles / CTA long slices
  bool use_sell = true;
  bool sell = false;
  // rows longer than kTileNnz (EQUIL_SELL_LONG): 0 kind-3 CTA groups on the
  // CSR arrays, 1 lane chains in the warp kernel, 2 warp-specialised CTAs
  // (sgd_sell_long_kernel) on the interleaved arrays
  int sell_long = 2;
  // long slices in the quad layout (128-bit stream loads; EQUIL_SELL_QUAD=0: 1-wide)
  bool sell_quad = true;
  int sell_variant = 0, sell_lvariant = 0;
  int n_sell_long = 0;  // leading slices with rows longer than kTileNnz
  int sell_order = 0;   // EQUIL_SELL_ORDER: warp slices longest first (0) / in window order (1)
  // EQUIL_SELL_BLOCKED=1: interleaved slices also with column blocks (c5: 17.8
  // vs 17.3 ms per iteration for the staged blocks, so off by default)
  bool sell_blocked = false;
  struct SellHost {
    std::vector<eqb::SellSlice> slices;
    std::vector<int32_t> r0;  // first row of each slice in its matrix's row list
    int64_t total[2] = {0, 0};
    // per matrix: its slices in launch order (indices into slices) and the
    // prefix of their 32-entry blocks (the device build's work items)
    std::vector<int32_t> midx[2];
    std::vector<int64_t> kbp[2];
    // per matrix: every slice in launch order (passes over one matrix) and
    // how many of them lead with rows longer than kTileNnz
    std::vector<int32_t> pidx[2];
    int plong[2] = {0, 0};
  } sell_host;
  DevBuf<eqb::SellSlice> sell_slices;
  DevBuf<int32_t> sell_row, sell_len, sell_ci[2];
  DevBuf<double> sell_va[2];
  int n_sell = 0;
  // column blocks (sell_nb > 1): per-block slice tables and lane counts,
  // block-major arrays, the running sums carried between block rounds
  int sell_nb = 1;
  DevBuf<eqb::SellSlice> sell_bslices;
  DevBuf<int32_t> sell_bln;
  DevBuf<double> sell_carry;
  // the generic passes (LSQR, apply, variants) over the same slices: columns
  // in padded coordinates (their vectors are not in slot layout), built on
  // first use; values shared with the SGD arrays
  // split epilogue (EQUIL_SPLIT_EPI): row sums to rowacc, then one update pass
  bool split_epi = true;
  DevBuf<double> rowacc;
  // column-synchronous sweep of A's long rows (sweep.cu, build_sweep_layout;
  // EQUIL_SWEEP=0 keeps the warp-specialised long-slice kernel for them)
  bool use_sweep = true;
  bool sweep_forced = false;  // EQUIL_SWEEP=1: also for one-shot calls of few iterations
  bool sweep = false;
  bool sweep_values_pending = false;
  int sweep_width = 0, sweep_stages = 2;  // width 0: sized from the rows (EQUIL_SWEEP_WIDTH)
  bool sweep_candidate = false;  // decided before the slot maps: xs keeps column order
  int64_t sweep_long_nnz = 0;
  std::vector<int32_t> sweep_rows_host;  // A's rows longer than kTileNnz, longest first
  bool oneshot_hint = false;    // created by the one-shot entry point
  bool sell_skip_long = false;  // A's long interleaved slices not built (the sweep serves them)
  bool sweep_plan_ok = false;  // plan_sweep_layout enqueued; build_sweep_layout finishes it
  int sweep_plan_G = 0, sweep_plan_R = 0, sweep_plan_W = 0;
  uint32_t* sweep_ne_host = nullptr;  // pinned (thread-cached): per-(CTA, panel) padded entry counts
  cudaEvent_t ev_sweep = nullptr;
  eqb::SweepArgs sweep_args{};
  DevBuf<unsigned char> sweep_blobs;
  DevBuf<int64_t> sweep_off;
  DevBuf<int32_t> sweep_crow, sweep_rstart;
  DevBuf<uint16_t> sweep_perm, sweep_srun;
  DevBuf<uint32_t> sweep_gbase, sweep_nepad;
  bool sell_passes = true;
  bool sell_values_pending = false;  // interleaved values not built yet (setup)  // EQUIL_SELL_PASSES=0: generic passes on the staged kernels
  bool sell_pass = false;
  bool sell_order_up = false;  // sell_pidx uploaded
  DevBuf<int32_t> sell_pci[2], sell_pidx[2];
  // column blocks of the gathered vectors (build_block_layout): per matrix
  int nblk[2] = {1, 1};
  int64_t bwidth[2] = {0, 0};
  DevBuf<int32_t> bnd[2];
  DevBuf<double> carry[2];  // wmap / smap: padded position -> slot

  // dense
  DevBuf<double> Ad, colpart;
  DevBuf<unsigned> colcnt;  // dense column strips: chunk CTAs done (dense.cu)

  // workspaces
  // padded gathered vectors e.*s (xs) and d.*w (xw), double-buffered, in one
  // allocation so a single L2 persisting window covers every gather target
  struct Slot {
    double* p = nullptr;
  } xs[2], xw[2];
  DevBuf<double> xbuf;  // cudaMalloc'ed when world > 1 (exportable over CUDA IPC)
  // fused all-gather of the SGD loop (setup_peers): every peer's xbuf as an
  // element offset from ours; p2p_state 0: not negotiated, 1: on, -1: off
  int p2p_state = 0;
  std::vector<int64_t> peer_delta;
  std::vector<void*> peer_mapped;  // IPC mappings, closed on destroy
  DevBuf<unsigned> bar;            // barrier word (EQUIL_P2P_BARRIER=nccl)
  int64_t xbar_off = 0;            // device barrier words: xbuf tail (eqb::kBarWords)
  unsigned long long* xbar() { return reinterpret_cast<unsigned long long*>(xbuf.p + xbar_off); }
  DevBuf<double> u, ub, v, vb;  // local
  DevBuf<uint32_t> signs;
  DevBuf<unsigned char> sign_scratch;
  DevBuf<unsigned> flags;
  DevBuf<double> red_part;
  DevBuf<unsigned> red_counter;
  DevBuf<double> scal;  // small device scalars
  struct LsqrSync {     // LSQR's per-iteration host read (pinned)
    double beta, alpha, rnorm;
    int inv;
  };
  LsqrSync* lsqr_sync = nullptr;
  bool pull_uploads = false;  // setup: host -> device copies by pull kernels (h2d)
  DevBuf<double> tmp_m, tmp_n, tmp_m2, tmp_n2;
  DevBuf<double> lin_u, lin_v;  // per-coordinate targets (sgd_equilibrate_targets)

  // graph cache for the SGD loop (not built for a one-shot handle, whose
  // single call would pay capture and instantiation for one replay)
  bool oneshot = false;
  cudaGraphExec_t graph = nullptr;
  long long graph_launches = 0;  // kernel nodes per replay
  struct Key {
    int T = -1;
    double alpha = 0, beta = 0, gamma = 0, M = 0;
    bool vec_lin = false;
    bool operator==(const Key& o) const {
      return T == o.T && alpha == o.alpha && beta == o.beta && gamma == o.gamma && M == o.M &&
             vec_lin == o.vec_lin;
    }
  } graph_key;

  int64_t m_loc() const { return dense ? m : a_bounds[rank + 1] - a_bounds[rank]; }
  int64_t n_loc() const { return dense ? n : t_bounds[rank + 1] - t_bounds[rank]; }
  int64_t a_goff() const { return dense ? 0 : a_bounds[rank]; }
  int64_t t_goff() const { return dense ? 0 : t_bounds[rank]; }
  int64_t m_pad() const { return world == 1 ? m : a_max * world; }
  int64_t n_pad() const { return world == 1 ? n : t_max * world; }

  // events bracketing the T-iteration loop of the last sgd call (also inside
  // the captured graph), for the live per-kernel roofline in bench.py
  cudaEvent_t ev_loop0 = nullptr, ev_loop1 = nullptr;
  double last_loop_ms = 0.0;
  int last_loop_iters = 0;

  ~equil_matrix() {
    if (lsqr_sync) cudaFreeHost(lsqr_sync);
    if (ev_loop0) cudaEventDestroy(ev_loop0);
    if (ev_loop1) cudaEventDestroy(ev_loop1);
    if (ev_sweep) cudaEventDestroy(ev_sweep);
    if (graph) cudaGraphExecDestroy(graph);
    for (void* q : peer_mapped) cudaIpcCloseMemHandle(q);
    if (comm && nccl().ok) nccl().CommDestroy(comm);
    if (ev_vals) cudaEventDestroy(ev_vals);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (sign_ev) cudaEventDestroy(sign_ev);
    if (sign_stream) cudaStreamDestroy(sign_stream);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (stream) cudaStreamDestroy(stream);
  }
};


namespace eqe {
// defined in engine.cu, used by the extension entry points (engine_ext.cu)
void set_l2_window(equil_matrix* M, cudaStream_t st, const void* base, size_t bytes);
void canon_reduce(equil_matrix* M, const double* x, int64_t len, double* out, int kind,
                  double coef = 0.0, bool sqrt_out = false);
void apply_pass(equil_matrix* M, bool adjoint, const double* xg, double* out, int mode,
                const double* scale, const double* prev, const double* coef,
                const int* skip = nullptr, bool slotted = false);
double read_scalar(equil_matrix* M, const double* dev);
// host -> device copy on M->stream: a pull kernel from a thread-local mapped
// pinned arena while M->pull_uploads (setup, A's values on the copy engine),
// else cudaMemcpyAsync
void h2d(equil_matrix* M, void* dst, const void* src, size_t bytes);
void pull_arena_reset();
void create_coo_impl(int64_t m, int64_t n, int64_t nnz, const int64_t* rows,
                     const int64_t* cols, const double* vals, const int64_t* lines,
                     const equil_device_cfg* cfg, equil_matrix** out);
}  // namespace eqe
