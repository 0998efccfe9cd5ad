// engine.cu -- host engine and C ABI (include/equil_b200.h).
//
// Owns the device-resident matrix (CSR(A), CSR(A^T) shards or dense A), the
// traversal plans, the sign stream and the SGD / LSQR drivers.  The T-iteration
// SGD loop is captured once as a CUDA graph per (T, targets, gamma, M) and
// replayed; LSQR keeps its scalar recurrence on the host (std::hypot, exactly
// as src/lsqr.cpp:58-64) with one device->host round trip per iteration.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/equil_b200.h"
#include "internal.h"
#include "mmio.h"
#include "mt64_host.h"

// ---------------------------------------------------------------------------
// NCCL, resolved at run time (the process that drives us -- e.g. torch -- has
// usually loaded libnccl.so.2 already; dlopen then returns that copy).
// ---------------------------------------------------------------------------
namespace {
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
constexpr int ncclUint8 = 1, ncclUint32 = 3, ncclFloat64 = 8, ncclMax = 2;

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& nccl() {
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
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(api.h, "ncclGetErrorString"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather &&
             api.AllReduce;
  });
  return api;
}

thread_local std::string g_err;

struct Fail {
  equil_status code;
  std::string msg;
};

[[noreturn]] void fail(equil_status c, const std::string& m) { throw Fail{c, m}; }
void require(bool c, const std::string& m) {
  if (!c) fail(EQUIL_EINVAL, m);
}
void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(e == cudaErrorMemoryAllocation ? EQUIL_ENOMEM : EQUIL_ECUDA,
         std::string(what) + ": " + cudaGetErrorString(e));
  }
}
#define CK(x) cuda_check((x), #x)
void nccl_check(ncclResult_t r, const char* what) {
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

// EQUIL_VERBOSE=1: per-phase wall times of setup calls (synchronizing; debug only)
struct PhaseTimer {
  const char* what;
  bool on;
  std::chrono::steady_clock::time_point t;
  explicit PhaseTimer(const char* w)
      : what(w), on(getenv("EQUIL_VERBOSE") != nullptr), t(std::chrono::steady_clock::now()) {}
  void mark(cudaStream_t s, const char* phase) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[equil] %s %-14s %8.2f ms\n", what, phase,
            std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// Device buffers come from the device's stream-ordered memory pool (release
// threshold kept at max), allocated on a private per-device stream and made
// visible before use, so repeated matrix setups reuse already-mapped memory
// instead of paying cudaMalloc / cudaFree page mapping every time.  Release
// keeps cudaFree's semantics: the device is synchronised before the memory goes
// back to the pool.
cudaStream_t alloc_stream(int dev) {
  static std::mutex mu;
  static cudaStream_t streams[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!streams[dev]) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
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
void resolve_targets(const equil_params& p, int64_t rows, int64_t cols,
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

void validate_params(const equil_params& p) {
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
struct Plan {
  std::vector<eqb::Tile> lng, slices;
  std::vector<int32_t> rowlist;
};

Plan plan_tiles(const int64_t* rp, int64_t rows, int mat) {
  Plan P;
  const int64_t nwin = (rows + eqb::kSliceWindow - 1) / eqb::kSliceWindow;
  const int nth = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()), nwin / 8)));
  struct Part {
    std::vector<eqb::Tile> slices;
    std::vector<int32_t> rowlist;
    std::vector<std::pair<int64_t, int64_t>> longs;
  };
  std::vector<Part> parts(nth);
  auto work = [&](int t) {
    Part& pt = parts[t];
    const int64_t wa = nwin * t / nth, wb = nwin * (t + 1) / nth;
    std::vector<std::pair<int64_t, int32_t>> win;
    for (int64_t w = wa; w < wb; ++w) {
      const int64_t w0 = w * eqb::kSliceWindow;
      const int64_t w1 = std::min<int64_t>(rows, w0 + eqb::kSliceWindow);
      win.clear();
      for (int64_t i = w0; i < w1; ++i) {
        const int64_t len = rp[i + 1] - rp[i];
        if (len > eqb::kTileNnz)
          pt.longs.push_back({len, i});
        else
          win.push_back({len, static_cast<int32_t>(i)});
      }
      std::stable_sort(win.begin(), win.end(),
                       [](const auto& a, const auto& b) { return a.first > b.first; });
      for (size_t q = 0; q < win.size(); q += eqb::kSliceRows) {
        const int cnt = static_cast<int>(std::min<size_t>(eqb::kSliceRows, win.size() - q));
        pt.slices.push_back({static_cast<int32_t>(pt.rowlist.size()), cnt, 2,
                             static_cast<int16_t>(mat), 0});
        for (int k = 0; k < cnt; ++k) pt.rowlist.push_back(win[q + k].second);
      }
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nth; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  std::vector<std::pair<int64_t, int64_t>> longs;
  for (Part& pt : parts) {
    const int32_t base = static_cast<int32_t>(P.rowlist.size());
    for (eqb::Tile s : pt.slices) {
      s.r0 += base;
      P.slices.push_back(s);
    }
    P.rowlist.insert(P.rowlist.end(), pt.rowlist.begin(), pt.rowlist.end());
    longs.insert(longs.end(), pt.longs.begin(), pt.longs.end());
  }
  // rows longer than a tile: CTA-cooperative long slices of 32 length-sorted
  // rows (kind 3), each replicated once per warp of the CTA
  std::stable_sort(longs.begin(), longs.end(),
                   [](const auto& a, const auto& b) { return a.first > b.first; });
  for (size_t q = 0; q < longs.size(); q += eqb::kLongRows) {
    const int cnt = static_cast<int>(std::min<size_t>(eqb::kLongRows, longs.size() - q));
    const eqb::Tile t{static_cast<int32_t>(P.rowlist.size()), cnt, 3,
                      static_cast<int16_t>(mat), 0};
    for (int k = 0; k < cnt; ++k) P.rowlist.push_back(static_cast<int32_t>(longs[q + k].second));
    for (int w = 0; w < eqb::kTileWarps; ++w) P.lng.push_back(t);
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

}  // namespace

// ---------------------------------------------------------------------------
struct equil_matrix {
  int device = 0, rank = 0, world = 1;
  bool dense = false;
  int64_t m = 0, n = 0, nnz = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // uploads that overlap work on `stream`
  cudaEvent_t ev_vals = nullptr;       // values of A on the device
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::mutex mu;
  ncclComm_t comm = nullptr;

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
  // column-panel layout of the local A / A^T shards (panel.cu), built when
  // EQUIL_PANEL=1 at creation; n_pbands == 0 selects the row-slice traversal
  // above (the default: faster on B200)
  bool use_panels = false;
  // hot-first slot layout of the gathered vectors (build_slot_layout): the SGD
  // passes read CSR copies whose column indices point at slots, and the
  // epilogues write each row's next value at its slot
  bool use_slots = true;
  bool slots = false;
  DevBuf<int32_t> a_ci_sgd, t_ci_sgd, wmap, smap;  // wmap / smap: padded position -> slot
  DevBuf<double> pval[2];
  DevBuf<uint16_t> pcol[2];
  DevBuf<uint32_t> pruns[2];
  DevBuf<eqb::PanelChunk> pchunks[2];
  DevBuf<eqb::PanelBand> pbands;
  int n_pbands = 0;

  // dense
  DevBuf<double> Ad, colpart;

  // workspaces
  // padded gathered vectors e.*s (xs) and d.*w (xw), double-buffered, in one
  // allocation so a single L2 persisting window covers every gather target
  struct Slot {
    double* p = nullptr;
  } xs[2], xw[2];
  DevBuf<double> xbuf;
  DevBuf<double> u, ub, v, vb;  // local
  DevBuf<uint32_t> signs;
  DevBuf<unsigned char> sign_scratch;
  DevBuf<unsigned> flags;
  DevBuf<double> red_part;
  DevBuf<unsigned> red_counter;
  DevBuf<double> scal;  // small device scalars
  DevBuf<double> tmp_m, tmp_n, tmp_m2, tmp_n2;
  DevBuf<double> lin_u, lin_v;  // per-coordinate targets (sgd_equilibrate_targets)

  // graph cache for the SGD loop
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
    if (ev_loop0) cudaEventDestroy(ev_loop0);
    if (ev_loop1) cudaEventDestroy(ev_loop1);
    if (graph) cudaGraphExecDestroy(graph);
    if (comm && nccl().ok) nccl().CommDestroy(comm);
    if (ev_vals) cudaEventDestroy(ev_vals);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

void setup_common(equil_matrix* M, const equil_device_cfg* cfg) {
  M->device = cfg ? cfg->device : 0;
  M->rank = cfg ? cfg->rank : 0;
  M->world = cfg ? std::max(1, cfg->world_size) : 1;
  if (const char* e = getenv("EQUIL_PANEL")) M->use_panels = atoi(e) != 0;  // A/B knob
  if (const char* e = getenv("EQUIL_SLOTS")) M->use_slots = atoi(e) != 0;
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
    if (!nccl().ok) fail(EQUIL_ENCCL, "libnccl.so.2 could not be loaded");
    ncclUniqueId id;
    std::memcpy(&id, cfg->nccl_id, sizeof id);
    nccl_check(nccl().CommInitRank(&M->comm, M->world, id, M->rank), "ncclCommInitRank");
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
void upload_plans(equil_matrix* M, const Plan& pa, const Plan& pt) {
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
    if (!h.empty())
      CK(cudaMemcpy(d.p, h.data(), h.size() * sizeof(h[0]), cudaMemcpyHostToDevice));
    return static_cast<int>(h.size());
  };
  M->n_sgd = upload(M->tiles_sgd, sgd);
  M->n_sgd_long = static_cast<int>(pa.lng.size() + pt.lng.size());
  M->n_a = upload(M->tiles_a, ta);
  M->n_t = upload(M->tiles_t, tt);
  upload(M->rowlist_a, pa.rowlist);
  upload(M->rowlist_t, pt.rowlist);
}

void allgather_padded(equil_matrix* M, double* buf, int64_t maxcnt) {
  if (M->world == 1) return;
  nccl_check(nccl().AllGather(buf + M->rank * maxcnt, buf, static_cast<size_t>(maxcnt),
                              ncclFloat64, M->comm, M->stream),
             "ncclAllGather");
}

// Bands for the column-panel traversal: consecutive rows, closed before a row
// that would push the band past `target` entries or kBandRows rows.
std::vector<int64_t> plan_bands(const int64_t* rp, int64_t rows, int64_t target) {
  std::vector<int64_t> b{0};
  for (int64_t i = 0; i < rows; ++i) {
    const int64_t r0 = b.back();
    if (i > r0 && (i - r0 >= eqb::kBandRows || rp[i + 1] - rp[r0] > target)) b.push_back(i);
  }
  if (rows > 0) b.push_back(rows);
  return b;
}

// Panel-major copies of the local A / A^T shards and the band list of the SGD
// launch (both matrices, largest bands first).  Band size targets about
// EQUIL_BANDS_PER_SM (default 2) bands per SM over the whole launch.
void build_panel_layout(equil_matrix* M, const int64_t* rpA, const int64_t* rpT) {
  M->n_pbands = 0;
  if (!M->use_panels) return;
  int dev = 0, sms = 148;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double per_sm = 2.0;
  if (const char* e = getenv("EQUIL_BANDS_PER_SM")) per_sm = std::max(0.1, atof(e));
  const int64_t total = M->A.nnz + M->AT.nnz;
  const int64_t target = std::max<int64_t>(1, static_cast<int64_t>(total / (per_sm * sms)));
  std::vector<std::pair<int64_t, eqb::PanelBand>> all;
  for (int mat = 0; mat < 2; ++mat) {
    const eqb::DevCsr& C = mat ? M->AT : M->A;
    const int64_t* rp = mat ? rpT : rpA;
    const std::vector<int64_t> bounds = plan_bands(rp, C.rows, target);
    const int nb = static_cast<int>(bounds.size()) - 1;
    if (nb <= 0) continue;
    M->pval[mat].alloc(C.nnz);
    M->pcol[mat].alloc(C.nnz);
    eqb::PanelChunk* ch = nullptr;
    uint32_t* runs = nullptr;
    int64_t nch = 0, nruns = 0;
    std::vector<int64_t> bc;
    CK(eqb::build_panels(C, mat ? M->m_pad() : M->n_pad(), bounds, M->pval[mat].p,
                         M->pcol[mat].p, &runs, &nruns, &ch, &nch, &bc, M->stream));
    M->pchunks[mat].adopt(ch, static_cast<size_t>(std::max<int64_t>(1, nch)));
    M->pruns[mat].adopt(runs, static_cast<size_t>(std::max<int64_t>(1, nruns)));
    for (int b = 0; b < nb; ++b) {
      eqb::PanelBand pb{static_cast<int32_t>(bounds[b]),
                        static_cast<int32_t>(bounds[b + 1] - bounds[b]),
                        static_cast<int32_t>(bc[b]), static_cast<int32_t>(bc[b + 1]), mat, 0};
      all.push_back({rp[bounds[b + 1]] - rp[bounds[b]], pb});
    }
  }
  std::stable_sort(all.begin(), all.end(),
                   [](const auto& x, const auto& y) { return x.first > y.first; });
  std::vector<eqb::PanelBand> h;
  for (const auto& x : all) h.push_back(x.second);
  M->pbands.alloc(h.size());
  if (!h.empty())
    CK(cudaMemcpy(M->pbands.p, h.data(), h.size() * sizeof(h[0]), cudaMemcpyHostToDevice));
  M->n_pbands = static_cast<int>(h.size());
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
  if (!M->use_slots || M->use_panels) return;
  cudaStream_t s = M->stream;
  const int G = M->world;
  DevBuf<int64_t> ab, tb;
  const int64_t* abd = M->a_bounds_d.p;
  const int64_t* tbd = M->t_bounds_d.p;
  if (G == 1) {  // bounds {0, rows}
    ab.alloc(2);
    tb.alloc(2);
    const int64_t a2[2] = {0, M->m}, t2[2] = {0, M->n};
    CK(cudaMemcpy(ab.p, a2, 16, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(tb.p, t2, 16, cudaMemcpyHostToDevice));
    abd = ab.p;
    tbd = tb.p;
  }
  M->wmap.alloc(M->m_pad());
  M->smap.alloc(M->n_pad());
  CK(eqb::launch_slot_map(rpA_dev, M->m, abd, G, M->a_max, M->wmap.p, s));
  CK(eqb::launch_slot_map(rpT_dev, M->n, tbd, G, M->t_max, M->smap.p, s));
  M->a_ci_sgd.alloc(M->A.nnz);
  M->t_ci_sgd.alloc(M->AT.nnz);
  CK(eqb::launch_remap_cols(M->a_ci_sgd.p, M->A.col, M->smap.p, M->A.nnz, s));
  CK(eqb::launch_remap_cols(M->t_ci_sgd.p, M->AT.col, M->wmap.p, M->AT.nnz, s));
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
  CK(cudaMemcpy(M->a_bounds_d.p, M->a_bounds.data(), (G + 1) * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(M->t_bounds_d.p, M->t_bounds.data(), (G + 1) * 8, cudaMemcpyHostToDevice));

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
        CK(cudaMemcpy(cb.p, colb.data(), (G + 1) * 8, cudaMemcpyHostToDevice));
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
  build_panel_layout(M, la.data(), lt.data());
  build_slot_layout(M, fullA.row_ptr, fullT.row_ptr);
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
      if (cudaEventSynchronize(ev_rp) == cudaSuccess) planT = plan_tiles(rpT.data(), n, 1);
    });
  CK(eqb::transpose_csr(fullA, fullT, s, M->ev_vals));
  CK(cudaStreamWaitEvent(s, M->ev_vals, 0));  // every later use of A's values
  pt.mark(s, "transpose");
  CK(cudaEventSynchronize(ev_rp));
  pt.mark(s, "rowptr copy");
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
    build_panel_layout(M, row_ptr, rpT.data());
    pt.mark(s, "panels");
  } else {
    const std::vector<int64_t> rpA(row_ptr, row_ptr + m + 1);
    shard_sparse(M, fullA, fullT, rpA, rpT);
  }
  pt.mark(s, "plan");
  alloc_workspaces(M, &pt);
  CK(cudaStreamSynchronize(s));
  pt.mark(s, "workspaces");
}

void alloc_workspaces(equil_matrix* M, PhaseTimer* pt) {
  // each vector padded to whole panels (the panel traversal bulk-copies them)
  auto whole = [](int64_t x) { return (x + eqb::kPanelW - 1) / eqb::kPanelW * eqb::kPanelW; };
  const int64_t np = whole(M->n_pad()), mp = whole(M->m_pad());
  M->xbuf.alloc(2 * (np + mp));
  CK(cudaMemset(M->xbuf.p, 0, 2 * (np + mp) * sizeof(double)));
  if (pt) pt->mark(M->stream, "xbuf");
  for (int b = 0; b < 2; ++b) {
    M->xs[b].p = M->xbuf.p + b * np;
    M->xw[b].p = M->xbuf.p + 2 * np + b * mp;
  }
  // Keep the gather targets resident in L2 while CSR(A)/CSR(A^T) stream past.
  int dev = 0, max_persist = 0, max_window = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
  cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
  const size_t bytes = static_cast<size_t>(2 * (np + mp)) * sizeof(double);
  static const bool l2win = !getenv("EQUIL_L2WIN") || atoi(getenv("EQUIL_L2WIN")) != 0;
  if (l2win && max_persist > 0 && max_window > 0) {
    const size_t win = std::min(bytes, static_cast<size_t>(max_window));
    const size_t carve = std::min(win, static_cast<size_t>(max_persist));
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve) == cudaSuccess) {
      cudaStreamAttrValue attr{};
      attr.accessPolicyWindow.base_ptr = M->xbuf.p;
      attr.accessPolicyWindow.num_bytes = win;
      attr.accessPolicyWindow.hitRatio =
          static_cast<float>(std::min(1.0, static_cast<double>(carve) / win));
      attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(M->stream, cudaStreamAttributeAccessPolicyWindow, &attr);
    }
    cudaGetLastError();  // the window is a hint; never fail on it
  }
  if (pt) pt->mark(M->stream, "l2 window");
  M->u.alloc(M->m_loc());
  M->ub.alloc(M->m_loc());
  M->v.alloc(M->n_loc());
  M->vb.alloc(M->n_loc());
  const int64_t big = std::max(M->m_pad(), M->n_pad());
  M->red_part.alloc((big + eqb::kChunk - 1) / eqb::kChunk + 1);
  M->tmp_m.alloc(M->m_pad());
  M->tmp_n.alloc(M->n_pad());
  M->tmp_m2.alloc(M->m_pad());
  M->tmp_n2.alloc(M->n_pad());
  if (M->dense) M->colpart.alloc(((M->m + eqb::kChunk - 1) / eqb::kChunk) * M->n);
}

}  // namespace

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

equil_status equil_matrix_create_csr(int64_t m, int64_t n, const int64_t* row_ptr,
                                     const int32_t* col, const double* val,
                                     const equil_device_cfg* cfg, equil_matrix** out) {
  return guarded([&] {
    require(out != nullptr, "ExplicitMatrix::sparse: null output handle");
    *out = nullptr;
    require(m > 0 && n > 0, "ExplicitMatrix::sparse: dimensions must be positive");
    require(row_ptr != nullptr, "ExplicitMatrix::sparse: null row_ptr");
    require(n < (1LL << 31) && m < (1LL << 31), "ExplicitMatrix::sparse: dimension too large");
    const int64_t nnz = row_ptr[m];
    require(nnz >= 0 && nnz < (1LL << 31), "ExplicitMatrix::sparse: bad nnz");
    // row_ptr is checked on the host before anything reads the arrays by it
    require(row_ptr[0] == 0, "ExplicitMatrix::sparse: row_ptr[0] must be 0");
    for (int64_t i = 0; i < m; ++i)
      if (row_ptr[i + 1] < row_ptr[i])
        fail(EQUIL_EINVAL, "ExplicitMatrix::sparse: row_ptr decreases at row " + std::to_string(i));
    require(nnz == 0 || (col && val), "ExplicitMatrix::sparse: null col/val");
    PhaseTimer pt("create_csr");
    auto M = std::make_unique<equil_matrix>();
    setup_common(M.get(), cfg);
    M->m = m;
    M->n = n;
    M->nnz = nnz;
    DeviceGuard dg(M->device);
    cudaStream_t s = M->stream;
    pt.mark(s, "setup");
    // full A on device (uploaded once; shards are sliced from it)
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
    } else {
      CK(cudaEventRecord(M->ev_vals, s));
    }
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
    if (M->world == 1) planner = std::thread([&] { planA = plan_tiles(row_ptr, m, 0); });
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
    if (wh != ~0ULL) {
      const int cls = static_cast<int>(wh >> 40);
      const int64_t k = static_cast<int64_t>(wh & ((1ULL << 40) - 1));
      const int64_t i = std::upper_bound(row_ptr, row_ptr + m + 1, k) - row_ptr - 1;
      const std::string at = "(" + std::to_string(i) + ", " + std::to_string(col[k]) + ")";
      if (cls == 0) fail(EQUIL_EINVAL, "ExplicitMatrix::sparse: entry " + at + " out of range");
      if (cls == 1) fail(EQUIL_EINVAL, "ExplicitMatrix::sparse: duplicate entry " + at);
      fail(EQUIL_EINVAL, "ExplicitMatrix::sparse: columns not ascending at entry " + at +
                             " (canonical CSR required)");
    }
    finish_sparse(M.get(), rp, ci, va, row_ptr, pt, &planA, &planner);
    *out = M.release();
  });
}

}  // extern "C"

namespace {
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
}  // namespace

extern "C" {

equil_status equil_matrix_create_coo(int64_t m, int64_t n, int64_t nnz, const int64_t* rows,
                                     const int64_t* cols, const double* vals,
                                     const equil_device_cfg* cfg, equil_matrix** out) {
  return guarded([&] { create_coo_impl(m, n, nnz, rows, cols, vals, nullptr, cfg, out); });
}

equil_status equil_matrix_create_dense(int64_t m, int64_t n, const double* rowmajor,
                                       const equil_device_cfg* cfg, equil_matrix** out) {
  return guarded([&] {
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
namespace {

struct DiagPlan {
  int stride = 0;
  bool obj = false, rms = false;
};

// canonical reduction of x[0, len) into *out (device): kind 0 sum of squares,
// 1 plain sum, 2 sum of coef * x; optional sqrt of the result
void canon_reduce(equil_matrix* M, const double* x, int64_t len, double* out, int kind,
                  double coef = 0.0, bool sqrt_out = false) {
  CK(eqb::launch_canon_reduce(x, len, kind, coef, M->red_part.p, M->red_counter.p, out,
                              sqrt_out ? 1 : 0, M->stream));
}

}  // namespace

namespace {

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

    // K1: all T*(n+m) signs up front (never depends on the iterate)
    if (total > 0) {
      M->signs.ensure((total + 31) / 32 + 1);
      const size_t sb = eqb::sign_stream_scratch_bytes(total);
      M->sign_scratch.ensure(sb);
      CK(eqb::sign_stream_generate(p->seed, 17, total, M->signs.p, M->sign_scratch.p, sb, s));
    }
    // init: u = v = 0, ubar = vbar = 0, xs = s_1, xw = w_1
    CK(cudaMemsetAsync(M->flags.p, 0, sizeof(unsigned), s));
    const int64_t a_poff = M->world == 1 ? M->a_goff() : M->rank * M->a_max;
    const int64_t t_poff = M->world == 1 ? M->t_goff() : M->rank * M->t_max;
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
      return a;
    };
    eqb::PanelArgs panel_args{};
    panel_args.bands = M->pbands.p;
    for (int k = 0; k < 2; ++k) {
      panel_args.chunks[k] = M->pchunks[k].p;
      panel_args.val[k] = M->pval[k].p;
      panel_args.col[k] = M->pcol[k].p;
      panel_args.runs[k] = M->pruns[k].p;
    }
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
      return a;
    };
    auto one_iter = [&](int t) {
      if (M->dense) {
        CK(eqb::launch_dense_sgd_iter(dense_args(t), s));
      } else {
        static const int conc = getenv("EQUIL_CONC") ? atoi(getenv("EQUIL_CONC")) : 1;
        if (M->n_pbands) {
          CK(eqb::launch_sgd_panel(iter_args(t), panel_args, M->n_pbands, s));
        } else if (conc && M->n_sgd_long > 0 && M->n_sgd_long < M->n_sgd) {
          // long-row CTA groups and warp tiles as two concurrent kernels (fork /
          // join on the copy stream): each kernel gets its own residency on the
          // SMs instead of one launch sized for both (c3: 4-5% faster)
          const eqb::SgdIterArgs a = iter_args(t);
          CK(cudaEventRecord(M->ev_fork, s));
          CK(cudaStreamWaitEvent(M->copy_stream, M->ev_fork, 0));
          CK(eqb::launch_sgd_iter_part(a, 0, M->n_sgd_long, true, conc >= 2 ? 8 : 6,
                                       M->copy_stream));
          CK(eqb::launch_sgd_iter_part(a, M->n_sgd_long, M->n_sgd - M->n_sgd_long, false,
                                       conc >= 3 ? 8 : 6, s));
          CK(cudaEventRecord(M->ev_join, M->copy_stream));
          CK(cudaStreamWaitEvent(s, M->ev_join, 0));
        } else {
          CK(eqb::launch_sgd_iter(iter_args(t), M->n_sgd, s));
        }
        if (t < T) {
          allgather_padded(M, M->xs[t & 1].p, M->t_max);
          allgather_padded(M, M->xw[t & 1].p, M->a_max);
        }
      }
    };

    if (dp.stride == 0 && T > 0) {
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

    // finalize: u = ubar, v = vbar, d = exp(ubar), e = exp(vbar) (:201-204)
    double* dloc = M->tmp_m.p;
    double* eloc = M->tmp_n.p;
    CK(eqb::launch_exp(M->ub.p, dloc, ml, 1.0, s));
    CK(eqb::launch_exp(M->vb.p, eloc, nl, 1.0, s));
    unsigned flags = 0;
    if (M->world > 1) {
      nccl_check(nccl().AllReduce(M->flags.p, M->flags.p, 1, ncclUint32, ncclMax, M->comm, s),
                 "ncclAllReduce");
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

}  // namespace

extern "C" equil_status equil_sgd_equilibrate(equil_matrix* M, const equil_params* p,
                                              const equil_diag_cfg* diag,
                                              equil_scaling_out* out) {
  return guarded([&] {
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
namespace {

// one matvec pass of B (scaled by scale when non-null) in the given mode
void apply_pass(equil_matrix* M, bool adjoint, const double* xg, double* out, int mode,
                const double* scale, const double* prev, const double* coef) {
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
    a.colpart = M->colpart.p;
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
  CK(eqb::launch_pass(a, adjoint ? M->n_t : M->n_a, M->stream));
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
  DevBuf<double> u, v, w, un, du, vn, ev, ex, r;
  u.alloc(L.mL); v.alloc(L.nL); w.alloc(L.nL); x.alloc(L.nL);
  un.alloc(L.mP); du.alloc(L.mP); r.alloc(L.mP);
  vn.alloc(L.nP); ev.alloc(L.nP); ex.alloc(L.nP);
  double* unL = un.p + L.pa;
  double* duL = du.p + L.pa;
  double* rL = r.p + L.pa;
  double* vnL = vn.p + L.pt;
  double* evL = ev.p + L.pt;
  double* exL = ex.p + L.pt;
  CK(cudaMemsetAsync(x.p, 0, L.nL * 8, s));
  double* sc = M->scal.p;  // [0] beta, [1] alpha, [2] residual norm
  int* dummy = reinterpret_cast<int*>(sc + 8);

  CK(cudaMemcpyAsync(unL, c, L.mL * 8, cudaMemcpyDeviceToDevice, s));
  L.norm(un.p, true, sc + 0);  // beta = |c|
  CK(eqb::launch_lsqr_normalize(u.p, c, sc + 0, duL, d, L.mL, nullptr, nullptr, s));
  L.gather(du.p, true);
  apply_pass(M, true, du.p, vnL, eqb::kPassScaled, e, nullptr, nullptr);  // v = B^T u
  ++st.adjoints;
  L.norm(vn.p, false, sc + 1);
  double beta = read_scalar(M, sc + 0);
  double alpha = read_scalar(M, sc + 1);
  if (alpha == 0.0) {
    st.breakdown = true;
    return;
  }
  CK(eqb::launch_lsqr_normalize(v.p, vnL, sc + 1, evL, e, L.nL, dummy, nullptr, s));
  L.gather(ev.p, false);
  CK(cudaMemcpyAsync(w.p, v.p, L.nL * 8, cudaMemcpyDeviceToDevice, s));
  double phibar = beta, rhobar = alpha;

  for (int t = 1; t <= max_iters; ++t) {
    bool invariant = false;
    apply_pass(M, false, ev.p, unL, eqb::kPassLsqrU, d, u.p, sc + 1);  // Bv - alpha u
    ++st.applies;
    L.norm(un.p, true, sc + 0);
    beta = read_scalar(M, sc + 0);
    if (beta > 0.0) {
      CK(eqb::launch_lsqr_normalize(u.p, unL, sc + 0, duL, d, L.mL, nullptr, nullptr, s));
      L.gather(du.p, true);
    } else {
      invariant = true;
    }
    alpha = 0.0;
    if (!invariant) {
      apply_pass(M, true, du.p, vnL, eqb::kPassLsqrV, e, v.p, sc + 0);  // B^T u - beta v
      ++st.adjoints;
      L.norm(vn.p, false, sc + 1);
      alpha = read_scalar(M, sc + 1);
      if (alpha > 0.0) {
        CK(eqb::launch_lsqr_normalize(v.p, vnL, sc + 1, evL, e, L.nL, nullptr, nullptr, s));
        L.gather(ev.p, false);
      } else {
        invariant = true;
      }
    }
    const double rho = std::hypot(rhobar, beta);  // :58-64
    const double cs = rhobar / rho;
    const double sn = beta / rho;
    const double theta = sn * alpha;
    rhobar = -cs * alpha;
    const double phi = cs * phibar;
    phibar = sn * phibar;
    CK(eqb::launch_lsqr_xw_update(x.p, w.p, v.p, phi / rho, theta / rho, e, exL, L.nL, s));
    L.gather(ex.p, false);
    st.iterations = t;
    apply_pass(M, false, ex.p, rL, eqb::kPassResid, nullptr, b_loc, nullptr);
    L.norm(r.p, true, sc + 2);
    const double rel = read_scalar(M, sc + 2) / bnorm;
    if (st.hist_len < hist_cap) hist[st.hist_len] = rel;
    ++st.hist_len;
    if (rel <= tol) {
      st.reached_tol = true;
      break;
    }
    if (invariant) {
      st.breakdown = true;
      break;
    }
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

}  // namespace

extern "C" {

equil_status equil_lsqr(equil_matrix* A, const double* b, int max_iters, double tol,
                        equil_lsqr_out* out) {
  return guarded([&] { lsqr_common(A, b, nullptr, max_iters, tol, out, "lsqr"); });
}

equil_status equil_lsqr_preconditioned(equil_matrix* A, const double* b,
                                       const equil_params* p, int max_iters, double tol,
                                       equil_lsqr_out* out) {
  return guarded([&] {
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
  equil_status rc = equil_matrix_create_csr(m, n, row_ptr, col, val, cfg, &M);
  if (rc != EQUIL_OK) return rc;
  rc = equil_sgd_equilibrate(M, p, nullptr, out);
  equil_matrix_destroy(M);
  return rc;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Engine variants (src/variants.cpp): symmetric (:35-103) and block
// (:156-240) equilibration.  Same sign stream, the same projected-SGD update
// (run_projected_sgd) and the same estimator arithmetic as sgd_row_col, but
// the passes run as generic pass kernels (kPassEst) between small kernels that
// form the scalings, sum estimates over blocks and update the block iterates.
// Single GPU; sparse and dense matrices (history for sparse ones).
// ---------------------------------------------------------------------------
namespace {

// SeededRng (src/rng.cpp:9-49) on the host: the symmetry check's probe
// normals (Box-Muller with the spare kept; glibc log/sin/cos like the
// reference build).
struct HostRng {
  uint64_t mt[eqb::mt::kN];
  int i = eqb::mt::kN;
  bool has_spare = false;
  double spare = 0.0;
  HostRng(uint64_t seed, uint64_t stream) { eqb::mt::seed_state(seed, stream, mt); }
  uint64_t next() {
    if (i >= eqb::mt::kN) {
      constexpr uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL;
      for (int k = 0; k < eqb::mt::kN; ++k) {
        const uint64_t x = (mt[k] & kUpper) | (mt[(k + 1) % eqb::mt::kN] & kLower);
        uint64_t xa = x >> 1;
        if (x & 1u) xa ^= 0xB5026F5AA96619E9ULL;
        mt[k] = mt[(k + eqb::mt::kM) % eqb::mt::kN] ^ xa;
      }
      i = 0;
    }
    return eqb::mt::temper(mt[i++]);
  }
  double uniform01() { return (static_cast<double>(next() >> 11) + 0.5) * 0x1.0p-53; }
  double normal() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    const double u1 = uniform01(), u2 = uniform01();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double theta = 6.283185307179586476925286766559 * u2;
    spare = r * std::sin(theta);
    has_spare = true;
    return r * std::cos(theta);
  }
};

enum class Variant { kSymmetric, kBlock };

// check_symmetry (src/variants.cpp:14-33) with device applies and canonical
// dots / norms; the probes come from stream 18 (streams::kSymmetryCheck).
void check_symmetry(equil_matrix* M, uint64_t seed) {
  const int64_t n = M->n;
  cudaStream_t s = M->stream;
  HostRng rng(seed, 18);
  std::vector<double> x(n), y(n);
  DevBuf<double> xd, yd, ax, ay, t;
  xd.alloc(n); yd.alloc(n); ax.alloc(n); ay.alloc(n); t.alloc(n);
  double* sc = M->scal.p + 32;
  for (int probe = 0; probe < 3; ++probe) {
    for (int64_t i = 0; i < n; ++i) x[i] = rng.normal();
    for (int64_t i = 0; i < n; ++i) y[i] = rng.normal();
    CK(cudaMemcpyAsync(xd.p, x.data(), n * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(yd.p, y.data(), n * 8, cudaMemcpyHostToDevice, s));
    apply_pass(M, false, xd.p, ax.p, eqb::kPassPlain, nullptr, nullptr, nullptr);
    apply_pass(M, false, yd.p, ay.p, eqb::kPassPlain, nullptr, nullptr, nullptr);
    CK(eqb::launch_mul(t.p, ax.p, yd.p, n, s));
    canon_reduce(M, t.p, n, sc + 0, 1);  // ax.dot(y)
    CK(eqb::launch_mul(t.p, xd.p, ay.p, n, s));
    canon_reduce(M, t.p, n, sc + 1, 1);  // x.dot(ay)
    canon_reduce(M, ax.p, n, sc + 2, 0, 0.0, true);
    canon_reduce(M, yd.p, n, sc + 3, 0, 0.0, true);
    canon_reduce(M, xd.p, n, sc + 4, 0, 0.0, true);
    canon_reduce(M, ay.p, n, sc + 5, 0, 0.0, true);
    double r[6];
    CK(cudaMemcpyAsync(r, sc, sizeof r, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const double scale = r[2] * r[3] + r[4] * r[5] + 1e-30;
    require(std::abs(r[0] - r[1]) <= 1e-10 * scale,
            "sgd_equilibrate_symmetric: operator failed symmetry check");
  }
}

void sgd_variant(equil_matrix* M, Variant kind, const equil_params* p,
                 const equil_diag_cfg* diag, equil_scaling_out* out, const int64_t* rb_host,
                 const int64_t* cb_host, int64_t R, int64_t C) {
  std::lock_guard<std::mutex> lk(M->mu);
  DeviceGuard dg(M->device);
  const bool sym = kind == Variant::kSymmetric;
  const char* who = sym ? "sgd_equilibrate_symmetric" : "sgd_equilibrate_block";
  require(M->world == 1, std::string(who) + ": single-GPU matrices only in this build");
  validate_params(*p);
  const int64_t m = M->m, n = M->n;
  double alpha = 0, beta = 0;
  std::vector<int32_t> rbm, cbm;
  std::vector<double> rcount, ccount;
  if (sym) {
    require(m == n, "sgd_equilibrate_symmetric: operator must be square");
    check_symmetry(M, p->seed);
    resolve_targets(*p, n, n, alpha, beta);
    require(std::abs(alpha - beta) <= 1e-12 * std::max(alpha, beta),
            "sgd_equilibrate_symmetric: targets must coincide");
    R = n;
    C = 0;
  } else {  // BlockStructure::validate (src/variants.cpp:131-154)
    require(rb_host != nullptr && cb_host != nullptr, "BlockStructure: assignment length mismatch");
    require(R > 0 && C > 0, "BlockStructure: block counts must be positive");
    require(R < (1LL << 31) && C < (1LL << 31), "BlockStructure: too many blocks");
    rcount.assign(R, 0.0);
    ccount.assign(C, 0.0);
    rbm.resize(m);
    cbm.resize(n);
    for (int64_t i = 0; i < m; ++i) {
      require(rb_host[i] >= 0 && rb_host[i] < R, "BlockStructure: row block index out of range");
      rbm[i] = static_cast<int32_t>(rb_host[i]);
    }
    for (int64_t j = 0; j < n; ++j) {
      require(cb_host[j] >= 0 && cb_host[j] < C, "BlockStructure: col block index out of range");
      cbm[j] = static_cast<int32_t>(cb_host[j]);
    }
    for (int64_t i = 0; i < m; ++i) rcount[rbm[i]] += 1.0;  // :165-169
    for (int64_t j = 0; j < n; ++j) ccount[cbm[j]] += 1.0;
    for (int64_t b = 0; b < R; ++b) require(rcount[b] != 0.0, "BlockStructure: empty row block");
    for (int64_t b = 0; b < C; ++b) require(ccount[b] != 0.0, "BlockStructure: empty col block");
    resolve_targets(*p, m, n, alpha, beta);
  }
  const int stride = diag ? diag->stride : 0;
  require(stride >= 0, std::string(who) + ": stride must be positive");
  const int T = p->iterations;
  const int nrec = stride ? T / stride + 1 : 0;
  if (stride) {
    require(!M->dense, std::string(who) + ": history is implemented for sparse matrices");
    require(out->hist_cap >= nrec, std::string(who) + ": history capacity too small");
  }
  cudaStream_t s = M->stream;
  const double gamma = p->gamma, Mx = p->max_log_scale;

  // signs: n per iteration (symmetric: one probe) or n + m (s then w)
  const uint64_t per_iter = static_cast<uint64_t>(sym ? n : n + m);
  const uint64_t total = per_iter * static_cast<uint64_t>(T);
  if (total > 0) {
    M->signs.ensure((total + 31) / 32 + 1);
    const size_t sb = eqb::sign_stream_scratch_bytes(total);
    M->sign_scratch.ensure(sb);
    CK(eqb::sign_stream_generate(p->seed, 17, total, M->signs.p, M->sign_scratch.p, sb, s));
  }
  // block iterates, linear terms, scalings, probes, estimates
  DevBuf<double> xu, xub, xv, xvb, lu, lv, d, e, xs, xw, er, ec, ebu, ebv;
  DevBuf<int32_t> rbd, cbd, memr, memc;
  DevBuf<int64_t> offr, offc;
  xu.alloc(R); xub.alloc(R); lu.alloc(R);
  d.alloc(m); e.alloc(n); xs.alloc(n); xw.alloc(m); er.alloc(m); ec.alloc(n);
  CK(cudaMemsetAsync(xu.p, 0, R * 8, s));
  CK(cudaMemsetAsync(xub.p, 0, R * 8, s));
  {
    std::vector<double> l(R);
    for (int64_t b = 0; b < R; ++b) l[b] = sym ? alpha * alpha : (alpha * alpha) * rcount[b];
    CK(cudaMemcpyAsync(lu.p, l.data(), R * 8, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  }
  if (!sym) {
    xv.alloc(C); xvb.alloc(C); lv.alloc(C); ebu.alloc(R); ebv.alloc(C);
    CK(cudaMemsetAsync(xv.p, 0, C * 8, s));
    CK(cudaMemsetAsync(xvb.p, 0, C * 8, s));
    std::vector<double> l(C);
    for (int64_t b = 0; b < C; ++b) l[b] = (beta * beta) * ccount[b];
    CK(cudaMemcpy(lv.p, l.data(), C * 8, cudaMemcpyHostToDevice));
    // members of every block in ascending index order (stable counting sort)
    auto members = [](const std::vector<int32_t>& map, int64_t nb, DevBuf<int32_t>& mem,
                      DevBuf<int64_t>& off) {
      std::vector<int64_t> o(nb + 1, 0);
      for (int32_t b : map) ++o[b + 1];
      for (int64_t b = 0; b < nb; ++b) o[b + 1] += o[b];
      std::vector<int32_t> list(map.size());
      std::vector<int64_t> pos(o.begin(), o.end() - 1);
      for (size_t i = 0; i < map.size(); ++i) list[pos[map[i]]++] = static_cast<int32_t>(i);
      mem.alloc(list.size());
      off.alloc(o.size());
      if (!list.empty())
        CK(cudaMemcpy(mem.p, list.data(), list.size() * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(off.p, o.data(), o.size() * 8, cudaMemcpyHostToDevice));
    };
    members(rbm, R, memr, offr);
    members(cbm, C, memc, offc);
    rbd.alloc(m);
    cbd.alloc(n);
    if (m) CK(cudaMemcpy(rbd.p, rbm.data(), m * 4, cudaMemcpyHostToDevice));
    if (n) CK(cudaMemcpy(cbd.p, cbm.data(), n * 4, cudaMemcpyHostToDevice));
  }
  CK(cudaMemsetAsync(M->flags.p, 0, sizeof(unsigned), s));
  eqb::SgdBlockConst c{};
  c.gamma = gamma;
  c.M = Mx;

  // history (src/variants.cpp:66-86, :197-214) at the expanded averages
  constexpr int kRec = 6;
  DevBuf<double> hist, terms, uf, vf, eu, ev;
  if (nrec) {
    hist.alloc(kRec * nrec);
    terms.alloc(m + n);
    uf.alloc(m); vf.alloc(n); eu.alloc(m); ev.alloc(n);
  }
  const double a2 = alpha * alpha, b2 = sym ? alpha * alpha : beta * beta;
  const double beta_rms = sym ? alpha : beta;
  auto expand_avg = [&]() {
    if (sym) {
      CK(cudaMemcpyAsync(uf.p, xub.p, n * 8, cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(vf.p, xub.p, n * 8, cudaMemcpyDeviceToDevice, s));
    } else {
      CK(eqb::launch_gather_map(xub.p, rbd.p, m, uf.p, s));
      CK(eqb::launch_gather_map(xvb.p, cbd.p, n, vf.p, s));
    }
  };
  int rec = 0;
  auto record = [&]() {
    double* slot = hist.p + kRec * rec;
    expand_avg();
    CK(eqb::launch_exp(uf.p, eu.p, m, 2.0, s));
    CK(eqb::launch_exp(vf.p, ev.p, n, 2.0, s));
    CK(eqb::launch_rms_terms(0, M->A, eu.p, ev.p, terms.p, 0, alpha, s));
    CK(eqb::launch_rms_terms(1, M->AT, eu.p, ev.p, terms.p + m, 0, beta_rms, s));
    canon_reduce(M, terms.p, m + n, slot + 0, 1);
    CK(eqb::launch_obj_terms(M->A, uf.p, vf.p, terms.p, s));
    canon_reduce(M, terms.p, m, slot + 1, 1);
    canon_reduce(M, uf.p, m, slot + 2, 2, a2);
    canon_reduce(M, vf.p, n, slot + 3, 2, b2);
    canon_reduce(M, uf.p, m, slot + 4, 0);
    canon_reduce(M, vf.p, n, slot + 5, 0);
    ++rec;
  };
  if (stride) record();
  for (int t = 1; t <= T; ++t) {
    eqb::SgdStep st;
    st.step = 2.0 / (gamma * static_cast<double>(t + 1));
    st.aw = 2.0 / (static_cast<double>(t) + 2.0);
    st.aw1 = 1.0 - st.aw;
    st.pad = 0;
    const int64_t base = static_cast<int64_t>(t - 1) * static_cast<int64_t>(per_iter);
    if (sym) {  // d = exp(u); est = (d .* A (d .* s))^2 (:60-64)
      CK(eqb::launch_expand_scale(xu.p, nullptr, n, M->signs.p, base, d.p, xs.p, s));
      apply_pass(M, false, xs.p, er.p, eqb::kPassEst, d.p, nullptr, nullptr);
      CK(eqb::launch_sgd_update(xu.p, xub.p, er.p, lu.p, c, st, n, M->flags.p, s));
    } else {  // :181-194
      CK(eqb::launch_expand_scale(xv.p, cbd.p, n, M->signs.p, base, e.p, xs.p, s));
      CK(eqb::launch_expand_scale(xu.p, rbd.p, m, M->signs.p, base + n, d.p, xw.p, s));
      apply_pass(M, false, xs.p, er.p, eqb::kPassEst, d.p, nullptr, nullptr);
      apply_pass(M, true, xw.p, ec.p, eqb::kPassEst, e.p, nullptr, nullptr);
      CK(eqb::launch_block_sum(er.p, memr.p, offr.p, R, ebu.p, s));
      CK(eqb::launch_block_sum(ec.p, memc.p, offc.p, C, ebv.p, s));
      CK(eqb::launch_sgd_update(xu.p, xub.p, ebu.p, lu.p, c, st, R, M->flags.p, s));
      CK(eqb::launch_sgd_update(xv.p, xvb.p, ebv.p, lv.p, c, st, C, M->flags.p, s));
    }
    if (stride && t % stride == 0) record();
  }
  // result: expanded averages and their exponentials (:93-96, :226-229)
  DevBuf<double> ufin, vfin, dfin, efin;
  ufin.alloc(m); vfin.alloc(n); dfin.alloc(m); efin.alloc(n);
  if (sym) {
    CK(cudaMemcpyAsync(ufin.p, xub.p, n * 8, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(vfin.p, xub.p, n * 8, cudaMemcpyDeviceToDevice, s));
  } else {
    CK(eqb::launch_gather_map(xub.p, rbd.p, m, ufin.p, s));
    CK(eqb::launch_gather_map(xvb.p, cbd.p, n, vfin.p, s));
  }
  CK(eqb::launch_exp(ufin.p, dfin.p, m, 1.0, s));
  CK(eqb::launch_exp(vfin.p, efin.p, n, 1.0, s));
  const cudaMemcpyKind k =
      out->outputs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (out->u) CK(cudaMemcpyAsync(out->u, ufin.p, m * 8, k, s));
  if (out->v) CK(cudaMemcpyAsync(out->v, vfin.p, n * 8, k, s));
  if (out->d) CK(cudaMemcpyAsync(out->d, dfin.p, m * 8, k, s));
  if (out->e) CK(cudaMemcpyAsync(out->e, efin.p, n * 8, k, s));
  unsigned flags = 0;
  CK(cudaMemcpyAsync(&flags, M->flags.p, sizeof flags, cudaMemcpyDeviceToHost, s));
  std::vector<double> hh(kRec * static_cast<size_t>(std::max(nrec, 1)));
  if (nrec) CK(cudaMemcpyAsync(hh.data(), hist.p, kRec * nrec * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  out->alpha = alpha;
  out->beta = sym ? alpha : beta;
  out->iterate_bound_ok = (flags & 1u) ? 0 : 1;
  out->box_feasible = (flags & 2u) ? 0 : 1;
  out->apply_count = T;
  out->adjoint_count = sym ? 0 : T;
  out->hist_len = nrec;
  for (int h = 0; h < nrec; ++h) {
    const double* r = hh.data() + kRec * h;
    const double obj = 0.5 * r[1] - r[2] - r[3] + 0.5 * gamma * (r[4] + r[5]);
    if (out->hist_iter) out->hist_iter[h] = h * stride;
    if (out->hist_objective)  // symmetric: each unordered pair once (:75-78)
      out->hist_objective[h] = (diag->want_objective ? (sym ? 0.5 * obj : obj) : 0.0);
    if (out->hist_rms)
      out->hist_rms[h] = diag->want_rms ? std::sqrt(r[0] / static_cast<double>(m + n)) : 0.0;
  }
}

}  // namespace

extern "C" {

equil_status equil_sgd_equilibrate_symmetric(equil_matrix* M, const equil_params* p,
                                             const equil_diag_cfg* diag,
                                             equil_scaling_out* out) {
  return guarded([&] {
    require(M != nullptr && p != nullptr && out != nullptr,
            "sgd_equilibrate_symmetric: null argument");
    sgd_variant(M, Variant::kSymmetric, p, diag, out, nullptr, nullptr, 0, 0);
  });
}

equil_status equil_sgd_equilibrate_block(equil_matrix* M, const int64_t* row_block,
                                         const int64_t* col_block, int64_t row_blocks,
                                         int64_t col_blocks, const equil_params* p,
                                         const equil_diag_cfg* diag, equil_scaling_out* out) {
  return guarded([&] {
    require(M != nullptr && p != nullptr && out != nullptr,
            "sgd_equilibrate_block: null argument");
    sgd_variant(M, Variant::kBlock, p, diag, out, row_block, col_block, row_blocks, col_blocks);
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// spectral_norm (src/lsqr.cpp:140-163) and the Chambolle-Pock lasso
// (src/ccp.cpp:27-160): the second consumer of the equilibration's d, e.
// Device vectors, canonical reductions; the lasso objective of every iterate
// is evaluated on the device into a history array, so a run without an early
// stop test synchronises only at its end.  Single GPU.
// ---------------------------------------------------------------------------
namespace {

// power iteration on diag(d) A diag(e) (d, e null: A), uncharged
double spectral_norm_dev(equil_matrix* M, const double* d, const double* e, int max_iters,
                         double rel_tol, uint64_t seed) {
  require(max_iters > 0, "spectral_norm: max_iters must be positive");
  const int64_t m = M->m, n = M->n;
  cudaStream_t s = M->stream;
  HostRng rng(seed, 19);  // streams::kPowerIteration
  std::vector<double> xh(n);
  for (int64_t j = 0; j < n; ++j) xh[j] = rng.normal();
  DevBuf<double> x, y, z, t;
  x.alloc(n); y.alloc(m); z.alloc(n); t.alloc(std::max(m, n));
  double* sc = M->scal.p + 40;
  CK(cudaMemcpyAsync(x.p, xh.data(), n * 8, cudaMemcpyHostToDevice, s));
  canon_reduce(M, x.p, n, sc + 0, 0, 0.0, true);
  const double xn = read_scalar(M, sc + 0);
  if (!(xn > 0.0)) fail(EQUIL_ERUNTIME, "spectral_norm: degenerate start");
  CK(eqb::launch_lsqr_normalize(x.p, x.p, sc + 0, nullptr, nullptr, n, nullptr, nullptr, s));
  double lambda = 0.0;
  for (int it = 0; it < max_iters; ++it) {
    const double* xg = x.p;
    if (e) {
      CK(eqb::launch_mul(t.p, e, x.p, n, s));
      xg = t.p;
    }
    apply_pass(M, false, xg, y.p, eqb::kPassScaled, d, nullptr, nullptr);
    canon_reduce(M, y.p, m, sc + 1, 0);
    const double next = read_scalar(M, sc + 1);
    if (next == 0.0) return 0.0;
    const bool settled = std::abs(next - lambda) <= rel_tol * next;
    lambda = next;
    if (settled) break;
    const double* yg = y.p;
    if (d) {
      CK(eqb::launch_mul(t.p, d, y.p, m, s));
      yg = t.p;
    }
    apply_pass(M, true, yg, z.p, eqb::kPassScaled, e, nullptr, nullptr);
    canon_reduce(M, z.p, n, sc + 2, 0, 0.0, true);
    const double zn = read_scalar(M, sc + 2);
    if (zn == 0.0) break;
    CK(eqb::launch_lsqr_normalize(x.p, z.p, sc + 2, nullptr, nullptr, n, nullptr, nullptr, s));
  }
  return std::sqrt(lambda);
}

// lasso_objective (src/ccp.cpp:115-123) of device x into *out (device)
void lasso_value_dev(equil_matrix* M, const double* b_d, double sqrt_lambda, const double* x,
                     const double* absx, double* r, double* out) {
  apply_pass(M, false, x, r, eqb::kPassResid, nullptr, b_d, nullptr);  // b - Ax: same squares
  double* sc = M->scal.p + 44;
  canon_reduce(M, r, M->m, sc + 0, 0);
  canon_reduce(M, absx, M->n, sc + 1, 1);
  CK(eqb::launch_lasso_value(sc + 0, sc + 1, sqrt_lambda, out, M->stream));
}

void ccp_common(equil_matrix* M, const double* b, double lambda, const equil_params* p,
                const equil_ccp_options* o, equil_ccp_out* out, const char* who) {
  require(M != nullptr && o != nullptr && out != nullptr, std::string(who) + ": null argument");
  require(b != nullptr, "lasso: rhs length mismatch");
  std::lock_guard<std::mutex> lk(M->mu);
  DeviceGuard dg(M->device);
  require(M->world == 1, std::string(who) + ": single-GPU matrices only in this build");
  cudaStream_t s = M->stream;
  const int64_t m = M->m, n = M->n;
  // validate_problem (:11-17)
  require(lambda > 0.0, "lasso: lambda must be positive");
  DevBuf<double> b_d;
  b_d.alloc(m);
  CK(cudaMemcpyAsync(b_d.p, b, m * 8, cudaMemcpyHostToDevice, s));
  canon_reduce(M, b_d.p, m, M->scal.p + 48, 0, 0.0, true);
  require(read_scalar(M, M->scal.p + 48) > 0.0, "lasso: rhs must be nonzero");
  require(o->max_iters >= 0, std::string(who) + ": max_iters must be nonnegative");
  const int T = p ? p->iterations : 0;
  require(out->objective_history != nullptr &&
              out->hist_cap >= std::max(o->max_iters, 0) + 1 + std::max(T, 0),
          std::string(who) + ": history capacity too small");
  const bool track = std::isfinite(o->p_star);
  require(!track || out->gap_history != nullptr, std::string(who) + ": gap_history missing");

  long long applies = 0, adjoints = 0;
  DevBuf<double> dd, ed;
  const double* d = nullptr;
  const double* e = nullptr;
  if (p) {  // sgd_equilibrate on the charged operator (:139)
    dd.alloc(m);
    ed.alloc(n);
    equil_scaling_out so{};
    so.d = dd.p;
    so.e = ed.p;
    so.outputs_on_device = 1;
    M->mu.unlock();
    const equil_status rc = equil_sgd_equilibrate(M, p, nullptr, &so);
    M->mu.lock();
    if (rc != EQUIL_OK) fail(rc, g_err);
    applies = so.apply_count;
    adjoints = so.adjoint_count;
    d = dd.p;
    e = ed.p;
  }
  // ccp_core (:27-110)
  const double sl = std::sqrt(lambda);
  double tau, sigma;
  if (o->tau > 0.0 && o->sigma > 0.0) {
    tau = o->tau;
    sigma = o->sigma;
  } else {
    const double norm2 = spectral_norm_dev(M, d, e, 100, 1e-9, 0);
    if (!(norm2 > 0.0)) fail(EQUIL_ERUNTIME, "ccp_lasso: zero operator");
    tau = 0.9 / norm2;
    sigma = 0.9 / norm2;
  }
  const double f0 = [&] {
    DevBuf<double> zero, r, v;
    zero.alloc(n);
    r.alloc(m);
    v.alloc(1);
    CK(cudaMemsetAsync(zero.p, 0, n * 8, s));
    lasso_value_dev(M, b_d.p, sl, zero.p, zero.p, r.p, v.p);
    return read_scalar(M, v.p);
  }();
  int hl = 0, gl = 0;
  bool reached = false;
  auto push = [&](double f) {
    out->objective_history[hl++] = f;
    if (track) out->gap_history[gl++] = (f - o->p_star) / f0;
  };
  for (int t = 0; t <= T; ++t) push(f0);
  if (track && o->gap_tol > 0.0 && out->gap_history[gl - 1] <= o->gap_tol) reached = true;

  DevBuf<double> y, kz, dy, z, ezt, g, x, absx, r, fh;
  y.alloc(m); kz.alloc(m); dy.alloc(m); r.alloc(m);
  z.alloc(n); ezt.alloc(n); g.alloc(n); x.alloc(n); absx.alloc(n);
  const int iters = std::max(o->max_iters, 0);
  fh.alloc(std::max(iters, 1));
  CK(cudaMemsetAsync(y.p, 0, m * 8, s));
  CK(cudaMemsetAsync(z.p, 0, n * 8, s));
  CK(cudaMemsetAsync(ezt.p, 0, n * 8, s));
  CK(cudaMemsetAsync(x.p, 0, n * 8, s));
  const bool early = track && o->gap_tol > 0.0;  // stop test needs f on the host
  int done = 0;
  for (int t = 1; t <= iters && !reached; ++t) {
    apply_pass(M, false, ezt.p, kz.p, eqb::kPassScaled, d, nullptr, nullptr);  // K z~
    ++applies;
    CK(eqb::launch_ccp_dual(y.p, kz.p, d, b_d.p, sigma, sl, m, dy.p, s));
    apply_pass(M, true, dy.p, g.p, eqb::kPassScaled, e, nullptr, nullptr);  // K^T y
    ++adjoints;
    CK(eqb::launch_ccp_primal(z.p, ezt.p, g.p, e, tau, tau * sl, o->theta, n, x.p, absx.p, s));
    lasso_value_dev(M, b_d.p, sl, x.p, absx.p, r.p, fh.p + (t - 1));  // uncharged probe
    done = t;
    if (early) {
      push(read_scalar(M, fh.p + (t - 1)));
      if (out->gap_history[gl - 1] <= o->gap_tol) reached = true;
    }
  }
  if (!early && done > 0) {
    std::vector<double> f(done);
    CK(cudaMemcpyAsync(f.data(), fh.p, done * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (double v : f) push(v);
  }
  if (out->x) CK(cudaMemcpyAsync(out->x, x.p, n * 8, cudaMemcpyDeviceToHost, s));  // e .* z
  CK(cudaStreamSynchronize(s));
  out->hist_len = hl;
  out->gap_len = gl;
  out->tau = tau;
  out->sigma = sigma;
  out->theta = o->theta;
  out->iterations = done;
  out->equil_iterations = T;
  out->reached_tol = reached ? 1 : 0;
  out->apply_count = applies;
  out->adjoint_count = adjoints;
}

}  // namespace

extern "C" {

equil_status equil_spectral_norm(equil_matrix* M, int max_iters, double rel_tol, uint64_t seed,
                                 double* out) {
  return guarded([&] {
    require(M != nullptr && out != nullptr, "spectral_norm: null argument");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    require(M->world == 1, "spectral_norm: single-GPU matrices only in this build");
    *out = spectral_norm_dev(M, nullptr, nullptr, max_iters, rel_tol, seed);
  });
}

equil_status equil_lasso_objective(equil_matrix* M, const double* b, double lambda,
                                   const double* x, double* out) {
  return guarded([&] {
    require(M != nullptr && b != nullptr && x != nullptr && out != nullptr,
            "lasso_objective: null argument");
    require(lambda > 0.0, "lasso_objective: malformed problem");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    require(M->world == 1, "lasso_objective: single-GPU matrices only in this build");
    cudaStream_t s = M->stream;
    DevBuf<double> b_d, x_d, ax, r, v;
    b_d.alloc(M->m); x_d.alloc(M->n); ax.alloc(M->n); r.alloc(M->m); v.alloc(1);
    CK(cudaMemcpyAsync(b_d.p, b, M->m * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(x_d.p, x, M->n * 8, cudaMemcpyHostToDevice, s));
    CK(eqb::launch_abs(x_d.p, M->n, ax.p, s));
    lasso_value_dev(M, b_d.p, std::sqrt(lambda), x_d.p, ax.p, r.p, v.p);
    *out = read_scalar(M, v.p);
  });
}

equil_status equil_ccp_lasso(equil_matrix* M, const double* b, double lambda,
                             const equil_ccp_options* o, equil_ccp_out* out) {
  return guarded([&] { ccp_common(M, b, lambda, nullptr, o, out, "ccp_lasso"); });
}

equil_status equil_ccp_lasso_preconditioned(equil_matrix* M, const double* b, double lambda,
                                            const equil_params* p, const equil_ccp_options* o,
                                            equil_ccp_out* out) {
  return guarded([&] {
    require(p != nullptr, "ccp_lasso_preconditioned: null params");
    ccp_common(M, b, lambda, p, o, out, "ccp_lasso_preconditioned");
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Matrix store ingest: Matrix Market files
// (src/matrix_market.cpp) parsed on host threads, sorted / checked / converted
// to CSR on the device; a binary CSR file for fast reloads; host export.
// ---------------------------------------------------------------------------
namespace {

// the local CSR(A) (world 1) or dense A on the host
void export_host(equil_matrix* M, std::vector<int64_t>& rp, std::vector<int32_t>& ci,
                 std::vector<double>& va, std::vector<double>& dense) {
  require(M->world == 1, "export: single-GPU matrices only");
  cudaStream_t s = M->stream;
  if (M->dense) {
    dense.resize(static_cast<size_t>(M->m * M->n));
    CK(cudaMemcpyAsync(dense.data(), M->Ad.p, M->m * M->n * 8, cudaMemcpyDeviceToHost, s));
  } else {
    rp.resize(M->m + 1);
    ci.resize(static_cast<size_t>(M->nnz));
    va.resize(static_cast<size_t>(M->nnz));
    CK(cudaMemcpyAsync(rp.data(), M->A.row_ptr, (M->m + 1) * 8, cudaMemcpyDeviceToHost, s));
    if (M->nnz) {
      CK(cudaMemcpyAsync(ci.data(), M->A.col, M->nnz * 4, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(va.data(), M->A.val, M->nnz * 8, cudaMemcpyDeviceToHost, s));
    }
  }
  CK(cudaStreamSynchronize(s));
}

}  // namespace

extern "C" {

equil_status equil_matrix_read_matrix_market(const char* path, const equil_device_cfg* cfg,
                                             equil_matrix** out) {
  return guarded([&] {
    require(path != nullptr && out != nullptr, "matrix market: null argument");
    *out = nullptr;
    std::string buf;
    eqb::mm::read_file(path, buf);
    eqb::mm::Matrix mm;
    eqb::mm::parse(buf.data(), buf.size(), mm);
    buf.clear();
    buf.shrink_to_fit();
    if (mm.dense) {
      const equil_status rc =
          equil_matrix_create_dense(mm.m, mm.n, mm.dense_rowmajor.data(), cfg, out);
      if (rc != EQUIL_OK) fail(rc, g_err);
      return;
    }
    create_coo_impl(mm.m, mm.n, mm.nnz, mm.row.data(), mm.col.data(), mm.val.data(),
                    mm.line.data(), cfg, out);
  });
}

equil_status equil_matrix_write_matrix_market(equil_matrix* M, const char* path) {
  return guarded([&] {
    require(M != nullptr && path != nullptr, "matrix market: null argument");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    std::vector<int64_t> rp;
    std::vector<int32_t> ci;
    std::vector<double> va, dense;
    export_host(M, rp, ci, va, dense);
    if (M->dense)
      eqb::mm::write_array(path, M->m, M->n, dense.data());
    else
      eqb::mm::write_coordinate(path, M->m, M->n, rp.data(), ci.data(), va.data());
  });
}

equil_status equil_matrix_save_binary(equil_matrix* M, const char* path) {
  return guarded([&] {
    require(M != nullptr && path != nullptr, "binary csr: null argument");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    std::vector<int64_t> rp;
    std::vector<int32_t> ci;
    std::vector<double> va, dense;
    export_host(M, rp, ci, va, dense);
    eqb::mm::write_binary(path, M->m, M->n, M->dense, rp.data(), ci.data(), va.data(),
                          dense.data());
  });
}

equil_status equil_matrix_load_binary(const char* path, const equil_device_cfg* cfg,
                                      equil_matrix** out) {
  return guarded([&] {
    require(path != nullptr && out != nullptr, "binary csr: null argument");
    *out = nullptr;
    FILE* f = std::fopen(path, "rb");
    if (!f) throw std::runtime_error(std::string("binary csr: cannot open '") + path + "'");
    struct Closer {
      FILE* f;
      ~Closer() { std::fclose(f); }
    } closer{f};
    int64_t hdr[4];
    eqb::mm::read_binary_header(f, path, hdr);
    const int64_t m = hdr[0], n = hdr[1], nnz = hdr[2];
    // read straight into pinned host buffers (fast H2D in the create call)
    auto pinned = [](size_t bytes) {
      void* p = nullptr;
      CK(cudaMallocHost(&p, std::max<size_t>(bytes, 8)));
      return p;
    };
    struct Pinned {
      void* p;
      ~Pinned() { if (p) cudaFreeHost(p); }
    };
    equil_status rc;
    if (hdr[3]) {
      Pinned a{pinned(static_cast<size_t>(nnz) * 8)};
      eqb::mm::read_exact(f, a.p, 8, static_cast<size_t>(nnz), path);
      rc = equil_matrix_create_dense(m, n, static_cast<const double*>(a.p), cfg, out);
    } else {
      Pinned rp{pinned(static_cast<size_t>(m + 1) * 8)};
      Pinned ci{pinned(static_cast<size_t>(nnz) * 4)};
      Pinned va{pinned(static_cast<size_t>(nnz) * 8)};
      eqb::mm::read_exact(f, rp.p, 8, static_cast<size_t>(m + 1), path);
      eqb::mm::read_exact(f, ci.p, 4, static_cast<size_t>(nnz), path);
      eqb::mm::read_exact(f, va.p, 8, static_cast<size_t>(nnz), path);
      rc = equil_matrix_create_csr(m, n, static_cast<const int64_t*>(rp.p),
                                   static_cast<const int32_t*>(ci.p),
                                   static_cast<const double*>(va.p), cfg, out);
    }
    if (rc != EQUIL_OK) fail(rc, g_err);
  });
}

equil_status equil_matrix_export_csr(equil_matrix* M, int64_t* row_ptr, int32_t* col,
                                     double* val) {
  return guarded([&] {
    require(M != nullptr && row_ptr != nullptr, "export_csr: null argument");
    require(!M->dense, "export_csr: dense matrix");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    std::vector<int64_t> rp;
    std::vector<int32_t> ci;
    std::vector<double> va, dense;
    export_host(M, rp, ci, va, dense);
    std::memcpy(row_ptr, rp.data(), rp.size() * 8);
    if (M->nnz) {
      std::memcpy(col, ci.data(), ci.size() * 4);
      std::memcpy(val, va.data(), va.size() * 8);
    }
  });
}

equil_status equil_matrix_export_dense(equil_matrix* M, double* rowmajor) {
  return guarded([&] {
    require(M != nullptr && rowmajor != nullptr, "export_dense: null argument");
    require(M->dense, "export_dense: sparse matrix");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    std::vector<int64_t> rp;
    std::vector<int32_t> ci;
    std::vector<double> va, dense;
    export_host(M, rp, ci, va, dense);
    std::memcpy(rowmajor, dense.data(), dense.size() * 8);
  });
}

int equil_matrix_is_dense(const equil_matrix* M) { return M && M->dense ? 1 : 0; }

}  // extern "C"

// Host-only Matrix Market access (no device needed): parse into a handle,
// fetch the entries, write a host CSR / dense array.
extern "C" {

equil_status equil_mm_parse(const char* path, int64_t* m, int64_t* n, int64_t* nnz, int* dense,
                            void** handle) {
  return guarded([&] {
    require(path && m && n && nnz && dense && handle, "matrix market: null argument");
    *handle = nullptr;
    std::string buf;
    eqb::mm::read_file(path, buf);
    auto mm = std::make_unique<eqb::mm::Matrix>();
    eqb::mm::parse(buf.data(), buf.size(), *mm);
    *m = mm->m;
    *n = mm->n;
    *nnz = mm->nnz;
    *dense = mm->dense ? 1 : 0;
    *handle = mm.release();
  });
}

equil_status equil_mm_fetch(void* handle, int64_t* rows, int64_t* cols, double* vals,
                            int64_t* lines) {
  return guarded([&] {
    require(handle != nullptr, "matrix market: null handle");
    const auto* mm = static_cast<const eqb::mm::Matrix*>(handle);
    if (mm->dense) {
      if (vals) std::memcpy(vals, mm->dense_rowmajor.data(), mm->dense_rowmajor.size() * 8);
      return;
    }
    if (rows) std::memcpy(rows, mm->row.data(), mm->row.size() * 8);
    if (cols) std::memcpy(cols, mm->col.data(), mm->col.size() * 8);
    if (vals) std::memcpy(vals, mm->val.data(), mm->val.size() * 8);
    if (lines) std::memcpy(lines, mm->line.data(), mm->line.size() * 8);
  });
}

void equil_mm_free(void* handle) { delete static_cast<eqb::mm::Matrix*>(handle); }

equil_status equil_mm_write_csr(const char* path, int64_t m, int64_t n, const int64_t* row_ptr,
                                const int32_t* col, const double* val) {
  return guarded([&] {
    require(path && row_ptr && m > 0 && n > 0, "matrix market: null argument");
    eqb::mm::write_coordinate(path, m, n, row_ptr, col, val);
  });
}

equil_status equil_mm_write_dense(const char* path, int64_t m, int64_t n,
                                  const double* rowmajor) {
  return guarded([&] {
    require(path && rowmajor && m > 0 && n > 0, "matrix market: null argument");
    eqb::mm::write_array(path, m, n, rowmajor);
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Public helpers of include/equil/equilibrate.hpp and metrics.hpp on the device
// matrix: objective / gradient (weighted and plain), the one-sample stochastic
// gradient estimate, rms_error, project_box.  Per-row sums follow CSR order
// (A's rows for u, A^T's rows = ascending original rows for v); whole-vector
// sums use the canonical reduction; exp is det_exp (the numerics contract).
// Single GPU, sparse matrices (the estimate also takes dense ones).
// ---------------------------------------------------------------------------
namespace {

struct HelperCtx {
  equil_matrix* M;
  cudaStream_t s;
  DevBuf<double> u, v, lu, lv, tm, tn;
  HelperCtx(equil_matrix* m, const double* uh, const double* vh, const char* who,
            bool need_csr = true)
      : M(m), s(m->stream) {
    require(M->world == 1, std::string(who) + ": single-GPU matrices only in this build");
    require(!need_csr || !M->dense, std::string(who) + ": sparse matrices only in this build");
    u.alloc(M->m);
    v.alloc(M->n);
    tm.alloc(M->m);
    tn.alloc(M->n);
    CK(cudaMemcpyAsync(u.p, uh, M->m * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(v.p, vh, M->n * 8, cudaMemcpyHostToDevice, s));
  }
  const double* upload_lin(DevBuf<double>& b, const double* h, int64_t len) {
    if (!h) return nullptr;
    b.alloc(len);
    CK(cudaMemcpyAsync(b.p, h, len * 8, cudaMemcpyHostToDevice, s));
    return b.p;
  }
};

// objective_weighted (src/equilibrate.cpp:10-22); lin arrays null: constants
double objective_dev(HelperCtx& c, const double* lin_u, double lu_c, const double* lin_v,
                     double lv_c, double gamma) {
  equil_matrix* M = c.M;
  double* sc = M->scal.p + 52;
  CK(eqb::launch_obj_terms(M->A, c.u.p, c.v.p, c.tm.p, c.s));
  canon_reduce(M, c.tm.p, M->m, sc + 0, 1);
  if (lin_u) {
    CK(eqb::launch_mul(c.tm.p, lin_u, c.u.p, M->m, c.s));
    canon_reduce(M, c.tm.p, M->m, sc + 1, 1);
  } else {
    canon_reduce(M, c.u.p, M->m, sc + 1, 2, lu_c);
  }
  if (lin_v) {
    CK(eqb::launch_mul(c.tn.p, lin_v, c.v.p, M->n, c.s));
    canon_reduce(M, c.tn.p, M->n, sc + 2, 1);
  } else {
    canon_reduce(M, c.v.p, M->n, sc + 2, 2, lv_c);
  }
  canon_reduce(M, c.u.p, M->m, sc + 3, 0);
  canon_reduce(M, c.v.p, M->n, sc + 4, 0);
  double r[5];
  CK(cudaMemcpyAsync(r, sc, sizeof r, cudaMemcpyDeviceToHost, c.s));
  CK(cudaStreamSynchronize(c.s));
  return 0.5 * r[0] - r[1] - r[2] + 0.5 * gamma * (r[3] + r[4]);
}

// gradient_weighted (src/equilibrate.cpp:24-37)
void gradient_dev(HelperCtx& c, const double* lin_u, double lu_c, const double* lin_v,
                  double lv_c, double gamma, double* gu_h, double* gv_h) {
  equil_matrix* M = c.M;
  CK(eqb::launch_obj_terms(M->A, c.u.p, c.v.p, c.tm.p, c.s));   // sum_j a^2 e^{2(u_i+v_j)}
  CK(eqb::launch_obj_terms(M->AT, c.v.p, c.u.p, c.tn.p, c.s));  // ascending i per column
  CK(eqb::launch_grad_finish(c.tm.p, c.u.p, lin_u, lu_c, gamma, M->m, c.s));
  CK(eqb::launch_grad_finish(c.tn.p, c.v.p, lin_v, lv_c, gamma, M->n, c.s));
  CK(cudaMemcpyAsync(gu_h, c.tm.p, M->m * 8, cudaMemcpyDeviceToHost, c.s));
  CK(cudaMemcpyAsync(gv_h, c.tn.p, M->n * 8, cudaMemcpyDeviceToHost, c.s));
  CK(cudaStreamSynchronize(c.s));
}

}  // namespace

extern "C" {

equil_status equil_objective_weighted(equil_matrix* M, const double* u, const double* v,
                                      const double* lin_u, const double* lin_v, double gamma,
                                      double* out) {
  return guarded([&] {
    require(M && u && v && lin_u && lin_v && out, "objective: null argument");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    HelperCtx c(M, u, v, "objective");
    const double* lu = c.upload_lin(c.lu, lin_u, M->m);
    const double* lv = c.upload_lin(c.lv, lin_v, M->n);
    *out = objective_dev(c, lu, 0.0, lv, 0.0, gamma);
  });
}

equil_status equil_objective(equil_matrix* M, const double* u, const double* v,
                             const equil_params* p, double* out) {
  return guarded([&] {
    require(M && u && v && p && out, "objective: null argument");
    validate_params(*p);
    double alpha = 0, beta = 0;
    resolve_targets(*p, M->m, M->n, alpha, beta);
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    HelperCtx c(M, u, v, "objective");
    *out = objective_dev(c, nullptr, alpha * alpha, nullptr, beta * beta, p->gamma);
  });
}

equil_status equil_gradient_weighted(equil_matrix* M, const double* u, const double* v,
                                     const double* lin_u, const double* lin_v, double gamma,
                                     double* grad_u, double* grad_v) {
  return guarded([&] {
    require(M && u && v && lin_u && lin_v && grad_u && grad_v, "gradient: null argument");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    HelperCtx c(M, u, v, "gradient");
    const double* lu = c.upload_lin(c.lu, lin_u, M->m);
    const double* lv = c.upload_lin(c.lv, lin_v, M->n);
    gradient_dev(c, lu, 0.0, lv, 0.0, gamma, grad_u, grad_v);
  });
}

equil_status equil_gradient(equil_matrix* M, const double* u, const double* v,
                            const equil_params* p, double* grad_u, double* grad_v) {
  return guarded([&] {
    require(M && u && v && p && grad_u && grad_v, "gradient: null argument");
    validate_params(*p);
    double alpha = 0, beta = 0;
    resolve_targets(*p, M->m, M->n, alpha, beta);
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    HelperCtx c(M, u, v, "gradient");
    gradient_dev(c, nullptr, alpha * alpha, nullptr, beta * beta, p->gamma, grad_u, grad_v);
  });
}

// stochastic_gradient_estimate (src/equilibrate.cpp:60-71): the probes are
// outputs [offset, offset + n + m) of SeededRng(seed, stream) (s then w)
equil_status equil_stochastic_gradient_estimate(equil_matrix* M, const double* u,
                                                const double* v, const equil_params* p,
                                                uint64_t seed, uint64_t stream, uint64_t offset,
                                                double* g_u, double* g_v) {
  return guarded([&] {
    require(M && u && v && p && g_u && g_v, "stochastic_gradient_estimate: null argument");
    validate_params(*p);
    double alpha = 0, beta = 0;
    resolve_targets(*p, M->m, M->n, alpha, beta);
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    HelperCtx c(M, u, v, "stochastic_gradient_estimate", false);
    const int64_t m = M->m, n = M->n;
    const uint64_t total = offset + static_cast<uint64_t>(m + n);
    DevBuf<uint32_t> bits;
    DevBuf<unsigned char> scratch;
    bits.alloc((total + 31) / 32 + 1);
    const size_t sb = eqb::sign_stream_scratch_bytes(total);
    scratch.alloc(sb);
    CK(eqb::sign_stream_generate(seed, stream, total, bits.p, scratch.p, sb, c.s));
    DevBuf<double> d, e, xs, xw;
    d.alloc(m); e.alloc(n); xs.alloc(n); xw.alloc(m);
    // d = exp(u), e = exp(v); xs = e .* s; xw = d .* w
    CK(eqb::launch_expand_scale(c.v.p, nullptr, n, bits.p, static_cast<int64_t>(offset), e.p,
                                xs.p, c.s));
    CK(eqb::launch_expand_scale(c.u.p, nullptr, m, bits.p, static_cast<int64_t>(offset) + n,
                                d.p, xw.p, c.s));
    apply_pass(M, false, xs.p, c.tm.p, eqb::kPassEst, d.p, nullptr, nullptr);
    apply_pass(M, true, xw.p, c.tn.p, eqb::kPassEst, e.p, nullptr, nullptr);
    CK(eqb::launch_sge_finish(c.tm.p, c.u.p, -alpha * alpha, p->gamma, m, c.s));
    CK(eqb::launch_sge_finish(c.tn.p, c.v.p, -beta * beta, p->gamma, n, c.s));
    CK(cudaMemcpyAsync(g_u, c.tm.p, m * 8, cudaMemcpyDeviceToHost, c.s));
    CK(cudaMemcpyAsync(g_v, c.tn.p, n * 8, cudaMemcpyDeviceToHost, c.s));
    CK(cudaStreamSynchronize(c.s));
  });
}

// rms_error (src/metrics.cpp:41-56)
equil_status equil_rms_error(equil_matrix* M, const double* u, const double* v, double alpha,
                             double beta, double* out) {
  return guarded([&] {
    require(M && u && v && out, "rms_error: null argument");
    require(alpha > 0.0 && beta > 0.0, "rms_error: targets must be positive");
    std::lock_guard<std::mutex> lk(M->mu);
    DeviceGuard dg(M->device);
    HelperCtx c(M, u, v, "rms_error");
    DevBuf<double> terms;
    terms.alloc(M->m + M->n);
    CK(eqb::launch_exp(c.u.p, c.tm.p, M->m, 2.0, c.s));
    CK(eqb::launch_exp(c.v.p, c.tn.p, M->n, 2.0, c.s));
    CK(eqb::launch_rms_terms(0, M->A, c.tm.p, c.tn.p, terms.p, 0, alpha, c.s));
    CK(eqb::launch_rms_terms(1, M->AT, c.tm.p, c.tn.p, terms.p + M->m, 0, beta, c.s));
    canon_reduce(M, terms.p, M->m + M->n, M->scal.p + 58, 1);
    *out = std::sqrt(read_scalar(M, M->scal.p + 58) / static_cast<double>(M->m + M->n));
  });
}

// project_box (src/equilibrate.cpp:73-76), host
equil_status equil_project_box(const double* x, int64_t n, double bound, double* out) {
  return guarded([&] {
    require(bound >= 0.0, "project_box: bound must be nonnegative");
    require(n == 0 || (x && out), "project_box: null argument");
    for (int64_t i = 0; i < n; ++i) {
      const double lo = x[i] < -bound ? -bound : x[i];  // cwiseMax(-bound)
      out[i] = bound < lo ? bound : lo;                  // cwiseMin(bound)
    }
  });
}

}  // extern "C"
