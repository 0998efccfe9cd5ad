// internal.h -- shared declarations between the kernels and the host engine.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <functional>
#include <vector>

#include "det_math.cuh"

namespace eqb {

// Checked build (EQUIL_DEFS=-DEQ_CHECKED, libequil_b200_checked.so): device-side
// bounds / protocol assertions that trap on failure.  compute-sanitizer is not
// available on the GPU pool, so tests/test_gpu_checked.py runs the workloads on
// this build instead.
#ifdef EQ_CHECKED
#define EQ_CHECK(c)                                                              \
  do {                                                                           \
    if (!(c)) {                                                                  \
      printf("EQ_CHECK failed at %s:%d: %s\n", __FILE__, __LINE__, #c);          \
      __trap();                                                                  \
    }                                                                            \
  } while (0)
#else
#define EQ_CHECK(c) \
  do {              \
  } while (0)
#endif

// Sparse traversal tile.  kind 2 (one warp): a slice of r1 (<= 32) rows listed
// at rowlist[r0 ...], sorted by length (longest first), summed one row per lane
// in lock-step chunks.  kind 3 (one CTA): a long slice of r1 rows longer than
// kTileNnz, staged cooperatively.  mat 0 = A (u block), mat 1 = A^T (v block).
struct Tile {
  int32_t r0, r1;
  int16_t kind, mat;
  int32_t pad;
};
#ifndef EQ_MAX_PEERS
#define EQ_MAX_PEERS 7  // fused all-gather up to 8 ranks (one NVSwitch node)
#endif
#ifndef EQ_SLICE_BATCH
#define EQ_SLICE_BATCH 6
#endif
#ifndef EQ_LONG_BATCH
#define EQ_LONG_BATCH 4
#endif
#ifndef EQ_LONG_THRESH
#define EQ_LONG_THRESH 512
#endif
constexpr int kTileNnz = EQ_LONG_THRESH;  // longest row of a slice; longer rows: kind 3
#ifndef EQ_MID_MAX
#define EQ_MID_MAX 0
#endif
constexpr int kMidMax = EQ_MID_MAX;  // rows in (kTileNnz, kMidMax]: globally sorted warp slices
constexpr int kSliceChunk = 16;  // products per row per lock-step round (kind 2)
constexpr int kSliceStride = 18; // padded row stride (doubles): conflict-free LDS.128
constexpr int kSliceBatch = EQ_SLICE_BATCH;  // row pairs staged per batch (loads in flight)
constexpr int kSliceRows = 32;
#ifndef EQ_SLICE_PREFETCH
#define EQ_SLICE_PREFETCH 0  // rounds of L2 prefetch ahead in kind-2 slices (0: off)
#endif
#ifndef EQ_SLICE_WINDOW
#define EQ_SLICE_WINDOW 4096
#endif
constexpr int kSliceWindow = EQ_SLICE_WINDOW;  // rows are length-sorted within windows
constexpr int kWarpSmem = kTileNnz > 32 * kSliceStride ? kTileNnz : 32 * kSliceStride;
constexpr int kTileWarps = 4;    // independent warps per CTA
constexpr int kTileThreads = 32 * kTileWarps;

struct __align__(16) RowMeta {
  int64_t start;  // chunk-aligned base of the row's CSR range
  int32_t k0;     // row start relative to start
  int32_t len;    // row end relative to start
};
#ifndef EQ_LONG_CHUNK
#define EQ_LONG_CHUNK 64
#endif
constexpr int kLongChunk = EQ_LONG_CHUNK;      // products per row per round (kind 3)
constexpr int kLongStride = kLongChunk + 2;    // padded stride: conflict-free LDS.128
constexpr int kLongBatch = EQ_LONG_BATCH;  // rows per staging batch per warp
#ifndef EQ_LONG_ROWS
#define EQ_LONG_ROWS 32
#endif
constexpr int kLongRows = EQ_LONG_ROWS;  // rows per CTA-cooperative long slice
static_assert(kLongRows <= 32 && kLongRows * kLongStride <= kTileWarps * kWarpSmem,
              "long slice staging must fit the CTA's buffers");
struct SliceMeta {
  RowMeta r[32];
  int maxr;  // long slices: rounds of the longest row
};
constexpr int kTileMinBlocks = 6;   // 24 warps/SM: <= 80 registers (no spills)

// CSR slice resident on the device (int64 row_ptr, int32 col, fp64 val).
struct DevCsr {
  int64_t rows = 0, cols = 0, nnz = 0;
  int64_t* row_ptr = nullptr;
  int32_t* col = nullptr;
  double* val = nullptr;
};

struct SgdIterArgs {
  const int64_t* rp[2];
  const int32_t* ci[2];
  const double* va[2];
  const int32_t* rl[2];  // slice row lists
  const Tile* tiles;
  int n_long;            // leading kind-3 entries of tiles
  const double* xs_cur;  // gathered e.*s (n, padded coords)
  const double* xw_cur;  // gathered d.*w (m, padded coords)
  double* xs_next;
  double* xw_next;
  double* x[2];    // u (local rows of A), v (local rows of A^T)
  double* avg[2];  // ubar, vbar
  int64_t goff[2];   // global index of local row 0 (A rows, A^T rows)
  int64_t poff[2];   // padded index of local row 0 (into xw / xs)
  const uint32_t* signs;  // packed sign bits
  int64_t sign_next[2];   // bit index of (local row 0) for iteration t+1: w, s
  int has_next;
  SgdBlockConst c[2];
  const double* lin[2];  // per-coordinate linear terms (local rows) or nullptr
  // slot of local row r in the gathered vector it feeds (xw for A rows, xs for
  // A^T rows), or nullptr for the plain padded position poff + r.  A layout
  // with the most-gathered coordinates packed first keeps them L1-resident.
  const int32_t* slot[2];
  // column blocks of the gathered vectors (gathers larger than L2): this
  // launch's round, blocks per matrix (1: none), per-row interior block
  // boundaries (nblk - 1 offsets into the row) and the carried running sums
  int round;
  int nblk[2];
  const int32_t* bnd[2];
  double* carry[2];
  SgdStep st;
  unsigned* flags;
  // fused all-gather (world > 1, EQUIL_P2P): the epilogue also stores each next
  // value at the same position of every peer rank's gathered vector, over
  // NVLink through CUDA IPC mappings (peer buffer = local buffer + peer_delta[g]
  // elements), so the exchange overlaps the passes; a one-word barrier follows
  int npeer;
  int64_t peer_delta[EQ_MAX_PEERS];
};

// ---- interleaved row slices (sell.cu) --------------------------------------
// The SGD passes' own copy of CSR(A) / CSR(A^T) with the entries of each slice
// of <= 32 length-sorted rows interleaved: entry k of lane l's row sits at
// off + 32 k + l.  A warp streams a slice with fully coalesced 256-byte value
// and 128-byte column loads, and every lane owns one row, so its sequential
// CSR-order sum runs in registers (no shared-memory staging).  Column indices
// are slots of the gathered vector (build_slot_layout).
struct SellSlice {
  int64_t off;     // first element (multiple of 32) in its matrix's arrays
  int32_t maxlen;  // entries of the slice's longest row
  int16_t cnt;     // rows (<= 32)
  int16_t mat;     // 0: A (u block), 1: A^T (v block)
};
struct SellArgs {
  const SellSlice* slices;  // both matrices, longest slices first
  int first, nslices;       // a launch covers positions [first, nslices)
  const int32_t* order;     // position -> slice (nullptr: identity)
  const int32_t* row;       // local row of lane l of slice w at 32 w + l
  const int32_t* len;       // its length (0 for empty lanes)
  const int32_t* ci[2];     // interleaved slot columns
  const double* va[2];      // interleaved values
  int64_t xlen[2];          // length of the gathered vector(s) (checked builds)
  int quad_min;             // slices with maxlen >= quad_min are in the quad layout
};
// Quad layout of a slice: entries 4q .. 4q+3 of lane l are adjacent, at
// off + 128 q + 4 l + (k % 4), so a lane streams its row with 128-bit loads
// (four columns, two pairs of values); the slice is padded to a multiple of 4
// entries.  Slices shorter than quad_min keep entry k of lane l at
// off + 32 k + l (short rows would pay more padding than the loads save).
constexpr int kQuad = 4;
__host__ __device__ inline int64_t sell_quad_len(int64_t maxlen) { return (maxlen + 3) & ~int64_t(3); }
// Device flag barrier of the fused all-gather (world > 1, NCCL transport): a
// tail of kBarWords 64-bit words behind the gathered vectors in xbuf (mapped by
// every peer): [0, world) the last epoch each rank signalled, [kBarEpoch] this
// rank's epoch counter, [kBarError] set if a wait timed out.  peer_delta: the
// peers' xbuf minus this rank's, in 8-byte words (npeer = world - 1).
constexpr int kBarWords = 16;
constexpr int kBarEpoch = 8;
constexpr int kBarError = 9;
cudaError_t launch_peer_barrier(unsigned long long* bar, int rank, int world,
                                const int64_t* peer_delta, int npeer, cudaStream_t s);
// host -> device copy by a kernel reading mapped pinned memory (setup)
cudaError_t launch_pull_copy(void* dst, const void* src_mapped, size_t bytes, cudaStream_t s);
// Fill one matrix's interleaved arrays from its CSR rows, columns mapped
// through map (slots; nullptr: unchanged).  midx: that matrix's slices (indices
// into slices) in launch order; kbp: prefix of their 32-entry blocks.
// kst (nullable): each lane's first entry within its row (column blocks).
// items: kbp[nmat_slices] (known on the host)
cudaError_t build_sell(const int64_t* rp, const int32_t* ci, const int32_t* map, const double* val,
                       const int64_t* kbp, int64_t items, const int32_t* midx, int nmat_slices,
                       const SellSlice* slices, const int32_t* row, const int32_t* len,
                       const int32_t* kst, int32_t* out_ci, double* out_va, cudaStream_t s,
                       int quad_min = 0x7fffffff);  // slices with maxlen >= quad_min: quad layout
// column blocks: per block b and slice lane q, the lane's first entry and
// entry count in block b (kst / bln[b * 32 nslices + q]) and the per-block
// slice maxima maxb[b * nslices + w]
cudaError_t launch_sell_block_lanes(const SellSlice* slices, int nslices, const int32_t* row,
                                    const int32_t* len, const int64_t* rpa, const int32_t* cia,
                                    const int64_t* rpt, const int32_t* cit, int nba, int nbt,
                                    int64_t wa, int64_t wt, int nbmax, int32_t* kst, int32_t* bln,
                                    int32_t* maxb, cudaStream_t s);
// row[32 w + l] / len[32 w + l] of every slice lane from the plans' row lists
// (slice w lists rows rowlist_{mat}[r0[w] ...]); empty lanes get 0 / 0
cudaError_t launch_sell_rows(const SellSlice* slices, const int32_t* r0, int nslices,
                             const int32_t* rowlist_a, const int32_t* rowlist_t,
                             const int64_t* rp_a, const int64_t* rp_t, int32_t* row,
                             int32_t* len, cudaStream_t s);
// one SGD iteration over every slice (both matrices); variant selects the
// compiled batch / pipelining / occupancy point (EQUIL_SELL_VARIANT)
cudaError_t launch_sgd_sell(const SgdIterArgs& a, const SellArgs& sa, int variant,
                            cudaStream_t s);
// split epilogue: the traversal stores row sums in a.carry[mat][row] (lng: the
// long-slice kernel), then the update runs over all local rows
cudaError_t launch_sgd_sell_split(const SgdIterArgs& a, const SellArgs& sa, bool lng,
                                  int variant, cudaStream_t s);
cudaError_t launch_sgd_update_rows(const SgdIterArgs& a, int64_t m_loc, int64_t n_loc,
                                   cudaStream_t s);
// the long slices (one warp-specialised CTA each, EQUIL_SELL_LVARIANT)
cudaError_t launch_sgd_sell_long(const SgdIterArgs& a, const SellArgs& sa, int variant,
                                 cudaStream_t s);

// ---- column-synchronous sweep of A's long rows (sweep.cu) --------------------
struct SweepArgs {
  const unsigned char* blobs;  // per (cta, panel): header | perm | runs | cols | vals
  const int64_t* blob_off;     // [nctas * npanels + 1] byte offsets (multiples of 16)
  const int32_t* crow;         // [nctas * rmax] local row of A, -1: none
  int nctas, rmax;             // persistent CTAs (one per SM), row slots per CTA (multiple of 128)
  int npanels, width;          // panels of `width` columns (even)
  int64_t ncols;               // length of the gathered vector
  int stages;                  // shared-memory stages (panel + blob each)
  unsigned blob_max;           // largest blob (bytes)
};
size_t sweep_smem_bytes(const SweepArgs& sw);
// rowsum[row] = sum_k val * x[col] of every swept row, CSR order
cudaError_t launch_sweep(const double* x, double* rowsum, const SweepArgs& sw, cudaStream_t s);
cudaError_t launch_sweep_runs(const int64_t* rp, const int32_t* ci, const int32_t* crow, int ncta,
                              int R, int P, int W, int32_t* rstart, int32_t* rowlen,
                              cudaStream_t s);
cudaError_t launch_sweep_sort(const int32_t* rstart, const int32_t* rowlen, int ncta, int R, int P,
                              uint16_t* perm, uint16_t* srun, uint32_t* gbase, uint32_t* nepad,
                              cudaStream_t s);
cudaError_t launch_sweep_fill(const int64_t* rp, const int32_t* ci, const double* va,
                              const int32_t* crow, int ncta, int R, int P, int W,
                              const uint16_t* perm, const uint16_t* srun, const uint32_t* gbase,
                              const uint32_t* nepad, const int32_t* rstart, const int64_t* blob_off,
                              unsigned char* blobs, bool do_struct, bool do_vals, cudaStream_t s);

enum PassMode : int {
  kPassPlain = 0,    // y = acc
  kPassLsqrU = 1,    // out = s_i*acc - alpha*u_i   (s = d or 1)
  kPassLsqrV = 2,    // out = s_j*acc - beta*v_j    (s = e or 1)
  kPassResid = 3,    // out = b_i - acc
  kPassScaled = 4,   // out = s_i*acc (s = scale or 1)
  kPassEst = 5,      // out = (s_i*acc)^2 (row-norm estimate, s = scale)
};

struct PassArgs {
  const int64_t* rp;
  const int32_t* ci;
  const double* va;
  const int32_t* rl;    // slice row list
  const Tile* tiles;
  const double* xg;     // gathered vector (padded coords)
  double* out;          // local rows
  const double* scale;  // d or e (local rows) or nullptr
  const double* prev;   // u or v (local rows), or b for kPassResid
  const double* coef;   // device scalar (alpha or beta) or nullptr
  const int* skip;      // device flag: when nonzero the pass is a no-op
  int mode;
};

// LSQR device scalars
struct LsqrDev {
  double alpha, beta, rel;
  double rnorm2;
  int invariant;
  int pad;
};

// -------------------- launchers (kernels.cu) ------------------------------
void note_launches(long long n);
long long launch_count();
void count_launch(cudaStream_t s, int n = 1);  // skipped while s is capturing
// where: min over (class << 40 | entry), class 0 out of range, 1 duplicate,
// 2 columns not ascending; must be preset to ~0
cudaError_t launch_validate_csr(const DevCsr& A, int* err, unsigned long long* where,
                                cudaStream_t s);
// row pointers of A^T from A's column indices (column counts + scan), available
// before the transpose itself
cudaError_t launch_col_rowptr(const int32_t* col, int64_t nnz, int64_t cols, int64_t* rp,
                              cudaStream_t s);
// K2 (transpose.cu).  transpose_structure needs AT.row_ptr (launch_col_rowptr)
// and A's columns only: it writes AT.col and records the value permutations in
// w; transpose_values then moves the values (after they have arrived).
// transpose_csr = both (val_ready: event the value step waits on).
struct TransposeWork {
  int64_t nnz = 0;
  cudaStream_t stream = nullptr;
  int32_t* srcT = nullptr;  // source entry of every CSR(A^T) entry
  TransposeWork() = default;
  TransposeWork(const TransposeWork&) = delete;
  TransposeWork& operator=(const TransposeWork&) = delete;
  ~TransposeWork();
  void release();
};
// rpT_host: CSR(A^T)'s row pointers on the host (the partition plan);
// upload (optional): the host -> device copy to use for the plan
using HostUpload = std::function<void(void* dst, const void* src, size_t bytes)>;
cudaError_t transpose_structure(const DevCsr& A, DevCsr& AT, const int64_t* rpT_host,
                                TransposeWork& w, cudaStream_t s,
                                const HostUpload& upload = nullptr);
cudaError_t transpose_values(const DevCsr& A, DevCsr& AT, TransposeWork& w, cudaStream_t s);
cudaError_t transpose_csr(const DevCsr& A, DevCsr& AT, const int64_t* rpT_host, cudaStream_t s,
                          cudaEvent_t val_ready = nullptr);
// hand-written exclusive scan (transpose.cu); in == out allowed
template <class T>
cudaError_t exclusive_scan(const T* in, T* out, int64_t n, cudaStream_t s);
// ExplicitMatrix::sparse on device from COO (rows/cols int64, device); out
// arrays preallocated (row_ptr m+1, col/val nnz).  On a precondition failure
// *bad_kind = 1 (out of range: *bad = first entry index in input order) or
// 2 (duplicate: *bad = row * n + col of the first duplicate in sorted order).
cudaError_t coo_to_csr(int64_t m, int64_t n, int64_t nnz, const int64_t* rows,
                       const int64_t* cols, const double* vals, DevCsr& out,
                       unsigned long long* bad, int* bad_kind, cudaStream_t s);
cudaError_t launch_sgd_init(double* xs, double* xw, double* u, double* ub,
                            double* v, double* vb, int64_t n_pad_len,
                            int64_t m_pad_len, const uint32_t* signs,
                            int64_t m_loc, int64_t n_loc, int64_t a_goff,
                            int64_t at_goff, int64_t a_poff, int64_t at_poff,
                            int64_t m_glob, int64_t n_glob, const int32_t* wslot,
                            const int32_t* sslot, cudaStream_t s);
// hot-first slot map of the rows of a (global) matrix partitioned by bounds
// (G + 1 device values): map_pad[padded position of row i] = its slot, rows
// of each rank ordered by decreasing floor(log2(length)), stable
cudaError_t launch_slot_map(const int64_t* rp, int64_t rows, const int64_t* bounds, int G,
                            int64_t maxcnt, int32_t* map_pad, cudaStream_t s, bool flat = false);
// column-block boundaries of every row (block b = columns [b*width, (b+1)*width))
cudaError_t launch_block_bounds(const DevCsr& M, int nb, int64_t width, int32_t* bnd,
                                cudaStream_t s);
// dst[k] = map[src[k]] (column indices into a slot layout)
cudaError_t launch_remap_cols(int32_t* dst, const int32_t* src, const int32_t* map, int64_t nnz,
                              cudaStream_t s);
cudaError_t launch_sgd_iter(const SgdIterArgs& a, int ntiles, cudaStream_t s);
cudaError_t launch_sgd_iter_part(const SgdIterArgs& a, int tile_base, int ntiles, bool long_part,
                                 int minb, cudaStream_t s);
cudaError_t launch_exp(const double* x, double* y, int64_t n, double scale,
                       cudaStream_t s);
cudaError_t launch_pass(const PassArgs& a, int ntiles, cudaStream_t s);
// two passes over the same matrix (same tiles) in one traversal: a and b differ
// only in the gathered vector and the epilogue (LSQR: residual + next B v)
cudaError_t launch_pass_dual(const PassArgs& a, const PassArgs& b, int ntiles, cudaStream_t s);
// a pass over the interleaved slices listed in sa (one matrix; columns in
// padded coordinates): lng selects the warp-specialised long-slice kernel;
// b non-null: the dual pass
cudaError_t launch_sell_pass(const PassArgs& a, const PassArgs* b, const SellArgs& sa, bool lng,
                             bool pair,
                             cudaStream_t s);
// tiles [tile_base, tile_base + ntiles); b non-null: the dual pass
cudaError_t launch_pass_range(const PassArgs& a, const PassArgs* b, int tile_base, int ntiles,
                              cudaStream_t s);

// canonical reduction (det_math.cuh) of terms x*x (kind 0), x (kind 1) or
// coef*x (kind 2); *out (device) = result, or its sqrt when sqrt_out
// part_cap: capacity of partials (checked builds; < 0: unknown)
cudaError_t launch_canon_reduce(const double* x, int64_t len, int kind, double coef,
                                double* partials, unsigned* counter, double* out,
                                int sqrt_out, cudaStream_t s, int64_t part_cap = -1);

// signs: MT19937-64 device generation
cudaError_t sign_stream_generate(uint64_t seed, uint64_t stream, uint64_t total,
                                 uint32_t* bits, void* scratch,
                                 size_t scratch_bytes, cudaStream_t s);
size_t sign_stream_scratch_bytes(uint64_t total);

// dense
struct DenseIterArgs {
  const double* A;  // row-major m x n
  int64_t m, n;
  const double* xs_cur;
  const double* xw_cur;
  double* xs_next;
  double* xw_next;
  double* u;
  double* ub;
  double* v;
  double* vb;
  const uint32_t* signs;
  int64_t sign_next_w, sign_next_s;
  int has_next;
  SgdBlockConst cu, cv;
  const double* lin_u;  // per-coordinate linear terms or nullptr
  const double* lin_v;
  SgdStep st;
  unsigned* flags;
  double* colpart;   // scratch: nchunks_m x n
  unsigned* colcnt;  // per 16-column strip: chunk CTAs done (zero between launches)
};
// s2 non-null: the row and column halves run concurrently on s2 / s
cudaError_t launch_dense_sgd_iter(const DenseIterArgs& a, cudaStream_t s, cudaStream_t s2 = nullptr,
                                  cudaEvent_t ev_fork = nullptr, cudaEvent_t ev_join = nullptr);
struct DensePassArgs {
  const double* A;
  int64_t m, n;
  int adjoint;
  const double* xg;
  double* out;
  const double* scale;
  const double* prev;
  const double* coef;
  const int* skip;
  int mode;
  double* colpart;
  unsigned* colcnt;
};
cudaError_t launch_dense_pass(const DensePassArgs& a, cudaStream_t s);

// engine variants (variants.cu): symmetric / block equilibration
// scale_i = exp(x[map ? map[i] : i]); signed_out_i = +-scale_i by sign bit sign0 + i
cudaError_t launch_expand_scale(const double* x, const int32_t* map, int64_t len,
                                const uint32_t* signs, int64_t sign0, double* scale,
                                double* signed_out, cudaStream_t s);
// out[b] = sequential sum of est over members[off[b] .. off[b+1]) (ascending)
cudaError_t launch_block_sum(const double* est, const int32_t* members, const int64_t* off,
                             int64_t nblocks, double* out, cudaStream_t s);
// projected SGD update of len coordinates with per-coordinate linear terms
cudaError_t launch_sgd_update(double* x, double* avg, const double* est, const double* lin,
                              const SgdBlockConst& c, const SgdStep& st, int64_t len,
                              unsigned* flags, cudaStream_t s);
// out_i = x[map[i]]
cudaError_t launch_gather_map(const double* x, const int32_t* map, int64_t len, double* out,
                              cudaStream_t s);

// Chambolle-Pock lasso steps (variants.cu; src/ccp.cpp:73-88), d / e may be null (= 1)
cudaError_t launch_ccp_dual(double* y, const double* kz, const double* d, const double* b,
                            double sigma, double sqrt_lambda, int64_t m, double* dy,
                            cudaStream_t s);
cudaError_t launch_ccp_primal(double* z, double* ezt, const double* g, const double* e,
                              double tau, double tau_sl, double theta, int64_t n, double* x,
                              double* absx, cudaStream_t s);
cudaError_t launch_lasso_value(const double* r2, const double* l1, double sqrt_lambda,
                               double* out, cudaStream_t s);
cudaError_t launch_abs(const double* x, int64_t n, double* out, cudaStream_t s);
// g = est + (neg_lin + gamma x)  (stochastic_gradient_estimate, equilibrate.cpp:69-70)
cudaError_t launch_sge_finish(double* g, const double* x, double neg_lin, double gamma,
                              int64_t n, cudaStream_t s);
// g = g + (gamma x - lin)  (gradient_weighted, equilibrate.cpp:35-36); lin null: lin_c
cudaError_t launch_grad_finish(double* g, const double* x, const double* lin, double lin_c,
                               double gamma, int64_t n, cudaStream_t s);

// LSQR elementwise helpers
cudaError_t launch_lsqr_normalize(double* dst, const double* src,
                                  const double* norm_dev, double* scaled_out,
                                  const double* scale, int64_t len,
                                  int* invariant, int* skip_in,
                                  cudaStream_t s, int64_t ostride = 1,
                                  const int32_t* slot = nullptr);
// ostride: scaled_out / ex element stride (2: one half of an interleaved pair);
// slot (nullable): element k goes to position slot[k] (the hot-first slot
// layout of the gathered vectors, engine.cu build_slot_layout), else to k
cudaError_t launch_lsqr_xw_update(double* x, double* w, const double* v,
                                  double c1, double c2, const double* e,
                                  double* ex, int64_t n, cudaStream_t s, int64_t ostride = 1,
                                  const int32_t* slot = nullptr);
cudaError_t launch_rms_terms(int mat, const DevCsr& M, const double* eu,
                             const double* ev, double* out, int64_t goff,
                             double target, cudaStream_t s);

cudaError_t launch_obj_terms(const DevCsr& A, const double* u, const double* v,
                             double* out, cudaStream_t s);
cudaError_t launch_mul(double* out, const double* a, const double* b, int64_t n,
                       cudaStream_t s);

}  // namespace eqb
