// panel.cu -- column-panel SGD traversal (K3/K4, second generation).
//
// Why: the row-slice traversal in kernels.cu gathers xs[col] / xw[col] once
// per nonzero.  Those gathers hit L2 (the vectors are L2-resident) but each
// 8-byte gather moves a 32-byte sector, so the pass is bound by L2->SM sector
// throughput, not by HBM.  Here the gathered vector is instead read in
// contiguous panels of kPanelW coordinates with bulk copies into shared memory
// (cp.async.bulk, double-buffered on an mbarrier), and every gather is a
// shared-memory load.  The row sums of a band of <= kBandRows rows live in
// shared memory while the band's entries stream past panel by panel.
//
// Order of the arithmetic (src/explicit_matrix.cpp:70-78, and the ascending-row
// scatter :85-92 which CSR(A^T) turns into the same row form): row i's sum is
// acc = 0; acc = acc + val[k] * x[col[k]] for its entries in ascending column
// order.  The panel-major layout keeps every row's entries of a panel
// contiguous and in column order, and panels are visited in ascending order,
// so each row still receives exactly that chain: the running sum just waits in
// shared memory between panels.  Products are single rounded multiplies
// whoever computes them; the adds of one row are done by one thread in order.
//
// Per round (<= kPanelChunk entries of one panel), with the round's row runs
// (maximal stretches of one row) listed by the layout builder:
//   step 1, all threads: product = val * panel[col] into a staging buffer;
//   step 2, one thread per run: extend that row's running sum over the run's
//           products in order.
// Rounds are software-pipelined over two staging buffers: in one barrier
// interval the CTA stages round c+1 and chains round c, while the entries of
// round c+2 and the runs of round c+1 are already in flight into registers.
#include <algorithm>
#include <atomic>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "internal.h"
#include "sgd_common.cuh"

namespace eqb {
namespace {

constexpr int kPer = kPanelChunk / kPanelThreads;  // entries (and runs) per thread per round
static_assert(kPanelChunk % kPanelThreads == 0 && kPanelThreads % 32 == 0, "round shape");

struct PanelSmem {
  double xp[2][kPanelW];           // panel of the gathered vector (double buffer)
  double acc[kBandRows];           // running row sums of the band
  double stage[2][kPanelChunk];    // products of two consecutive rounds
  PanelChunk desc[4];              // descriptors of rounds c .. c+3 (ring)
  unsigned long long bar[2];       // bulk-copy completion, one per panel buffer
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// one thread: panel `panel` of xg -> dst, completion signalled on bar
__device__ __forceinline__ void load_panel(double* dst, const double* xg, int panel,
                                           unsigned long long* bar) {
  constexpr unsigned kBytes = kPanelW * sizeof(double);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(kBytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(xg + static_cast<int64_t>(panel) * kPanelW), "r"(kBytes), "r"(smem_addr(bar))
      : "memory");
}

__global__ void __launch_bounds__(kPanelThreads, 1)
sgd_panel_kernel(const SgdIterArgs a, const PanelArgs p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  PanelSmem& S = *reinterpret_cast<PanelSmem*>(smem_raw);
  const PanelBand B = p.bands[blockIdx.x];
  const int mat = B.mat;
  const double* __restrict__ xg = mat ? a.xw_cur : a.xs_cur;
  const PanelChunk* __restrict__ ch = p.chunks[mat];
  const double* __restrict__ pv = p.val[mat];
  const uint16_t* __restrict__ pc = p.col[mat];
  const uint32_t* __restrict__ pr = p.runs[mat];
  const int tid = threadIdx.x, lane = tid & 31;
  const int c0 = B.c0, c1 = B.c1;

  for (int r = tid; r < B.rows; r += kPanelThreads) S.acc[r] = 0.0;  // acc = 0.0
  if (tid == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < 3 && c0 + q < c1; ++q) S.desc[q] = ch[c0 + q];
    if (c0 < c1) load_panel(S.xp[0], xg, S.desc[0].panel, &S.bar[0]);
  }
  __syncthreads();

  double ev[kPer];
  uint16_t ec[kPer];
  uint32_t rn[kPer], rnl[kPer];  // runs in flight (+ lane 31's successor run)
  auto fetch_entries = [&](const PanelChunk& d) {
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      if (u * kPanelThreads >= d.len) break;  // uniform: rounds are often part-full
      const int k = tid + u * kPanelThreads;
      if (k < d.len) {
        ev[u] = ld_na(pv + d.e0 + k);
        ec[u] = ld_na(pc + d.e0 + k);
      }
    }
  };
  auto fetch_runs = [&](const PanelChunk& d) {
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      if (j * kPanelThreads >= d.nruns) break;
      const int q = tid + j * kPanelThreads;
      rn[j] = q < d.nruns ? ld_na(pr + d.q0 + q) : 0u;
      rnl[j] = (lane == 31 && q + 1 < d.nruns) ? ld_na(pr + d.q0 + q + 1) : 0u;
    }
  };
  int xb = 1, panel = -1;
  unsigned phase = 0u;  // bit b: parity of the next completion of panel buffer b
  auto stage = [&](const PanelChunk& d, double* __restrict__ st) {
    if (d.panel != panel) {
      xb ^= 1;
      panel = d.panel;
      mbar_wait(&S.bar[xb], (phase >> xb) & 1u);
      phase ^= 1u << xb;
      // the other buffer was last read before the previous barrier: prefetch
      // the band's next panel into it
      if (tid == 0 && d.next_panel >= 0)
        load_panel(S.xp[xb ^ 1], xg, d.next_panel, &S.bar[xb ^ 1]);
    }
    const double* __restrict__ X = S.xp[xb];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      if (u * kPanelThreads >= d.len) break;
      const int k = tid + u * kPanelThreads;
      if (k < d.len) st[k] = __dmul_rn(ev[u], X[ec[u]]);
    }
  };

  if (c0 < c1) {
    fetch_entries(S.desc[0]);
    fetch_runs(S.desc[0]);
    stage(S.desc[0], S.stage[0]);
    if (c0 + 1 < c1) fetch_entries(S.desc[1]);
    __syncthreads();
  }
  for (int c = c0; c < c1; ++c) {
    const int sb = (c - c0) & 1, slot = (c - c0) & 3;
    uint32_t rc[kPer], rcl[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      rc[j] = rn[j];
      rcl[j] = rnl[j];
    }
    if (tid == 0 && c + 3 < c1) S.desc[(slot + 3) & 3] = ch[c + 3];
    if (c + 1 < c1) {
      const PanelChunk& d1 = S.desc[(slot + 1) & 3];
      stage(d1, S.stage[sb ^ 1]);  // round c+1: products
      fetch_runs(d1);
      if (c + 2 < c1) fetch_entries(S.desc[(slot + 2) & 3]);
    }
    // round c: one thread per run extends the run's row sum in order
    const double* __restrict__ st = S.stage[sb];
    const int len = S.desc[slot].len, nr = S.desc[slot].nruns;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      if (j * kPanelThreads >= nr) break;
      const int q = tid + j * kPanelThreads;
      uint32_t nx = __shfl_down_sync(0xffffffffu, rc[j], 1);
      if (lane == 31) nx = rcl[j];
      if (q < nr) {
        const int r = static_cast<int>(rc[j] & 0xffffu);
        int k = static_cast<int>(rc[j] >> 16);
        const int e = q + 1 < nr ? static_cast<int>(nx >> 16) : len;
        double acc = S.acc[r];
        for (; k + 4 <= e; k += 4) {
          const double t0 = st[k], t1 = st[k + 1], t2 = st[k + 2], t3 = st[k + 3];
          acc = __dadd_rn(acc, t0);
          acc = __dadd_rn(acc, t1);
          acc = __dadd_rn(acc, t2);
          acc = __dadd_rn(acc, t3);
        }
        for (; k < e; ++k) acc = __dadd_rn(acc, st[k]);
        S.acc[r] = acc;
      }
    }
    __syncthreads();
  }
  // ---- fused epilogue (equilibrate.cpp:106-129) for every row of the band
  unsigned fl = 0;
  for (int r = tid; r < B.rows; r += kPanelThreads)
    sgd_epilogue(a, mat, static_cast<int64_t>(B.r0) + r, S.acc[r], fl);
  if (fl) atomicOr(a.flags, fl);
}

// ---------------------------------------------------------------------------
// layout builder
// ---------------------------------------------------------------------------
constexpr int kLogW = __builtin_ctz(kPanelW);

__global__ void band_of_row_kernel(const int64_t* __restrict__ band_r0,
                                   int32_t* __restrict__ row_band) {
  const int b = blockIdx.x;
  for (int64_t r = band_r0[b] + threadIdx.x; r < band_r0[b + 1]; r += blockDim.x)
    row_band[r] = b;
}

// warp per row: key = band * P + panel, band-local row of every entry
__global__ void panel_keys_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                  int64_t rows, const int32_t* __restrict__ row_band,
                                  const int64_t* __restrict__ band_r0, int64_t P,
                                  uint32_t* __restrict__ key, uint16_t* __restrict__ rloc) {
  const int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= rows) return;
  const int b = row_band[i];
  const uint16_t rl = static_cast<uint16_t>(i - band_r0[b]);
  const uint32_t kb = static_cast<uint32_t>(b * P);
  for (int64_t k = rp[i] + lane; k < rp[i + 1]; k += 32) {
    key[k] = kb + static_cast<uint32_t>(col[k] >> kLogW);
    rloc[k] = rl;
  }
}

__global__ void iota32_kernel(int32_t* v, int64_t n) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < n) v[k] = static_cast<int32_t>(k);
}

__global__ void panel_gather_kernel(const int32_t* __restrict__ perm,
                                    const double* __restrict__ val,
                                    const int32_t* __restrict__ col,
                                    const uint16_t* __restrict__ rloc, int64_t nnz,
                                    double* __restrict__ pv, uint16_t* __restrict__ pc,
                                    uint16_t* __restrict__ srl) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q >= nnz) return;
  const int64_t k = perm[q];
  pv[q] = val[k];
  pc[q] = static_cast<uint16_t>(col[k] & (kPanelW - 1));
  srl[q] = rloc[k];
}

__global__ void seg_bounds_kernel(const uint32_t* __restrict__ skey, int64_t nnz,
                                  int64_t* __restrict__ lo, int64_t* __restrict__ hi) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q >= nnz) return;
  const uint32_t k = skey[q];
  if (q == 0 || skey[q - 1] != k) lo[k] = q;
  if (q == nnz - 1 || skey[q + 1] != k) hi[k] = q + 1;
}

__global__ void seg_rounds_kernel(const int64_t* __restrict__ lo, const int64_t* __restrict__ hi,
                                  int64_t K, int64_t* __restrict__ cnt) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < K) cnt[k] = (hi[k] - lo[k] + kPanelChunk - 1) / kPanelChunk;
  if (k == K) cnt[k] = 0;
}

// entry q starts a run when it starts a round or its row differs from q-1's
__global__ void run_flags_kernel(const uint32_t* __restrict__ skey,
                                 const int64_t* __restrict__ lo,
                                 const uint16_t* __restrict__ srl, int64_t nnz,
                                 int32_t* __restrict__ flag) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q > nnz) return;
  if (q == nnz) {
    flag[q] = 0;
    return;
  }
  const int64_t pos = q - lo[skey[q]];
  flag[q] = (pos % kPanelChunk == 0 || srl[q] != srl[q - 1]) ? 1 : 0;
}

__global__ void run_write_kernel(const uint32_t* __restrict__ skey,
                                 const int64_t* __restrict__ lo,
                                 const uint16_t* __restrict__ srl,
                                 const int32_t* __restrict__ ridx, int64_t nnz,
                                 uint32_t* __restrict__ runs) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q >= nnz || ridx[q + 1] == ridx[q]) return;
  const uint32_t pos = static_cast<uint32_t>((q - lo[skey[q]]) % kPanelChunk);
  runs[ridx[q]] = (pos << 16) | srl[q];
}

__global__ void chunk_fill_kernel(const int64_t* __restrict__ lo, const int64_t* __restrict__ hi,
                                  const int64_t* __restrict__ off, const int32_t* __restrict__ ridx,
                                  int64_t K, int64_t P, PanelChunk* __restrict__ ch) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= K) return;
  const int64_t n = off[k + 1] - off[k];
  for (int64_t q = 0; q < n; ++q) {
    PanelChunk c;
    c.e0 = lo[k] + q * kPanelChunk;
    const int64_t rem = hi[k] - c.e0;
    c.len = static_cast<int32_t>(rem < kPanelChunk ? rem : kPanelChunk);
    c.q0 = ridx[c.e0];
    c.nruns = ridx[c.e0 + c.len] - c.q0;
    c.panel = static_cast<int32_t>(k % P);
    c.next_panel = -1;
    c.band = static_cast<int32_t>(k / P);
    ch[off[k] + q] = c;
  }
}

__global__ void chunk_next_kernel(PanelChunk* __restrict__ ch, int64_t nch,
                                  const int64_t* __restrict__ off, int64_t P) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= nch) return;
  const int32_t band = ch[c].band, panel = ch[c].panel;
  const int64_t end = off[(band + 1) * P];
  int64_t j = c + 1;
  while (j < end && ch[j].panel == panel) ++j;
  ch[c].next_panel = j < end ? ch[j].panel : -1;
}

__global__ void band_chunks_kernel(const int64_t* __restrict__ off, int nbands, int64_t P,
                                   int64_t* __restrict__ band_c) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b <= nbands) band_c[b] = off[b * P];
}

unsigned blocks(int64_t n, int t = 256) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

cudaError_t build_panels(const DevCsr& M, int64_t vec_len, const std::vector<int64_t>& band_r0,
                         double* out_val, uint16_t* out_col, uint32_t** runs, int64_t* nruns,
                         PanelChunk** chunks, int64_t* nchunks, std::vector<int64_t>* band_c,
                         cudaStream_t s) {
  const int nb = static_cast<int>(band_r0.size()) - 1;
  const int64_t nnz = M.nnz;
  const int64_t P = std::max<int64_t>(1, (vec_len + kPanelW - 1) / kPanelW);
  const int64_t K = static_cast<int64_t>(nb) * P;
  *chunks = nullptr;
  *runs = nullptr;
  *nchunks = 0;
  *nruns = 0;
  band_c->assign(nb + 1, 0);
  if (nb <= 0 || nnz >= (1LL << 31) - 1 || K >= (1LL << 32)) return cudaErrorInvalidValue;
  int bits = 1;
  while (bits < 32 && (1LL << bits) < K) ++bits;
  int64_t *br = nullptr, *lo = nullptr, *hi = nullptr, *off = nullptr, *bc = nullptr;
  int32_t *rb = nullptr, *perm0 = nullptr, *perm1 = nullptr, *ridx = nullptr;
  uint32_t *key0 = nullptr, *key1 = nullptr;
  uint16_t *rloc = nullptr, *srl = nullptr;
  void* temp = nullptr;
  size_t tb = 0, tb2 = 0, tb3 = 0;
  const int64_t nn = std::max<int64_t>(1, nnz);
  cudaError_t e = cudaSuccess;
  do {
    e = cudaMallocAsync(&br, (nb + 1) * 8, s); if (e) break;
    e = cudaMemcpyAsync(br, band_r0.data(), (nb + 1) * 8, cudaMemcpyHostToDevice, s); if (e) break;
    e = cudaMallocAsync(&lo, K * 8, s); if (e) break;
    e = cudaMallocAsync(&hi, K * 8, s); if (e) break;
    e = cudaMallocAsync(&off, (K + 1) * 8, s); if (e) break;
    e = cudaMallocAsync(&bc, (nb + 1) * 8, s); if (e) break;
    e = cudaMemsetAsync(lo, 0, K * 8, s); if (e) break;
    e = cudaMemsetAsync(hi, 0, K * 8, s); if (e) break;
    e = cudaMallocAsync(&rb, std::max<int64_t>(1, M.rows) * 4, s); if (e) break;
    e = cudaMallocAsync(&perm0, nn * 4, s); if (e) break;
    e = cudaMallocAsync(&perm1, nn * 4, s); if (e) break;
    e = cudaMallocAsync(&key0, nn * 4, s); if (e) break;
    e = cudaMallocAsync(&key1, nn * 4, s); if (e) break;
    e = cudaMallocAsync(&rloc, nn * 2, s); if (e) break;
    e = cudaMallocAsync(&srl, nn * 2, s); if (e) break;
    e = cudaMallocAsync(&ridx, (nnz + 1) * 4, s); if (e) break;
    e = cub::DeviceRadixSort::SortPairs(nullptr, tb, key0, key1, perm0, perm1, nn, 0, bits, s);
    if (e) break;
    e = cub::DeviceScan::ExclusiveSum(nullptr, tb2, off, off, K + 1, s); if (e) break;
    e = cub::DeviceScan::ExclusiveSum(nullptr, tb3, ridx, ridx, nnz + 1, s); if (e) break;
    tb = std::max(tb, std::max(tb2, tb3));
    e = cudaMallocAsync(&temp, tb, s); if (e) break;
    band_of_row_kernel<<<nb, 256, 0, s>>>(br, rb);
    count_launch(s);
    if (nnz > 0) {
      panel_keys_kernel<<<blocks(M.rows * 32), 256, 0, s>>>(M.row_ptr, M.col, M.rows, rb, br, P,
                                                            key0, rloc);
      iota32_kernel<<<blocks(nnz), 256, 0, s>>>(perm0, nnz);
      count_launch(s, 2);
      e = cudaGetLastError(); if (e) break;
      // stable: within one (band, panel) key the CSR order (row, column) stays
      size_t t = tb;
      e = cub::DeviceRadixSort::SortPairs(temp, t, key0, key1, perm0, perm1, nnz, 0, bits, s);
      if (e) break;
      panel_gather_kernel<<<blocks(nnz), 256, 0, s>>>(perm1, M.val, M.col, rloc, nnz, out_val,
                                                      out_col, srl);
      seg_bounds_kernel<<<blocks(nnz), 256, 0, s>>>(key1, nnz, lo, hi);
      count_launch(s, 2);
    }
    run_flags_kernel<<<blocks(nnz + 1), 256, 0, s>>>(key1, lo, srl, nnz, ridx);
    seg_rounds_kernel<<<blocks(K + 1), 256, 0, s>>>(lo, hi, K, off);
    count_launch(s, 2);
    e = cudaGetLastError(); if (e) break;
    size_t t2 = tb;
    e = cub::DeviceScan::ExclusiveSum(temp, t2, ridx, ridx, nnz + 1, s); if (e) break;
    t2 = tb;
    e = cub::DeviceScan::ExclusiveSum(temp, t2, off, off, K + 1, s); if (e) break;
    int64_t total = 0;
    int32_t total_runs = 0;
    e = cudaMemcpyAsync(&total, off + K, 8, cudaMemcpyDeviceToHost, s); if (e) break;
    e = cudaMemcpyAsync(&total_runs, ridx + nnz, 4, cudaMemcpyDeviceToHost, s); if (e) break;
    e = cudaStreamSynchronize(s); if (e) break;
    e = cudaMalloc(chunks, std::max<int64_t>(1, total) * sizeof(PanelChunk)); if (e) break;
    e = cudaMalloc(runs, std::max<int64_t>(1, total_runs) * sizeof(uint32_t)); if (e) break;
    *nchunks = total;
    *nruns = total_runs;
    if (nnz > 0) {
      run_write_kernel<<<blocks(nnz), 256, 0, s>>>(key1, lo, srl, ridx, nnz, *runs);
      count_launch(s);
    }
    if (total > 0) {
      chunk_fill_kernel<<<blocks(K), 256, 0, s>>>(lo, hi, off, ridx, K, P, *chunks);
      chunk_next_kernel<<<blocks(total), 256, 0, s>>>(*chunks, total, off, P);
      count_launch(s, 2);
    }
    band_chunks_kernel<<<blocks(nb + 1), 256, 0, s>>>(off, nb, P, bc);
    count_launch(s);
    e = cudaGetLastError(); if (e) break;
    e = cudaMemcpyAsync(band_c->data(), bc, (nb + 1) * 8, cudaMemcpyDeviceToHost, s); if (e) break;
    e = cudaStreamSynchronize(s);
  } while (0);
  for (void* q : {static_cast<void*>(br), static_cast<void*>(lo), static_cast<void*>(hi),
                  static_cast<void*>(off), static_cast<void*>(bc), static_cast<void*>(rb),
                  static_cast<void*>(perm0), static_cast<void*>(perm1), static_cast<void*>(key0),
                  static_cast<void*>(key1), static_cast<void*>(rloc), static_cast<void*>(srl),
                  static_cast<void*>(ridx), temp})
    if (q) cudaFreeAsync(q, s);
  if (e) {
    if (*chunks) cudaFree(*chunks);
    if (*runs) cudaFree(*runs);
    *chunks = nullptr;
    *runs = nullptr;
  }
  return e;
}

cudaError_t launch_sgd_panel(const SgdIterArgs& a, const PanelArgs& p, int nbands,
                             cudaStream_t s) {
  if (nbands == 0) return cudaSuccess;
  // the attribute is per device; setting it is idempotent, so racing threads
  // at worst set it twice
  static std::atomic<bool> attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_set[dev].load(std::memory_order_acquire)) {
    const cudaError_t e = cudaFuncSetAttribute(
        sgd_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
        static_cast<int>(sizeof(PanelSmem)));
    if (e != cudaSuccess) return e;
    attr_set[dev].store(true, std::memory_order_release);
  }
  sgd_panel_kernel<<<nbands, kPanelThreads, sizeof(PanelSmem), s>>>(a, p);
  count_launch(s);
  return cudaGetLastError();
}

}  // namespace eqb
