// dsmem_bench.cu -- random fp64 gathers: L2/L1 (__ldg) vs thread-block-cluster
// distributed shared memory (mapa + ld.shared::cluster) vs CTA-local shared
// memory.  Answers VERDICT r1 task 3(a): would serving the SGD pass's gathers
// from a cluster's DSMEM (16 CTAs x ~200 KB = 3.2 MB per column block) beat the
// ~250 G gathers/s measured from L2?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dsmem_bench tools/dsmem_bench.cu
//
// Every variant streams the same 12 B/entry (int32 index + fp64 value) and
// forms sum(val * x[idx]); only where x lives changes.
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__global__ void fill_idx(int* idx, int64_t n, int range, uint64_t seed) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  uint64_t z = (k + 1) * 0x9E3779B97F4A7C15ULL ^ seed;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z ^= z >> 31;
  idx[k] = (int)(z % range);
}

// x in global memory (L2 / L1 resident when small)
__global__ void __launch_bounds__(512) gather_l2(const int* __restrict__ idx,
                                                 const double* __restrict__ x,
                                                 const double* __restrict__ val, int64_t n,
                                                 double* out) {
  double acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; k + 3 * stride < n; k += 4 * stride) {
    int c[4];
    double v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j] = __ldcs(idx + k + j * stride);
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = __ldcs(val + k + j * stride);
#pragma unroll
    for (int j = 0; j < 4; ++j) acc += v[j] * __ldg(x + c[j]);
  }
  for (; k < n; k += stride) acc += __ldcs(val + k) * __ldg(x + __ldcs(idx + k));
  if (acc == 12345.678) out[0] = acc;
}

// x split over the cluster's CTAs: CTA r holds x[r * per, (r + 1) * per) in its
// shared memory; a gather maps the owner's copy (mapa) and loads it over DSMEM
template <int CS>
__global__ void __launch_bounds__(512) gather_dsmem(const int* __restrict__ idx,
                                                    const double* __restrict__ x,
                                                    const double* __restrict__ val, int64_t n,
                                                    int per, double* out) {
  extern __shared__ double part[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  for (int i = threadIdx.x; i < per; i += blockDim.x) part[i] = x[rank * per + i];
  cl.sync();
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(part));
  double acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; k + 3 * stride < n; k += 4 * stride) {
    int c[4];
    double v[4], g[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j] = __ldcs(idx + k + j * stride);
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = __ldcs(val + k + j * stride);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const unsigned owner = static_cast<unsigned>(c[j]) / per;
      const uint32_t loc = base + 8u * (static_cast<unsigned>(c[j]) - owner * per);
      uint32_t rem;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rem) : "r"(loc), "r"(owner));
      asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(g[j]) : "r"(rem));
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) acc += v[j] * g[j];
  }
  cl.sync();
  if (acc == 12345.678) out[0] = acc;
}

// x entirely in this CTA's shared memory (range <= per)
__global__ void __launch_bounds__(512) gather_smem(const int* __restrict__ idx,
                                                   const double* __restrict__ x,
                                                   const double* __restrict__ val, int64_t n,
                                                   int per, double* out) {
  extern __shared__ double part[];
  for (int i = threadIdx.x; i < per; i += blockDim.x) part[i] = x[i];
  __syncthreads();
  double acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; k + 3 * stride < n; k += 4 * stride) {
    int c[4];
    double v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j] = __ldcs(idx + k + j * stride);
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = __ldcs(val + k + j * stride);
#pragma unroll
    for (int j = 0; j < 4; ++j) acc += v[j] * part[c[j]];
  }
  if (acc == 12345.678) out[0] = acc;
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("  CUDA error: %s\n", cudaGetErrorString(e));
  return ms / 5;
}

template <int CS>
void run_dsmem(const int* idx, const double* x, const double* val, int64_t n, double* out,
               int per) {
  auto kern = gather_dsmem<CS>;
  const size_t smem = static_cast<size_t>(per) * 8;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (CS > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  int ncl = 0;
  cfg.gridDim = dim3(CS);
  cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
  cudaGetLastError();
  if (ncl <= 0) {
    printf("cluster %2d x %6.1f KB: cannot be resident\n", CS, smem / 1024.0);
    return;
  }
  cfg.gridDim = dim3(CS * ncl);
  const float t = timeit([&] { cudaLaunchKernelEx(&cfg, kern, idx, x, val, n, per, out); });
  printf("DSMEM cluster %2d x %6.1f KB (%5.2f MB, %d clusters resident): %.3f ms  %.1f G gathers/s\n",
         CS, smem / 1024.0, CS * smem / 1e6, ncl, t, n / t / 1e6);
}

int main() {
  const int64_t n = 150000000;
  int* idx;
  double *x, *val, *out;
  cudaMalloc(&idx, n * 4);
  cudaMalloc(&val, n * 8);
  cudaMalloc(&out, 8);
  cudaMalloc(&x, 2000000 * 8);
  cudaMemset(val, 0, n * 8);
  cudaMemset(x, 0, 2000000 * 8);
  const int per16 = 24 * 1024;  // 192 KB per CTA
  for (int range : {1000000, 2000000, 16 * per16, 8 * per16, per16}) {
    fill_idx<<<(n + 255) / 256, 256>>>(idx, n, range, 7);
    const float t = timeit([&] { gather_l2<<<148 * 4, 512>>>(idx, x, val, n, out); });
    printf("global x, range %8d (%6.2f MB): %.3f ms  %.1f G gathers/s  (stream %.2f TB/s)\n",
           range, range * 8 / 1e6, t, n / t / 1e6, n * 12.0 / t / 1e9);
    if (range == 16 * per16) run_dsmem<16>(idx, x, val, n, out, per16);
    if (range == 8 * per16) run_dsmem<8>(idx, x, val, n, out, per16);
    if (range == per16) {
      cudaFuncSetAttribute(gather_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, per16 * 8);
      const float ts = timeit(
          [&] { gather_smem<<<148, 512, per16 * 8>>>(idx, x, val, n, per16, out); });
      printf("CTA-local smem x (%d doubles): %.3f ms  %.1f G gathers/s\n", per16, ts,
             n / ts / 1e6);
    }
  }
  return 0;
}
