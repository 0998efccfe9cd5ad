// tma_gather_bench.cu -- can the TMA unit's 2-D gather (cp.async.bulk.tensor
// .tile::gather4: four arbitrary 16-byte rows per instruction, straight from L2
// into shared memory, no LSU / L1TEX tag stage) beat the LSU gather rate that
// bounds the SGD traversals (~260 G random 8-byte gathers/s through L1TEX)?
//
// x (range doubles) is a 2-D tensor {4, range/4}: row r = x[4r .. 4r+3] (one
// 32-byte L2 sector; a gather4 destination must be 128-byte aligned).  Each
// CTA: warp 0 = producers (every lane issues G4 gather4s per stage into a ring
// of D stages, one mbarrier per stage with the stage's transaction bytes),
// warps 1..3 = consumers (sum the stage, release it).  Reports gathered rows/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_gather_bench tools/tma_gather_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t sa(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void wait(unsigned long long* b, unsigned par) {
  unsigned done;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(sa(b)), "r"(par) : "memory");
  } while (!done);
}

template <int G4, int D, int PW>
__global__ void __launch_bounds__(32 * (PW + 1)) tma_gather(const __grid_constant__ CUtensorMap tm,
                                                  const int* __restrict__ idx, int64_t per_cta,
                                                  double* out) {
  constexpr int ROWS = 32 * G4 * 4;  // rows per stage
  __shared__ __align__(128) double buf[D][ROWS * 4];
  __shared__ __align__(8) unsigned long long full[D], empty[D];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < D) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&full[threadIdx.x])), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[threadIdx.x])), "r"(32));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int stages = static_cast<int>(per_cta / ROWS);
  const int* my = idx + blockIdx.x * per_cta;
  if (warp < PW) {  // producer warp `warp` fills stages warp, warp + PW, ...
    for (int s = warp; s < stages; s += PW) {
      const int st = s % D;
      if (s >= D) wait(&empty[st], ((s / D) - 1) & 1);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[st])),
                     "r"(ROWS * 32) : "memory");
      __syncwarp();
#pragma unroll
      for (int g = 0; g < G4; ++g) {
        const int4 r = *reinterpret_cast<const int4*>(my + s * ROWS + (g * 32 + lane) * 4);
        double* dst = &buf[st][(g * 32 + lane) * 16];
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sa(dst)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w),
            "r"(sa(&full[st]))
            : "memory");
      }
    }
    return;
  }
  double acc = 0.0;
  for (int s = 0; s < stages; ++s) {
    const int st = s % D;
    wait(&full[st], (s / D) & 1);
    for (int k = lane; k < ROWS; k += 32) acc += buf[st][4 * k];
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[st])) : "memory");
  }
  if (acc == 12345.678) out[0] = acc;
}

// LSU baseline: 8-byte gathers of the same row indices (element 2r)
__global__ void __launch_bounds__(256) lsu_gather(const int* __restrict__ idx, const double* __restrict__ x,
                                                  int64_t n, double* out) {
  double acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += stride)
    acc += __ldg(x + 4 * (int64_t)__ldcs(idx + k));
  if (acc == 12345.678) out[0] = acc;
}

__global__ void fill_idx(int* idx, int64_t n, int range, uint64_t seed) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  uint64_t z = (k + 1) * 0x9E3779B97F4A7C15ULL ^ seed;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z ^= z >> 31;
  idx[k] = (int)(z % range);
}

template <int G4, int D, int PW>
void run_tma(const CUtensorMap& tm, const int* idx, int64_t n, int ctas, double* out, const char* tag) {
  constexpr int ROWS = 32 * G4 * 4;
  const int64_t per = (n / ctas) / ROWS * ROWS;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  tma_gather<G4, D, PW><<<ctas, 32 * (PW + 1)>>>(tm, idx, per, out);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) tma_gather<G4, D, PW><<<ctas, 32 * (PW + 1)>>>(tm, idx, per, out);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  printf("tma gather4 %-4s G4=%d D=%d PW=%d ctas=%5d: %.3f ms  %.1f G rows/s  (%s)\n", tag, G4, D, PW, ctas, ms,
         per * ctas / ms / 1e6, cudaGetErrorString(e));
}

int main() {
  const int64_t n = 100000000;
  int* idx;
  double* out;
  cudaMalloc(&idx, n * 4);
  cudaMalloc(&out, 8);
  EncodeTiled enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  if (!enc) {
    printf("no cuTensorMapEncodeTiled\n");
    return 1;
  }
  // concurrency: LSU gathers (stream a) and TMA gather4 (stream b) at the same
  // time -- does the TMA unit add gather capacity beside the LSU / L1TEX path?
  auto concurrent = [&](const CUtensorMap& tm, const double* x, int lsu_ctas, int tma_ctas) {
    cudaStream_t sa, sb;
    cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking);
    constexpr int ROWS = 32 * 1 * 4;
    const int64_t per = (n / tma_ctas) / ROWS * ROWS;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(a, 0);
      cudaStreamWaitEvent(sa, a, 0);
      cudaStreamWaitEvent(sb, a, 0);
      lsu_gather<<<lsu_ctas, 256, 0, sa>>>(idx, x, n, out);
      if (tma_ctas) tma_gather<1, 4, 3><<<tma_ctas, 128, 0, sb>>>(tm, idx, per, out);
      cudaEvent_t ea, eb;
      cudaEventCreate(&ea);
      cudaEventCreate(&eb);
      cudaEventRecord(ea, sa);
      cudaEventRecord(eb, sb);
      cudaStreamWaitEvent(0, ea, 0);
      cudaStreamWaitEvent(0, eb, 0);
      cudaEventRecord(b, 0);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double tot = static_cast<double>(n) + (tma_ctas ? static_cast<double>(per) * tma_ctas : 0.0);
      if (rep == 1)
        printf("concurrent lsu ctas %5d + tma ctas %5d: %.3f ms for %.0fM + %.0fM gathers = %.1f G/s total\n",
               lsu_ctas, tma_ctas, ms, n / 1e6, tma_ctas ? per * tma_ctas / 1e6 : 0.0, tot / ms / 1e6);
    }
  };
  for (int range : {1000000, 2000000}) {  // doubles (8 / 16 MB)
    double* x;
    cudaMalloc(&x, (size_t)range * 8);
    cudaMemset(x, 0, (size_t)range * 8);
    fill_idx<<<(n + 255) / 256, 256>>>(idx, n, range / 4, 7);
    CUtensorMap tm;
    const cuuint64_t dims[2] = {4, (cuuint64_t)range / 4};
    const cuuint64_t strides[1] = {32};
    const cuuint32_t box[2] = {4, 1}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode failed %d\n", (int)r);
      return 1;
    }
    printf("range %d doubles (%.1f MB)\n", range, range * 8 / 1e6);
    {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      lsu_gather<<<148 * 8, 256>>>(idx, x, n, out);
      cudaEventRecord(a);
      for (int k = 0; k < 5; ++k) lsu_gather<<<148 * 8, 256>>>(idx, x, n, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("lsu ldg 8B gathers (one per 32-byte row): %.3f ms  %.1f G/s\n", ms / 5, n / (ms / 5) / 1e6);
    }
    run_tma<1, 4, 3>(tm, idx, n, 148 * 12, out, "");
    concurrent(tm, x, 148 * 8, 0);
    concurrent(tm, x, 148 * 4, 148 * 8);
    concurrent(tm, x, 148 * 6, 148 * 6);
    concurrent(tm, x, 148 * 8, 148 * 4);
    cudaFree(x);
  }
  return 0;
}
