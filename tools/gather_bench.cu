// gather_bench.cu -- random fp64 gather throughput on B200 by load flavour.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_bench tools/gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__device__ __forceinline__ double ld(const double* p) {
  double v;
  if (MODE == 0) v = __ldg(p);
  else if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else if (MODE == 2) v = __ldcg(p);
  else {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(v) : "l"(p), "l"(pol));
  }
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(256) gather(const int* __restrict__ idx, const double* __restrict__ x,
                                              const double* __restrict__ val, int64_t n,
                                              double* out) {
  double acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; k + 3 * stride < n; k += 4 * stride) {
    int c0 = __ldcs(idx + k), c1 = __ldcs(idx + k + stride), c2 = __ldcs(idx + k + 2 * stride),
        c3 = __ldcs(idx + k + 3 * stride);
    double v0 = __ldcs(val + k), v1 = __ldcs(val + k + stride), v2 = __ldcs(val + k + 2 * stride),
           v3 = __ldcs(val + k + 3 * stride);
    acc += v0 * ld<MODE>(x + c0) + v1 * ld<MODE>(x + c1) + v2 * ld<MODE>(x + c2) + v3 * ld<MODE>(x + c3);
  }
  for (; k < n; k += stride) acc += __ldcs(val + k) * ld<MODE>(x + __ldcs(idx + k));
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

template <int MODE>
float run(const int* idx, const double* x, const double* val, int64_t n, double* out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather<MODE><<<148 * 8, 256>>>(idx, x, val, n, out);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) gather<MODE><<<148 * 8, 256>>>(idx, x, val, n, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  const int64_t n = 150000000;
  int* idx;
  double *x, *val, *out;
  cudaMalloc(&idx, n * 4);
  cudaMalloc(&val, n * 8);
  cudaMalloc(&out, 8);
  cudaMemset(val, 0, n * 8);
  for (int range : {1000000, 2000000, 16000, 100000000}) {
    cudaMalloc(&x, (size_t)range * 8);
    cudaMemset(x, 0, (size_t)range * 8);
    fill_idx<<<(n + 255) / 256, 256>>>(idx, n, range, 7);
    float t0 = run<0>(idx, x, val, n, out), t1 = run<1>(idx, x, val, n, out),
          t2 = run<2>(idx, x, val, n, out), t3 = run<3>(idx, x, val, n, out);
    printf("range %9d (%6.1f MB): ldg %.3f ms  nc.no_alloc %.3f  ldcg %.3f  ef/el %.3f  "
           "(Ggathers/s ldg %.1f; streamed %.2f TB/s)\n",
           range, range * 8 / 1e6, t0, t1, t2, t3, n / t0 / 1e6, n * 12.0 / t0 / 1e9);
    cudaFree(x);
  }
  return 0;
}
