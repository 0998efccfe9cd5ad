// l2_bw_bench.cu -- L2 -> SM read bandwidth on B200: every SM streams a buffer
// that stays L2-resident (16-64 MB, read many times), with the load flavours the
// traversals use.  Also the random 32-byte-sector rate (one 8-byte load per
// sector, like a cold gather) expressed in bytes moved.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_bw_bench tools/l2_bw_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(512) stream_kernel(const double* __restrict__ x, int64_t n4,
                                                     int reps, double* out) {
  double acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n4; k += stride) {
      double v[4];
      if (MODE == 0)
        asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
                     : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(x + 4 * k));
      else {
        asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                     : "=d"(v[0]), "=d"(v[1]) : "l"(x + 4 * k));
        asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                     : "=d"(v[2]), "=d"(v[3]) : "l"(x + 4 * k + 2));
      }
      acc += v[0] + v[1] + v[2] + v[3];
    }
  if (acc == 12345.678) out[0] = acc;
}

// one 8-byte load per (pseudo-random) 32-byte sector of an L2-resident buffer
__global__ void __launch_bounds__(512) sector_kernel(const double* __restrict__ x, int64_t nsec,
                                                     int64_t total, double* out) {
  double acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += 4 * stride) {
    double v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint64_t z = (uint64_t)(k + j * stride + 1) * 0x9E3779B97F4A7C15ULL;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
      z ^= z >> 31;
      asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v[j]) : "l"(x + 4 * (z % nsec)));
    }
    acc += v[0] + v[1] + v[2] + v[3];
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  double *x, *out;
  const int64_t maxn = 64LL << 20 >> 3;  // 64 MB of doubles
  cudaMalloc(&x, maxn * 8);
  cudaMalloc(&out, 8);
  cudaMemset(x, 0, maxn * 8);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mb : {8, 16, 32, 64}) {
    const int64_t n = (int64_t)mb << 20 >> 3;
    for (int mode = 0; mode < 2; ++mode) {
      const int reps = 4096 / mb;  // 4 GB of reads per launch
      for (int it = 0; it < 2; ++it) {
        cudaEventRecord(a);
        if (mode == 0) stream_kernel<0><<<148 * 4, 512>>>(x, n / 4, reps, out);
        else stream_kernel<1><<<148 * 4, 512>>>(x, n / 4, reps, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("stream %2d MB %s: %.3f ms, %.1f GB/s L2->SM\n", mb, mode ? "2x128-bit" : "256-bit", ms,
             (double)n * 8 * reps / ms * 1e-6);
    }
    const int64_t total = 1LL << 28;
    for (int it = 0; it < 2; ++it) {
      cudaEventRecord(a);
      sector_kernel<<<148 * 4, 512>>>(x, n / 4, total, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("random sectors %2d MB: %.3f ms, %.1f G sectors/s = %.1f GB/s of 32-byte sectors\n", mb, ms,
           total / ms * 1e-6, total * 32.0 / ms * 1e-6);
  }
  printf("cudaDevAttrClockRate %d kHz; %s\n", clk, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
