#include <cstdio>
#include <cuda_runtime.h>
int main() {
  int v1 = 0, v2 = 0, v3 = 0;
  cudaDeviceGetAttribute(&v1, cudaDevAttrMaxPersistingL2CacheSize, 0);
  cudaDeviceGetAttribute(&v2, cudaDevAttrMaxAccessPolicyWindowSize, 0);
  cudaDeviceGetAttribute(&v3, cudaDevAttrL2CacheSize, 0);
  printf("max persisting %d MB, max window %d MB, L2 %d MB\n", v1 >> 20, v2 >> 20, v3 >> 20);
  return 0;
}
