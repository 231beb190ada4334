// Probe: L2 size and persisting-L2 limits (development aid).
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  int l2 = 0, maxp = 0, maxwin = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0);
  cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, 0);
  printf("l2 %d MB, max persisting %d MB, max window %d MB\n", l2 >> 20, maxp >> 20, maxwin >> 20);
  return 0;
}
