// Random row-gather read bandwidth probe (development aid): one warp per 480-byte row,
// 16-byte loads, rows visited in identity / random / windowed-random order.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void gather_sum(const double2* __restrict__ s, int pitch2, const int* __restrict__ perm, long n, double* out) {
  const int lane = threadIdx.x & 31;
  const long warps = (long)gridDim.x * blockDim.x / 32;
  double acc = 0;
  for (long r = ((long)blockIdx.x * blockDim.x + threadIdx.x) / 32; r < n; r += warps) {
    const int src = perm[r];
    if (lane < pitch2) {
      double2 v = __ldcs(s + (long)src * pitch2 + lane);
      acc += v.x + v.y;
    }
  }
  if (acc == 123.456) out[0] = acc;
}

int main(int argc, char** argv) {
  const long n = 10000000;
  const int d = argc > 1 ? atoi(argv[1]) : 60;
  const int pitch2 = d / 2;
  double2* s;
  int* perm;
  double* out;
  cudaMalloc(&s, n * d * 8);
  cudaMemset(s, 0, n * d * 8);
  cudaMalloc(&perm, n * 4);
  cudaMalloc(&out, 8);
  std::vector<int> h(n);
  std::mt19937 rng(1);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"identity", "random", "win64k", "win1M", "sorted-blocks"};
  for (int mode = 0; mode < 4; ++mode) {
    for (long i = 0; i < n; ++i) h[i] = (int)i;
    if (mode == 1) std::shuffle(h.begin(), h.end(), rng);
    if (mode >= 2) {
      const long w = mode == 2 ? 65536 : 1048576;
      for (long i = 0; i < n; i += w) std::shuffle(h.begin() + i, h.begin() + std::min(n, i + w), rng);
    }
    cudaMemcpy(perm, h.data(), n * 4, cudaMemcpyHostToDevice);
    for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
      gather_sum<<<blocks, 512>>>(s, pitch2, perm, n, out);
      cudaEventRecord(a);
      for (int it = 0; it < 5; ++it) gather_sum<<<blocks, 512>>>(s, pitch2, perm, n, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ms /= 5;
      printf("%-9s d=%d blocks=%5d %7.3f ms %7.0f GB/s\n", names[mode], d, blocks, ms, n * (d * 8.0 + 4) / ms / 1e6);
    }
  }
  return 0;
}
