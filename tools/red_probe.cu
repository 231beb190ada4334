// red_probe.cu — L2 f64 RED throughput for the X·K scatter of RMM (c2: 20M rows -> 1M bins).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/red_probe tools/red_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void k_read(const int* fk, const double* x, int64_t n, double* sink) {
  double s = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += x[i] + fk[i];
  if (s == 12345.678) *sink = s;
}
__global__ void k_red(const int* fk, const double* x, int64_t n, double* bins) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(bins + fk[i], x[i]);
}
// unrolled: 4 independent loads in flight per thread before the REDs
__global__ void k_red4(const int* fk, const double* x, int64_t n, double* bins) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    int k0 = fk[i], k1 = fk[i + stride], k2 = fk[i + 2 * stride], k3 = fk[i + 3 * stride];
    double v0 = x[i], v1 = x[i + stride], v2 = x[i + 2 * stride], v3 = x[i + 3 * stride];
    atomicAdd(bins + k0, v0); atomicAdd(bins + k1, v1); atomicAdd(bins + k2, v2); atomicAdd(bins + k3, v3);
  }
  for (; i < n; i += stride) atomicAdd(bins + fk[i], x[i]);
}
__global__ void k_red_f32(const int* fk, const double* x, int64_t n, float* bins) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(bins + fk[i], (float)x[i]);
}

int main() {
  const int64_t n = 20000000, nr = 1000000;
  std::vector<int> hfk(n);
  std::mt19937 rng(1);
  for (auto& v : hfk) v = rng() % nr;
  std::vector<int> hsorted = hfk;
  std::sort(hsorted.begin(), hsorted.end());
  int *fk, *fks;
  double *x, *bins, *sink;
  float* binsf;
  cudaMalloc(&fk, n * 4); cudaMalloc(&fks, n * 4); cudaMalloc(&x, n * 8); cudaMalloc(&bins, nr * 8 * 64);
  cudaMalloc(&binsf, nr * 4); cudaMalloc(&sink, 8);
  cudaMemcpy(fk, hfk.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(fks, hsorted.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemset(x, 0, n * 8);
  void* flush; cudaMalloc(&flush, 512 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](const char* name, auto fn) {
    float best = 1e9;
    for (int t = 0; t < 5; ++t) {
      cudaMemset(flush, t, 512 << 20);
      cudaMemset(bins, 0, nr * 8);
      cudaEventRecord(a); fn(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
    }
    printf("%-40s %.4f ms  (%.1f G ops/s)  %s\n", name, best, n / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  for (int bpsm : {4, 8, 16}) {
    int grid = 148 * bpsm;
    char nm[64];
    snprintf(nm, 64, "read fk+x grid=%d", grid); timeit(nm, [&] { k_read<<<grid, 256>>>(fk, x, n, sink); });
    snprintf(nm, 64, "red f64 uniform grid=%d", grid); timeit(nm, [&] { k_red<<<grid, 256>>>(fk, x, n, bins); });
    snprintf(nm, 64, "red4 f64 uniform grid=%d", grid); timeit(nm, [&] { k_red4<<<grid, 256>>>(fk, x, n, bins); });
    snprintf(nm, 64, "red f64 sorted grid=%d", grid); timeit(nm, [&] { k_red<<<grid, 256>>>(fks, x, n, bins); });
    snprintf(nm, 64, "red f32 uniform grid=%d", grid); timeit(nm, [&] { k_red_f32<<<grid, 256>>>(fk, x, n, binsf); });
  }
  return 0;
}
