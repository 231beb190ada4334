// DMMA.8x8x4 issue probe: clocks per DMMA per SM sub-partition for W warps per sub-partition, each
// running C independent accumulator chains (register operands only). Build: nvcc -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void probe(double* out, long long* clk, int iters) {
  double acc[C][2];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c][0] = acc[c][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += acc[c][0] + acc[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
template <int C>
void run(int wps, double* out, long long* clk) {
  const int iters = 4096;
  probe<C><<<148, 128 * wps>>>(out, clk, iters);
  probe<C><<<148, 128 * wps>>>(out, clk, iters);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
  printf("warps/SMSP %d chains %d: %.2f clk per DMMA per SMSP (chain step %.1f clk)\n", wps, C,
         (double)h / (iters * (double)C * wps), (double)h / iters);
}
int main() {
  double* out; long long* clk;
  cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&clk, 148 * 8);
  for (int wps : {1, 2, 4}) { run<1>(wps, out, clk); run<2>(wps, out, clk); run<4>(wps, out, clk); run<8>(wps, out, clk); }
  return 0;
}
