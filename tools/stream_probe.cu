// stream_probe.cu — find the best bulk-copy ring shape for HBM streaming on B200.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1612_07448_b200/csrc stream_probe.cu
// Reads a 4 GiB buffer of doubles and sums it, via (a) vectorised LDG, (b) the
// fb::TileRing bulk-copy ring with varied tile size / stages / CTAs per SM.
#include <cstdio>
#include <vector>

#include "fb_stream.cuh"

namespace fb {
void count_launch() {}
}  // namespace fb

using namespace fb;

__global__ void ldg_sum(const double2* __restrict__ a, int64_t n2, double* out) {
  double s = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
    double2 v = ld_stream_d2(a + i);
    s += v.x + v.y;
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

__device__ long long* g_trace;
__global__ void __launch_bounds__(kRingThreads) ring_sum(StreamSet ss, int64_t n_rows, int tile_rows, int stages, double* out) {
  extern __shared__ __align__(128) char smem[];
  TileRing ring;
  ring.init(smem, stages, tile_rows, n_rows);
  ring.start();
  if (is_producer_warp()) { ring.produce(ss); return; }
  double s = 0;
  const int words = ss.row_bytes[0] / 8;
  for (int64_t k = 0; k < ring.count(); ++k) {
    long long t0 = clock64();
    int st = ring.acquire(ss, k);
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 32 && k < 32 && g_trace) { g_trace[k] = t1; g_trace[32 + k] = t1 - t0; }
    const double* A = reinterpret_cast<const double*>(ring.stage_ptr(st, ss, 0));
    int n = ring.rows_of(ring.tile_begin + k) * words;
    for (int i = consumer_tid() * 2; i < n; i += kConsumerThreads * 2) {
      double2 v = *reinterpret_cast<const double2*>(A + i);
      s += v.x + v.y;
    }
    ring.release();
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

__global__ void burst(const char* a, int64_t bytes_per_cta, int chunk, int nchunks, int hint, double* out) {
  extern __shared__ __align__(128) char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  char* buf = smem + 128;
  if (threadIdx.x == 0) { for (int i = 0; i < nchunks; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
  __syncthreads();
  const char* base = a + blockIdx.x * bytes_per_cta;
  int64_t iters = bytes_per_cta / ((int64_t)chunk * nchunks);
  uint64_t pol = policy_evict_first();
  double s = 0;
  for (int64_t it = 0; it < iters; ++it) {
    if (threadIdx.x == 0) {
      for (int c = 0; c < nchunks; ++c) {
        mbar_arrive_expect_tx(&bar[c], chunk);
        const char* src = base + (it * nchunks + c) * (int64_t)chunk;
        if (hint) bulk_g2s_stream(buf + c * chunk, src, chunk, &bar[c], pol);
        else bulk_g2s(buf + c * chunk, src, chunk, &bar[c]);
      }
    }
    for (int c = 0; c < nchunks; ++c) mbar_wait(&bar[c], it & 1);
    s += reinterpret_cast<double*>(buf)[threadIdx.x];
    __syncthreads();
  }
  if (s == 12345.0) *out = s;
}


__global__ void mini_ring(const char* a, int64_t total_bytes, int tile, int stages, double* out) {
  extern __shared__ __align__(128) char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  char* buf = smem + 128;
  int64_t ntiles = total_bytes / tile;
  int64_t tb = ntiles * blockIdx.x / gridDim.x, te = ntiles * (blockIdx.x + 1) / gridDim.x;
  int64_t nt = te - tb;
  uint64_t pol = policy_evict_first();
  if (threadIdx.x == 0) { for (int i = 0; i < stages; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < stages && k < nt; ++k) {
      mbar_arrive_expect_tx(&bar[k], tile);
      bulk_g2s_stream(buf + k * tile, a + (tb + k) * (int64_t)tile, tile, &bar[k], pol);
    }
  double s = 0;
  int st = 0; uint32_t ph = 0;
  for (int64_t k = 0; k < nt; ++k) {
    long long t0 = clock64();
    mbar_wait(&bar[st], ph);
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0 && k < 32 && g_trace) { g_trace[k] = t1; g_trace[32 + k] = t1 - t0; }
    const double* A = reinterpret_cast<const double*>(buf + st * tile);
    for (int i = threadIdx.x * 2; i < tile / 8; i += blockDim.x * 2) { double2 v = *reinterpret_cast<const double2*>(A + i); s += v.x + v.y; }
    __syncthreads();
    if (threadIdx.x == 0 && k + stages < nt) {
      mbar_arrive_expect_tx(&bar[st], tile);
      bulk_g2s_stream(buf + st * tile, a + (tb + k + stages) * (int64_t)tile, tile, &bar[st], pol);
    }
    if (++st == stages) { st = 0; ph ^= 1; }
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

int main() {
  const int64_t bytes = 4LL << 30;
  const int64_t n = bytes / 8;
  double *a, *out;
  cudaMalloc(&a, bytes);
  cudaMalloc(&out, 8);
  cudaMemset(a, 0, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto fn) {
    for (int i = 0; i < 2; ++i) fn();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return bytes / (ms / 5 * 1e-3) / 1e9;
  };
  for (int per_sm : {1, 2, 4, 8}) {
    double gbs = timeit([&] { ldg_sum<<<sms * per_sm, 512>>>(reinterpret_cast<double2*>(a), n / 2, out); });
    printf("ldg   ctas/sm=%d threads=512 : %.0f GB/s\n", per_sm, gbs);
  }
  for (int hint : {1}) for (int chunk : {7680, 8192, 16384}) for (int nch : {1, 6}) {
    if (chunk * nch > 200 * 1024) continue;
    int grid = sms;
    int64_t per = bytes / grid;
    per -= per % ((int64_t)chunk * nch);
    size_t smem = 128 + (size_t)chunk * nch;
    cudaFuncSetAttribute(burst, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    double gbs = timeit([&] { burst<<<grid, 256, smem>>>(reinterpret_cast<const char*>(a), per, chunk, nch, hint, out); });
    printf("burst hint=%d chunk=%dKB nchunks=%d (1 cta/sm): %.0f GB/s %s\n", hint, chunk / 1024, nch, gbs * ((double)per * grid / bytes), cudaGetErrorString(cudaGetLastError()));
  }
  const int row_bytes = 160;  // 20 doubles, like S at c2
  {
    long long* tr; cudaMalloc(&tr, 64 * 8); cudaMemcpyToSymbol(g_trace, &tr, sizeof(tr));
    int tile_rows = 64; StreamSet ss{}; ss.count = 1; ss.base[0] = (const char*)a; ss.row_bytes[0] = 128; stream_layout(ss, tile_rows, bytes / 128);
    size_t smem = 256 + 6 * ss.stage_bytes; cudaFuncSetAttribute(ring_sum, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ring_sum<<<sms, kRingThreads, smem>>>(ss, bytes / 128, tile_rows, 6, out); cudaDeviceSynchronize();
    long long h[64]; cudaMemcpy(h, tr, 512, cudaMemcpyDeviceToHost);
    printf("waitcyc:"); for (int i = 0; i < 32; ++i) printf(" %lld", h[32 + i]); printf(" aligned=%d stage_bytes=%u pitch=%u\n", (int)ss.bulk_full, ss.stage_bytes, ss.pitch[0]);
    printf("trace:"); for (int i = 1; i < 32; ++i) printf(" %lld", h[i] - h[i-1]); printf("\n");
    cudaFuncSetAttribute(mini_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 + 6 * 8192);
    mini_ring<<<sms, 256, 128 + 6 * 8192>>>((const char*)a, bytes, 8192, 6, out); cudaDeviceSynchronize();
    cudaMemcpy(h, tr, 512, cudaMemcpyDeviceToHost);
    printf("mini waitcyc:"); for (int i = 0; i < 32; ++i) printf(" %lld", h[32 + i]); printf("\n");
    printf("mini trace:"); for (int i = 1; i < 32; ++i) printf(" %lld", h[i] - h[i-1]); printf("\n");
    long long* z = nullptr; cudaMemcpyToSymbol(g_trace, &z, sizeof(z));
    for (int tile : {8192, 16384, 32768}) for (int stg : {2, 4, 6}) { if (tile * stg > 200 * 1024) continue;
      cudaFuncSetAttribute(mini_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 + stg * tile);
      double gbs = timeit([&] { mini_ring<<<sms, 256, 128 + stg * tile>>>((const char*)a, bytes, tile, stg, out); });
      printf("mini tile=%d stages=%d: %.0f GB/s\n", tile, stg, gbs); }
  }
  for (int tile_kb : {8, 16, 32, 40}) {
    for (int stages : {2, 3, 4, 6}) {
      for (int per_sm : {1, 2, 3, 4}) {
        int tile_rows = (tile_kb * 1024 / row_bytes) & ~3;
        StreamSet ss{};
        ss.count = 1;
        ss.base[0] = reinterpret_cast<const char*>(a);
        ss.row_bytes[0] = row_bytes;
        stream_layout(ss, tile_rows, bytes / row_bytes);
        size_t smem = 256 + (size_t)stages * ss.stage_bytes;
        if ((smem + 1024) * per_sm > 228 * 1024) continue;
        cudaFuncSetAttribute(ring_sum, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int64_t rows = bytes / row_bytes;
        double gbs = timeit([&] { ring_sum<<<sms * per_sm, kRingThreads, smem>>>(ss, rows, tile_rows, stages, out); });
        cudaError_t err = cudaGetLastError();
        printf("ring  tile=%2dKB stages=%d ctas/sm=%d : %.0f GB/s %s\n", tile_kb, stages, per_sm, gbs,
               err ? cudaGetErrorString(err) : "");
      }
    }
  }
  return 0;
}
