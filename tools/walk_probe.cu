// KᵀS walker micro-benchmark (development aid): the crossprod S-pass walk (batches of 8
// sorted rows, one thread per column) over synthetic shared-memory tiles (mean run
// length 20), alone on 2 warps. V=0: run sums stored to global memory as they close (the
// product walk); V=1: stored to a shared-memory staging buffer. Prints cycles per tile.
#include "../paper_1612_07448_b200/csrc/fb_crossprod.cu"
#include <cstdio>

namespace fb {
void count_launch(const char*, int) {}

template <int V>
struct Walk {
  const GramArgs& a;
  double* stg;
  int base;
  __device__ void flush(SegState& st, int col) {
    if (st.key < 0) return;
    if (V == 1)
      stg[((st.key - base) & 31) * a.seg_cols + col] = st.sum;
    else
      a.bins[static_cast<int64_t>(st.key) * a.seg_cols + col] = st.sum;
  }
  __device__ void row(SegState& st, int col, int key, double v) {
    if (key == st.key) {
      st.sum += v;
      return;
    }
    flush(st, col);
    if (st.key >= 0) st.first = false;
    st.key = key;
    st.sum = v;
  }
};

// Run-mask walk: boundaries of the tile from 4 ballots; each run segment is a branch-free
// two-accumulator sum; one staged store per closed run.
__device__ __forceinline__ int next_start(int r, int rows, uint32_t m0, uint32_t m1, uint32_t m2, uint32_t m3) {
  // first run start > r (rows if none)
  const int s = r + 1;
  uint32_t w;
  if (s < 32 && (w = m0 & (0xffffffffu << s))) return __ffs(w) - 1;
  if (s < 64 && (w = m1 & (s > 32 ? 0xffffffffu << (s - 32) : 0xffffffffu))) return 32 + __ffs(w) - 1;
  if (s < 96 && (w = m2 & (s > 64 ? 0xffffffffu << (s - 64) : 0xffffffffu))) return 64 + __ffs(w) - 1;
  if (s < 128 && (w = m3 & (s > 96 ? 0xffffffffu << (s - 96) : 0xffffffffu))) return 96 + __ffs(w) - 1;
  return rows;
}

__global__ void walk_probe_mask(GramArgs a, int tiles, int rows, int p, long long* cyc) {
  extern __shared__ double S[];
  __shared__ int32_t keys[128];
  __shared__ double stg[32 * 64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < rows * p; i += blockDim.x) S[i] = 1.0 + i;
  __syncthreads();
  const int c = warp * 32 + lane;
  int key = -1;
  double sum = 0.0;
  int key0 = 0;
  long long t0 = clock64();
  for (int t = 0; t < tiles; ++t) {
    if (threadIdx.x < 32)
      for (int r = lane; r < rows; r += 32) keys[r] = key0 + (r + (t * 7) % 20) / 20;
    __syncthreads();
    const int base = key;
    auto bnd = [&](int r) {
      const int cur = r < rows ? keys[r] : 0;
      const int prev = r == 0 ? key : keys[r - 1 < rows ? r - 1 : 0];
      return __ballot_sync(0xffffffffu, r < rows && cur != prev);
    };
    const uint32_t m0 = bnd(lane), m1 = bnd(32 + lane), m2 = bnd(64 + lane), m3 = bnd(96 + lane);
    int r = 0;
    while (r < rows) {
      const int e = next_start(r, rows, m0, m1, m2, m3);
      const bool start = r == 0 ? (m0 & 1u) : true;
      if (start) {
        if (key >= 0 && c < a.seg_cols) stg[((key - base) & 31) * a.seg_cols + c] = sum;
        key = keys[r];
        sum = 0.0;
      }
      if (c < a.seg_cols) {
        const double* col = S + c;
        double s0 = 0.0, s1 = 0.0;
        int k = r;
        for (; k + 4 <= e; k += 4) {
          s0 += col[k * p] + col[(k + 1) * p];
          s1 += col[(k + 2) * p] + col[(k + 3) * p];
        }
        for (; k < e; ++k) s0 += col[k * p];
        sum += s0 + s1;
      }
      r = e;
    }
    key0 = keys[rows - 1];
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (sum == 123.0) a.bins[0] = sum;
}

template <int V>
__global__ void walk_probe(GramArgs a, int tiles, int rows, int p, long long* cyc) {
  extern __shared__ double S[];  // rows x p
  __shared__ int32_t keys[128];
  __shared__ double stg[32 * 64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < rows * p; i += blockDim.x) S[i] = 1.0 + i;
  __syncthreads();
  const int i = warp * 32 + lane;
  SegState st{-1, 0.0, true};
  int key0 = 0;
  long long t0 = clock64();
  for (int t = 0; t < tiles; ++t) {
    if (threadIdx.x < 32)
      for (int r = lane; r < rows; r += 32) keys[r] = key0 + (r + (t * 7) % 20) / 20;
    __syncthreads();
    Walk<V> w{a, stg, key0};
    if (i < a.seg_cols) {
      int r = 0;
      for (; r + 8 <= rows; r += 8) {
        int kk[8];
        double vv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          kk[j] = keys[r + j];
          vv[j] = S[(r + j) * p + i];
        }
        if (kk[7] == st.key) {
          st.sum += ((vv[0] + vv[1]) + (vv[2] + vv[3])) + ((vv[4] + vv[5]) + (vv[6] + vv[7]));
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) w.row(st, i, kk[j], vv[j]);
        }
      }
      for (; r < rows; ++r) w.row(st, i, keys[r], S[r * p + i]);
    }
    key0 = keys[rows - 1];
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (st.sum == 123.0) a.bins[0] = st.sum;
}
}  // namespace fb

int main() {
  fb::GramArgs a{};
  a.seg = 1;
  a.seg_cols = 60;
  cudaMalloc(&a.bins, 64ull << 20);
  long long* cyc;
  cudaMallocManaged(&cyc, 64);
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 60 * 8);
    kern<<<1, 64, 96 * 60 * 8>>>(a, 2000, 96, 60, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%-28s %.0f cycles per 96-row tile (%s)\n", name, cyc[0] / 2000.0, cudaGetErrorString(e));
  };
  run(fb::walk_probe<0>, "walk, global run stores");
  run(fb::walk_probe<1>, "walk, shared staging");
  run(fb::walk_probe_mask, "run-mask walk, staging");
  return 0;
}
