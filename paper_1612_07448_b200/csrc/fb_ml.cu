#include <algorithm>
// fb_ml.cu — fused iteration kernels of the ML drivers (ml.py).
//
// GLM step (logistic_gd ml.py:199-215, linreg_gd ml.py:239-254), one pass over S per
// iteration instead of the reference's two (lmm then lmm on T.T):
//   phase 1 (per tile, L lanes per row as in the rowdot LMM): t_i = S_i·w_S + Σ_q z_q[fk_q,i]
//           (z_q = R_q·w_q from the previous z-pass); logistic: p_i = y_i/(1+exp(t_i)),
//           loss_i = log1p(exp(-|y_i t_i|)) + max(-y_i t_i, 0); linear: p_i = t_i - y_i,
//           loss_i = p_i²; p_i is scattered into bins_q[fk_q,i] (Kᵀp) and kept in shared memory;
//   phase 2 (same tile, threads <-> columns): g_S += p_i·S_i.
// Per-CTA partials of (g_S, loss) are summed in CTA order by the last CTA (deterministic).
// The R side (g_q = bins_qᵀ R_q) is the weighted column reduction of fb_reduce.cu, and
// glm_update applies w ± α·g, records the objective and the first non-finite iteration.
#include <cmath>
#include <cstdlib>

#include "fb_kernels.cuh"

namespace fb {

constexpr int kZStride = 2;  // z rows are padded to 16 bytes (bulk-copy gathers)

struct GlmDev {
  GlmArgs g;
  int debug;  // development bisection bits (FB_GLM_DEBUG)
  int lanes, cols;
  int y_stream, fk_stream0;
};

__global__ void __launch_bounds__(kRingThreads, 1) glm_spass_kernel(GlmDev p, StreamSet ss, int stages, int tile_rows) {
  extern __shared__ __align__(128) char smem[];
  const int d = p.g.d;
  double* ws = reinterpret_cast<double*>(smem);  // w_S
  const size_t ws_bytes = (static_cast<size_t>(d > 0 ? d : 1) * 8 + 127) & ~size_t(127);
  double* pt = reinterpret_cast<double*>(smem + ws_bytes);  // p of the current tile: [2][tile_rows]
  const size_t pt_bytes = (static_cast<size_t>(2 * tile_rows) * 8 + 127) & ~size_t(127);
  double* red = reinterpret_cast<double*>(smem + ws_bytes + pt_bytes);  // [kConsumerThreads] fold space
  const size_t red_bytes = (static_cast<size_t>(kConsumerThreads) * 8 + 127) & ~size_t(127);
  char* buf = smem + ws_bytes + pt_bytes + red_bytes;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ws[i] = p.g.w[i];

  TileRing ring;
  ring.init(buf, stages, tile_rows, p.g.n);
  ring.start(ss);
  if (ring.service(ss)) return;
  const int lane = lane_id();
  const int warp = consumer_warp();
  const int tid = consumer_tid();
  const int rw = tile_rows / kConsumerWarps;
  const int wrow = warp * rw;
  const int L = p.lanes, C = p.cols;
  const int rpi = 32 / L;
  const int iters = (rw + rpi - 1) / rpi;
  const int sub = lane % L, rsub = lane / L;
  const uint64_t keep = policy_evict_last();
  const bool logistic = p.g.mode == 0;
  // phase-2 layout
  const int groups = d > 0 ? kConsumerThreads / d : 0;
  const int col = d > 0 ? tid % d : 0, grp = d > 0 ? tid / d : 0;
  const bool colthread = grp < groups;
  double gacc = 0.0, lacc = 0.0;

  for (int64_t kt = 0; kt < ring.count(); ++kt) {
    const int cur = ring.acquire(ss, kt);
    const int64_t tile = ring.tile_begin + kt;
    const int rows = ring.rows_of(tile);
    const double* A = reinterpret_cast<const double*>(ring.stage_ptr(cur, ss, 0));
    const double* Y = reinterpret_cast<const double*>(ring.stage_ptr(cur, ss, p.y_stream));
    double* ptile = pt + (kt & 1) * tile_rows;

    // ---- phase 1: row dot products, p and loss
    for (int it = 0; it < iters; ++it) {
      const int rl = it * rpi + rsub;
      const int r = wrow + rl;
      const bool live = rl < rw && r < rows;
      double acc = 0.0;
      if (live) {
        const double* arow = A + static_cast<size_t>(r) * d + sub;
        const double* xc = ws + sub;
#pragma unroll 4
        for (int m = 0; m < C; ++m) acc = fma(arow[m * L], xc[m * L], acc);
      }
      for (int o = L >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (live && sub == 0) {
        // + z_q[fk_q] in part order (rewrite.py:186-190), gathered into the stage
        if (!(p.debug & 4))
          for (int q = 0; q < p.g.nfk; ++q)
            acc += reinterpret_cast<const double*>(ring.gather_ptr(cur, ss, q))[r * kZStride];
        const double y = Y[r];
        double pv, lv;
        if (logistic) {
          const double yt = y * acc;
          pv = y / (1.0 + exp(acc));
          lv = log1p(exp(-fabs(yt))) + fmax(-yt, 0.0);
        } else {
          pv = acc - y;
          lv = pv * pv;
        }
        ptile[r] = pv;
        lacc += lv;
      }
      // Kᵀp scatter
      for (int q = 0; q < p.g.nfk; ++q) {
        const int32_t* fkt = reinterpret_cast<const int32_t*>(ring.stage_ptr(cur, ss, p.fk_stream0 + q));
        const bool act = live && sub == 0;
        if (act && !(p.debug & 1)) {
          const double pv = ptile[r];
          red_add(p.g.bins[q] + fkt[r], pv);
        }
      }
    }
    consumer_sync();
    // ---- phase 2: g_S += p_i S_i (threads <-> columns)
    if (colthread && !(p.debug & 2)) {
      for (int r = grp; r < rows; r += groups) gacc = fma(ptile[r], A[static_cast<size_t>(r) * d + col], gacc);
    }
    ring.release();
  }

  // fold: loss over all consumer threads, gradient over row groups
  consumer_sync();
  red[tid] = lacc;
  consumer_sync();
  double* part = p.g.partials + static_cast<size_t>(blockIdx.x) * (d + 1);
  if (tid < 32) {  // fixed order: lane i adds red[i], red[i + 32], ..., then an xor tree
    double s = 0.0;
    for (int i = tid; i < kConsumerThreads; i += 32) s += red[i];
    s = warp_sum(s);
    if (tid == 0) part[d] = s;
  }
  consumer_sync();
  if (colthread) red[grp * d + col] = gacc;
  consumer_sync();
  for (int c = tid; c < d; c += kConsumerThreads) {
    double s = 0.0;
    for (int gI = 0; gI < groups; ++gI) s += red[gI * d + c];
    part[c] = s;
  }
  __threadfence();
  __shared__ unsigned int ticket;
  consumer_sync();
  if (tid == 0) ticket = atomicAdd(p.g.counter, 1u);
  consumer_sync();
  if (ticket != gridDim.x - 1) return;
  __threadfence();
  for (int c = tid >> 5; c <= d; c += kConsumerWarps) {  // one warp per output
    const double s = warp_sum_strided(p.g.partials + c, gridDim.x, static_cast<size_t>(d + 1));
    if ((tid & 31) == 0) {
      if (c < d)
        p.g.g_out[c] = s;
      else
        *p.g.loss_out = s;
    }
  }
  if (tid == 0) *p.g.counter = 0u;
}

cudaError_t launch_glm_spass(const GlmArgs& g, cudaStream_t st, int num_sms) {
  if (g.n <= 0) return cudaSuccess;
  if (g.d > 256) return cudaErrorNotSupported;
  GlmDev p{};
  p.g = g;
  int L = 1;
  while (g.d > 0 && L < 32 && (g.d % (2 * L)) == 0) L *= 2;
  p.lanes = L;
  p.cols = g.d / L;
  StreamSet ss{};
  int ns = 0;
  ss.base[ns] = reinterpret_cast<const char*>(g.s);
  ss.row_bytes[ns++] = static_cast<uint32_t>(g.d) * 8u;
  p.y_stream = ns;
  ss.base[ns] = reinterpret_cast<const char*>(g.y);
  ss.row_bytes[ns++] = 8u;
  p.fk_stream0 = ns;
  for (int q = 0; q < g.nfk; ++q) {
    ss.gkeys[q] = g.fk[q];
    ss.gbase[q] = reinterpret_cast<const char*>(g.z[q]);
    ss.grow_bytes[q] = kZStride * 8u;
    ss.base[ns] = reinterpret_cast<const char*>(g.fk[q]);
    ss.row_bytes[ns++] = 4u;
  }
  ss.ngather = g.nfk;
  ss.count = ns;
  if (const char* dbg = getenv("FB_GLM_DEBUG")) p.debug = atoi(dbg);
  if (p.debug & 8) ss.ngather = 0;
  uint32_t row_bytes = kZStride * 8u * g.nfk;
  for (int i = 0; i < ns; ++i) row_bytes += ss.row_bytes[i];
  int rw = 32;
  while (rw > 4 && static_cast<size_t>(row_bytes) * rw * kConsumerWarps > 48 * 1024) rw >>= 1;
  const int tile_rows = rw * kConsumerWarps;
  stream_layout(ss, tile_rows, g.n);
  const size_t fixed = ((static_cast<size_t>(g.d > 0 ? g.d : 1) * 8 + 127) & ~size_t(127)) +
                       ((static_cast<size_t>(2 * tile_rows) * 8 + 127) & ~size_t(127)) +
                       ((static_cast<size_t>(kConsumerThreads) * 8 + 127) & ~size_t(127));
  const size_t budget = 200 * 1024;
  int stages = static_cast<int>((budget - fixed - kRingHeader) / ss.stage_bytes);
  if (stages > 8) stages = 8;
  if (stages < 2) return cudaErrorNotSupported;
  const size_t smem = fixed + kRingHeader + static_cast<size_t>(stages) * ss.stage_bytes;
  cudaError_t e = cudaFuncSetAttribute(glm_spass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int64_t ntiles = (g.n + tile_rows - 1) / tile_rows;
  const int grid = grid_for(ntiles, 1, 1, num_sms);
  e = cudaMemsetAsync(g.counter, 0, sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  glm_spass_kernel<<<grid, kRingThreads, smem, st>>>(p, ss, stages, tile_rows);
  FB_LAUNCHED();
  return cudaGetLastError();
}

size_t glm_partials_doubles(int d, int num_sms) { return static_cast<size_t>(num_sms) * (d + 1); }

// w ± α·g, objective trace, first non-finite iteration (ml.py:190-192).
__global__ void glm_update_kernel(double* w, const double* g, int d, double alpha, const double* loss, double* trace,
                                  int it, int* diverged) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    const double v = w[j] + alpha * g[j];
    w[j] = v;
    if (!isfinite(v)) bad = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    trace[it] = *loss;
    if (bad && *diverged < 0) *diverged = it;
  }
}

cudaError_t launch_glm_update(double* w, const double* g, int d, double alpha, const double* loss, double* trace,
                              int it, int* diverged, cudaStream_t st) {
  glm_update_kernel<<<1, 256, 0, st>>>(w, g, d, alpha, loss, trace, it, diverged);
  FB_LAUNCHED();
  return cudaGetLastError();
}


// ======================================================================== K-Means
// (ml.py:257-285) One iteration after the LMM tc = T·(2C) (bitwise (2T)·C: scaling by 2 is
// exact): dist_ik = (d_t[i] + cc[k]) - tc[i,k]; argmin with ties to the lowest index
// (kernel.row_min_mask, kernel.py:327-339); objective Σ_i dist_i,a_i; integer cluster sizes
// and integer FK/cluster histograms (Aᵀ K_q, exact); the S-side cluster sums are a
// separate one-hot column reduction.
namespace {
__device__ __forceinline__ double warp_sum_d(double v) { return warp_sum(v); }
}  // namespace

__global__ void kmeans_assign_kernel(const double* __restrict__ tc, const double* __restrict__ d_t,
                                     const double* __restrict__ cc, int64_t n, int k, KmFk fks,
                                     int32_t* __restrict__ assign, int32_t* __restrict__ sizes,
                                     double* __restrict__ partials, unsigned* counter, double* trace, int it,
                                     unsigned long long* nan_row) {
  extern __shared__ double km_assign_smem[];  // cc[k], then the CTA's k size counters
  double* ccs = km_assign_smem;
  int32_t* ssz = reinterpret_cast<int32_t*>(km_assign_smem + k);
  __shared__ double wsum[32];
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    ccs[j] = cc[j];
    ssz[j] = 0;
  }
  __syncthreads();
  double acc = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double dt = d_t[i];
    const double* row = tc + i * k;
    int best = 0;
    double bv = (dt + ccs[0]) - row[0];
    bool nan = isnan(bv);
    for (int j = 1; j < k; ++j) {
      const double v = (dt + ccs[j]) - row[j];
      nan |= isnan(v);
      if (v < bv) {
        bv = v;
        best = j;
      }
    }
    // (iteration, row) packed: the smallest is the first NaN row of the FIRST iteration that
    // saw one — the row the reference reports when row_min_mask raises (kernel.py:330-332)
    if (nan) atomicMin(nan_row, (static_cast<unsigned long long>(it) << 40) | static_cast<unsigned long long>(i));
    assign[i] = best;
    acc += bv;
    atomicAdd(&ssz[best], 1);
    for (int q = 0; q < fks.nfk; ++q) red_add(fks.bins[q] + static_cast<int64_t>(fks.fk[q][i]) * k + best, 1);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x)
    if (ssz[j]) red_add(sizes + j, ssz[j]);
  // deterministic objective: warp tree, block in warp order, CTAs in order by the last CTA
  acc = warp_sum_d(acc);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += wsum[w];
    partials[blockIdx.x] = s;
  }
  __threadfence();
  __shared__ unsigned ticket;
  if (threadIdx.x == 0) ticket = atomicAdd(counter, 1u);
  __syncthreads();
  if (ticket != gridDim.x - 1) return;
  __threadfence();
  if (threadIdx.x < 32) {
    const double s = warp_sum_strided(partials, gridDim.x, 1);
    if (threadIdx.x == 0) {
      trace[it] = s;
      *counter = 0u;
    }
  }
}

cudaError_t launch_kmeans_assign(const double* tc, const double* d_t, const double* cc, int64_t n, int k,
                                 const KmFk& fks, int32_t* assign, int32_t* sizes, double* partials, unsigned* counter,
                                 double* trace, int it, unsigned long long* nan_row, cudaStream_t st, int num_sms) {
  if (k < 1 || k > kKmeansMaxK) return cudaErrorNotSupported;
  cudaError_t e = cudaMemsetAsync(sizes, 0, sizeof(int32_t) * k, st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(counter, 0, sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  const int grid = grid_for(n, 256, 4, num_sms);
  kmeans_assign_kernel<<<grid, 256, static_cast<size_t>(k) * 12, st>>>(tc, d_t, cc, n, k, fks, assign, sizes, partials,
                                                                       counter, trace, it, nan_row);
  FB_LAUNCHED();
  return cudaGetLastError();
}

// out[c*k + j] = Σ_{i: assign[i] = j} S[i, c]: per-thread private accumulators in shared
// memory (stride k+1 doubles: conflict-free), per-CTA partials summed in CTA order.
// Clusters [j0, j0 + kc) of k per launch (kc <= 64: the shared accumulators of wider k do not fit):
// rows of other clusters fall into the spare slot kc, so every cluster's rows are summed in the
// order one unwindowed launch would use.
__global__ void onehot_colsum_kernel(const double* __restrict__ s, int64_t n, int d, const int32_t* __restrict__ assign,
                                     int k, int j0, int kc, double* partials, unsigned* counter, double* out) {
  extern __shared__ double accs[];  // [blockDim.x][kc + 1]
  const int tid = threadIdx.x;
  const int ks = kc + 1;
  auto slot = [&](int a) { return static_cast<unsigned>(a - j0) < static_cast<unsigned>(kc) ? a - j0 : kc; };
  for (int j = 0; j < ks; ++j) accs[tid * ks + j] = 0.0;
  const int groups = blockDim.x / d;
  const int col = tid % d, grp = tid / d;
  if (grp < groups) {
    // 8 rows per batch: all loads issued before the shared-memory updates (ILP)
    const int64_t step = static_cast<int64_t>(gridDim.x) * groups;
    int64_t r = blockIdx.x * static_cast<int64_t>(groups) + grp;
    for (; r + 7 * step < n; r += 8 * step) {
      int a[8];
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a[u] = __ldg(assign + r + u * step);
        v[u] = __ldg(s + (r + u * step) * d + col);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) accs[tid * ks + slot(a[u])] += v[u];
    }
    for (; r < n; r += step) accs[tid * ks + slot(assign[r])] += s[r * d + col];
  }
  __syncthreads();
  // fold groups -> per-CTA partial [d][kc]
  double* part = partials + static_cast<size_t>(blockIdx.x) * d * kc;
  for (int e = tid; e < d * kc; e += blockDim.x) {
    const int c = e / kc, j = e % kc;
    double v = 0.0;
    for (int gI = 0; gI < groups; ++gI) v += accs[(gI * d + c) * ks + j];
    part[e] = v;
  }
  __threadfence();
  __shared__ unsigned ticket;
  __syncthreads();
  if (tid == 0) ticket = atomicAdd(counter, 1u);
  __syncthreads();
  if (ticket != gridDim.x - 1) return;
  __threadfence();
  for (int e = tid >> 5; e < d * kc; e += blockDim.x >> 5) {  // one warp per output
    const double v = warp_sum_strided(partials + e, gridDim.x, static_cast<size_t>(d) * kc);
    if ((tid & 31) == 0) out[(e / kc) * k + j0 + e % kc] = v;
  }
  if (tid == 0) *counter = 0u;
}

// Narrow S (d <= 32): lanes over columns, rows in contiguous per-warp ranges, 16 rows' loads
// in flight per warp, then each row added into the warp's own shared accumulator row
// acc[a_i][c] (consecutive lanes, consecutive banks). Warps folded in warp order, CTAs in CTA
// order (deterministic). The per-thread private accumulators above (stride k + 1) ran at half
// of HBM bandwidth at c4 (0.50 ms for 1.6 GB).
constexpr int kOhThreads = 512;
__global__ void __launch_bounds__(kOhThreads) onehot_colsum_lanes_kernel(const double* __restrict__ s, int64_t n, int d,
                                                                        const int32_t* __restrict__ assign, int k,
                                                                        double* partials, unsigned* counter, double* out) {
  extern __shared__ double wacc[];  // [2][warps][k][d]: even / odd rows (two independent RMW chains)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kOhThreads / 32;
  const int kd = k * d;
  for (int e = threadIdx.x; e < 2 * nw * kd; e += kOhThreads) wacc[e] = 0.0;
  __syncthreads();
  double* acc0 = wacc + warp * kd;
  double* acc1 = wacc + (nw + warp) * kd;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * nw + warp, nwarps = static_cast<int64_t>(gridDim.x) * nw;
  const int64_t lo = n * gw / nwarps, hi = n * (gw + 1) / nwarps;
  const bool on = lane < d;
  constexpr int U = 16;
  for (int64_t r0 = lo; r0 < hi; r0 += U) {
    const int cnt = hi - r0 < U ? static_cast<int>(hi - r0) : U;
    const int al = lane < cnt ? __ldg(assign + r0 + lane) : 0;
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = (on && u < cnt) ? __ldcs(s + (r0 + u) * d + lane) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int a = __shfl_sync(0xffffffffu, al, u);
      if (on && u < cnt) ((u & 1) ? acc1 : acc0)[a * d + lane] += v[u];
    }
  }
  __syncthreads();
  double* part = partials + static_cast<size_t>(blockIdx.x) * kd;  // layout [c][j]
  for (int e = threadIdx.x; e < kd; e += kOhThreads) {
    const int j = e / d, c = e % d;
    double v = 0.0;
    for (int w = 0; w < 2 * nw; ++w) v += wacc[w * kd + e];
    part[c * k + j] = v;
  }
  __threadfence();
  __shared__ unsigned ticket;
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(counter, 1u);
  __syncthreads();
  if (ticket != gridDim.x - 1) return;
  __threadfence();
  for (int e = warp; e < kd; e += nw) {  // one warp per output, CTAs in a fixed order
    const double v = warp_sum_strided(partials + e, gridDim.x, static_cast<size_t>(kd));
    if (lane == 0) out[e] = v;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// Bulk-staged variant for even d: each warp streams its contiguous row range through its own
// ring of `stages` shared-memory buffers, 16 rows (16·d·8 bytes, one cp.async.bulk) per buffer,
// so ~stages·16 rows per warp stay in flight without holding them in registers; the warp's
// assignments for the next batch are prefetched one batch ahead. The shared accumulators and
// the deterministic fold are those of onehot_colsum_lanes_kernel.
constexpr int kOhBatch = 16;
__global__ void __launch_bounds__(kOhThreads, 1) onehot_colsum_bulk_kernel(const double* __restrict__ s, int64_t n,
                                                                           int d, const int32_t* __restrict__ assign,
                                                                           int k, int stages, double* partials,
                                                                           unsigned* counter, double* out) {
  extern __shared__ __align__(16) double oh_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kOhThreads / 32;
  const int kd = k * d;
  double* wacc = oh_smem;                               // [2][warps][k][d]
  double* ring = wacc + 2 * nw * kd;                    // [warps][stages][16][d]
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + static_cast<size_t>(nw) * stages * kOhBatch * d);
  for (int e = threadIdx.x; e < 2 * nw * kd; e += kOhThreads) wacc[e] = 0.0;
  uint64_t* mb = bars + warp * stages;
  if (lane == 0) {
    for (int st = 0; st < stages; ++st) mbar_init(&mb[st], 1);
    fence_mbar_init();
  }
  __syncthreads();
  double* acc0 = wacc + warp * kd;
  double* acc1 = wacc + (nw + warp) * kd;
  double* my = ring + static_cast<size_t>(warp) * stages * kOhBatch * d;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * nw + warp, nwarps = static_cast<int64_t>(gridDim.x) * nw;
  const int64_t lo = n * gw / nwarps, hi = n * (gw + 1) / nwarps;
  const int64_t nb = (hi - lo + kOhBatch - 1) / kOhBatch;
  auto issue = [&](int64_t b, int st) {
    const int64_t r0 = lo + b * kOhBatch;
    const int cnt = hi - r0 < kOhBatch ? static_cast<int>(hi - r0) : kOhBatch;
    const uint32_t bytes = static_cast<uint32_t>(cnt) * d * 8u;
    mbar_arrive_expect_tx(&mb[st], bytes);
    bulk_g2s(my + st * kOhBatch * d, s + r0 * d, bytes, &mb[st]);
  };
  if (lane == 0)
    for (int b = 0; b < stages && b < nb; ++b) issue(b, b);
  const bool on = lane < d;
  int al_next = (nb > 0 && lane < hi - lo) ? __ldg(assign + lo + lane) : 0;
  int st = 0;
  uint32_t phase = 0;
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t r0 = lo + b * kOhBatch;
    const int cnt = hi - r0 < kOhBatch ? static_cast<int>(hi - r0) : kOhBatch;
    const int al = al_next;
    if (b + 1 < nb) al_next = (lane < hi - r0 - kOhBatch) && lane < kOhBatch ? __ldg(assign + r0 + kOhBatch + lane) : 0;
    mbar_wait(&mb[st], phase);
    const double* buf = my + st * kOhBatch * d;
#pragma unroll
    for (int u = 0; u < kOhBatch; ++u) {
      const int a = __shfl_sync(0xffffffffu, al, u);
      if (on && u < cnt) ((u & 1) ? acc1 : acc0)[a * d + lane] += buf[u * d + lane];
    }
    __syncwarp();
    if (lane == 0 && b + stages < nb) {
      fence_proxy_async();
      issue(b + stages, st);
    }
    if (++st == stages) {
      st = 0;
      phase ^= 1u;
    }
  }
  __syncthreads();
  double* part = partials + static_cast<size_t>(blockIdx.x) * kd;  // layout [c][j]
  for (int e = threadIdx.x; e < kd; e += kOhThreads) {
    const int j = e / d, c = e % d;
    double v = 0.0;
    for (int w = 0; w < 2 * nw; ++w) v += wacc[w * kd + e];
    part[c * k + j] = v;
  }
  __threadfence();
  __shared__ unsigned ticket;
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(counter, 1u);
  __syncthreads();
  if (ticket != gridDim.x - 1) return;
  __threadfence();
  for (int e = warp; e < kd; e += nw) {
    const double v = warp_sum_strided(partials + e, gridDim.x, static_cast<size_t>(kd));
    if (lane == 0) out[e] = v;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

size_t onehot_partials_doubles(int d, int k, int num_sms) { return static_cast<size_t>(num_sms) * 2 * d * k; }

cudaError_t launch_onehot_colsum(const double* s, int64_t n, int d, const int32_t* assign, int k, double* partials,
                                 unsigned* counter, double* out, cudaStream_t st, int num_sms) {
  if (d < 1) return cudaSuccess;
  const size_t lane_smem = 2 * static_cast<size_t>(kOhThreads / 32) * k * d * 8;
  const size_t stage_bytes = static_cast<size_t>(kOhThreads / 32) * kOhBatch * d * 8;
  const int stages = lane_smem < 200 * 1024 ? static_cast<int>(std::min<size_t>(4, (200 * 1024 - lane_smem) / stage_bytes)) : 0;
  if (d <= 32 && d % 2 == 0 && stages >= 2 && (reinterpret_cast<uintptr_t>(s) & 15) == 0 && !getenv("FB_KM_ONEHOT_LANES") &&
      !getenv("FB_KM_ONEHOT_OLD")) {
    const size_t smem = lane_smem + static_cast<size_t>(stages) * stage_bytes + (kOhThreads / 32) * stages * 8;
    cudaError_t e = cudaFuncSetAttribute(onehot_colsum_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(counter, 0, sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    const int grid = grid_for(n, 16 * kOhBatch, 1, num_sms);
    onehot_colsum_bulk_kernel<<<grid, kOhThreads, smem, st>>>(s, n, d, assign, k, stages, partials, counter, out);
    FB_LAUNCHED();
    return cudaGetLastError();
  }
  if (d <= 32 && lane_smem <= 100 * 1024 && !getenv("FB_KM_ONEHOT_OLD")) {
    cudaError_t e = cudaFuncSetAttribute(onehot_colsum_lanes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(lane_smem));
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(counter, 0, sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    const int grid = grid_for(n, 16 * 256, 2, num_sms);  // <= 2 CTAs per SM: the partials slots
    onehot_colsum_lanes_kernel<<<grid, kOhThreads, lane_smem, st>>>(s, n, d, assign, k, partials, counter, out);
    FB_LAUNCHED();
    return cudaGetLastError();
  }
  if (d > 256 || k > kKmeansMaxK) return cudaErrorNotSupported;
  int threads = 256;
  const int kc_max = k < 64 ? k : 64;
  const size_t smem = static_cast<size_t>(threads) * (kc_max + 1) * 8;
  cudaError_t e = cudaFuncSetAttribute(onehot_colsum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(counter, 0, sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  const int groups = threads / d;
  const int grid = grid_for(n, groups * 16, 2, num_sms);
  for (int j0 = 0; j0 < k; j0 += kc_max) {  // one pass over S per window of 64 clusters
    const int kc = k - j0 < kc_max ? k - j0 : kc_max;
    onehot_colsum_kernel<<<grid, threads, smem, st>>>(s, n, d, assign, k, j0, kc, partials, counter, out);
    FB_LAUNCHED();
  }
  return cudaGetLastError();
}

// c[:, j] = tta[:, j] / sizes[j] for non-empty clusters (empty ones keep their centroid,
// ml.py:281-283); cc[j] = Σ_c c[c, j]².
__global__ void kmeans_update_kernel(double* c, const double* tta, const int32_t* sizes, int d, int k, double* cc) {
  for (int e = threadIdx.x; e < d * k; e += blockDim.x) {
    const int j = e % k;
    if (sizes[j] > 0) c[e] = tta[e] / static_cast<double>(sizes[j]);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < d; ++r) s += c[r * k + j] * c[r * k + j];
    cc[j] = s;
  }
}

cudaError_t launch_kmeans_update(double* c, const double* tta, const int32_t* sizes, int d, int k, double* cc,
                                 cudaStream_t st) {
  kmeans_update_kernel<<<1, 256, 0, st>>>(c, tta, sizes, d, k, cc);
  FB_LAUNCHED();
  return cudaGetLastError();
}

// ======================================================================== GNMF
// (ml.py:288-317) Multiplicative updates with the 1e-12 guard, in the reference's
// operation order: h = h*ttw / (h@cpw + eps); w = w*th / (w@cph + eps).
template <int R>
__global__ void nmf_update_kernel(double* __restrict__ f, const double* __restrict__ num, const double* __restrict__ g,
                                  int64_t rows, double eps) {
  __shared__ double gs[R * R];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) gs[e] = g[e];
  __syncthreads();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double fr[R], nr[R];
#pragma unroll
    for (int s = 0; s < R; ++s) {
      fr[s] = f[i * R + s];
      nr[s] = num[i * R + s];
    }
#pragma unroll
    for (int s = 0; s < R; ++s) {
      double den = 0.0;
#pragma unroll
      for (int t = 0; t < R; ++t) den = fma(fr[t], gs[t * R + s], den);
      f[i * R + s] = fr[s] * nr[s] / (den + eps);
    }
  }
}

// 16 < r <= 64: a warp per row, lane s owning columns s and s + 32; the old row is broadcast by
// shuffles, the denominators accumulate over t in ascending order exactly as above.
__global__ void nmf_update_wide_kernel(double* __restrict__ f, const double* __restrict__ num,
                                       const double* __restrict__ g, int64_t rows, int r, double eps) {
  extern __shared__ double gw[];  // r × r
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) gw[e] = g[e];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const bool on0 = lane < r, on1 = lane + 32 < r;
  for (int64_t i = warp; i < rows; i += nwarps) {
    const double f0 = on0 ? f[i * r + lane] : 0.0, f1 = on1 ? f[i * r + lane + 32] : 0.0;
    double den0 = 0.0, den1 = 0.0;
    for (int t = 0; t < r; ++t) {
      const double ft = __shfl_sync(0xffffffffu, t < 32 ? f0 : f1, t & 31);
      if (on0) den0 = fma(ft, gw[t * r + lane], den0);
      if (on1) den1 = fma(ft, gw[t * r + lane + 32], den1);
    }
    if (on0) f[i * r + lane] = f0 * num[i * r + lane] / (den0 + eps);
    if (on1) f[i * r + lane + 32] = f1 * num[i * r + lane + 32] / (den1 + eps);
  }
}

// r > 64: a warp per row with the old row staged in the warp's shared slice; lane s owns columns
// s, s + 32, ...; g is read through L1 (r² doubles: up to 512 KB); denominators accumulate over t in
// ascending order exactly as above.
__global__ void nmf_update_any_kernel(double* __restrict__ f, const double* __restrict__ num,
                                      const double* __restrict__ g, int64_t rows, int r, double eps) {
  extern __shared__ double frow[];  // [warps][r]
  const int lane = threadIdx.x & 31;
  double* fs = frow + (threadIdx.x >> 5) * r;
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = warp; i < rows; i += nwarps) {
    for (int c = lane; c < r; c += 32) fs[c] = f[i * r + c];
    __syncwarp();
    for (int c = lane; c < r; c += 32) {
      double den = 0.0;
      for (int t = 0; t < r; ++t) den = fma(fs[t], __ldg(g + t * r + c), den);
      f[i * r + c] = fs[c] * num[i * r + c] / (den + eps);
    }
    __syncwarp();
  }
}

cudaError_t launch_nmf_update(double* f, const double* num, const double* g, int64_t rows, int r, double eps,
                              cudaStream_t st, int num_sms) {
  const int grid = grid_for(rows, 256, 8, num_sms);
  if (r > 64 && r <= kNmfStepMaxR) {
    nmf_update_any_kernel<<<grid_for(rows, 8, 8, num_sms), 256, static_cast<size_t>(8) * r * 8, st>>>(f, num, g, rows,
                                                                                                   r, eps);
    FB_LAUNCHED();
    return cudaGetLastError();
  }
  if (r > 16 && r <= 64) {
    nmf_update_wide_kernel<<<grid_for(rows, 8, 8, num_sms), 256, static_cast<size_t>(r) * r * 8, st>>>(f, num, g, rows,
                                                                                                   r, eps);
    FB_LAUNCHED();
    return cudaGetLastError();
  }
  switch (r) {
#define FB_R_CASE(R)                                                     \
  case R:                                                                \
    nmf_update_kernel<R><<<grid, 256, 0, st>>>(f, num, g, rows, eps);   \
    break;
    FB_R_CASE(1) FB_R_CASE(2) FB_R_CASE(3) FB_R_CASE(4) FB_R_CASE(5) FB_R_CASE(6) FB_R_CASE(7) FB_R_CASE(8)
    FB_R_CASE(9) FB_R_CASE(10) FB_R_CASE(11) FB_R_CASE(12) FB_R_CASE(13) FB_R_CASE(14) FB_R_CASE(15) FB_R_CASE(16)
#undef FB_R_CASE
    default:
      return cudaErrorNotSupported;
  }
  FB_LAUNCHED();
  return cudaGetLastError();
}

// g = fᵀf (r × r) of a small d × r factor, upper triangle mirrored exactly (kernel.crossprod).
__global__ void small_gram_kernel(const double* f, int64_t rows, int r, double* g) {
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) {
    const int a = e / r, b = e % r;
    if (a > b) continue;
    double s = 0.0;
    for (int64_t i = 0; i < rows; ++i) s = fma(f[i * r + a], f[i * r + b], s);
    g[a * r + b] = s;
    g[b * r + a] = s;
  }
}

cudaError_t launch_small_gram(const double* f, int64_t rows, int r, double* g, cudaStream_t st) {
  small_gram_kernel<<<1, 256, 0, st>>>(f, rows, r, g);
  FB_LAUNCHED();
  return cudaGetLastError();
}

// trace[it] = sqrt(max(sum_t2 - 2 Σ(ttw∘h) + Σ(cpw∘cph), 0))  (ml.py:314-315)
__global__ void nmf_objective_kernel(const double* sum_t2, const double* ttw, const double* h, int64_t dr,
                                     const double* cpw, const double* cph, int rr, double* trace, int it) {
  __shared__ double a_s[256], b_s[256];
  double a = 0.0, b = 0.0;
  for (int64_t e = threadIdx.x; e < dr; e += blockDim.x) a += ttw[e] * h[e];
  for (int e = threadIdx.x; e < rr; e += blockDim.x) b += cpw[e] * cph[e];
  a_s[threadIdx.x] = a;
  b_s[threadIdx.x] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sa = 0.0, sb = 0.0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      sa += a_s[i];
      sb += b_s[i];
    }
    const double sq = *sum_t2 - 2.0 * sa + sb;
    trace[it] = sqrt(fmax(sq, 0.0));
  }
}

cudaError_t launch_nmf_objective(const double* sum_t2, const double* ttw, const double* h, int64_t dr,
                                 const double* cpw, const double* cph, int rr, double* trace, int it,
                                 cudaStream_t st) {
  nmf_objective_kernel<<<1, 256, 0, st>>>(sum_t2, ttw, h, dr, cpw, cph, rr, trace, it);
  FB_LAUNCHED();
  return cudaGetLastError();
}

}  // namespace fb
