// fb_glm_run.cu — a whole gradient-descent run (logistic_gd ml.py:199-215, linreg_gd
// ml.py:239-254) in ONE cooperative launch, for problems whose factors sit in L2 (c1:
// S 100k×20, R 10k×40 — 24 MB). Per-iteration launches (z-pass, fused S pass, R-side
// reduction, update: fb_glm_step) are latency bound there (~60 µs per iteration even as a
// CUDA graph); here an iteration is two grid barriers:
//   phase 2  t_i = S_i·w_S + Σ_q R_q[fk_q,i]·w_q (the R rows are dotted in place: at c1 the
//            extra 0.2 µs of FP64 work replaces a z-pass and its grid barrier); p_i / loss_i
//            as in fb_ml.cu; Kᵀp scattered into bins_q (atomics, as the per-iteration path);
//            g_S += p_i S_i in registers → per-warp shared partials
//   -- barrier --
//   phase 3  g_q = bins_qᵀ R_q per CTA slice → per-CTA partials; the next iteration's bins
//            zeroed
//   -- barrier --
//   phase 4  every CTA sums the partials in CTA order itself (identical in every CTA,
//            deterministic) and applies w ± α·g to its own shared-memory copy of w.
// bins / partials are double-buffered by iteration parity, so a CTA racing ahead into the
// next iteration never touches buffers a slower CTA still reads. (Four barriers per
// iteration — a separate z-pass and a grid-distributed g — cost ~34 µs per c1 iteration.)
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

#include "fb_kernels.cuh"

namespace cg = cooperative_groups;

namespace fb {

constexpr int kRunThreads = 512;
constexpr int kRunWarps = kRunThreads / 32;
constexpr int kRunRCols = 8;      // R columns per lane loaded together in the S phase
constexpr int kRunMaxCtas = 320;  // co-resident CTAs the phase-4 sum unrolls for (2 per SM × 148 = 296)

struct GlmRunArgs {
  const double* s;
  int64_t n;
  int ds;
  const double* y;
  int mode;       // 0 logistic, 1 least squares
  double alpha;   // signed: +α (logistic), -α (least squares)
  int q;
  const int32_t* fk[kMaxParts];
  const double* r[kMaxParts];
  int64_t nr[kMaxParts];
  int dr[kMaxParts];
  int off[kMaxParts];  // column offset of part q in w
  int d;               // total width
  double* w;           // d (in: initial weights, out: final)
  int iters;
  double* trace;       // iters
  int* diverged;       // first iteration with a non-finite w (-1 otherwise)
  double* bins[2][kMaxParts];
  double* partials[2];  // [gridDim.x][d + 1]
  int lanes;            // lanes per S row (power of two)
  unsigned long long* prof;  // development: CTA 0's globaltimer at each phase end (FB_GLM_PROF)
  int debug;                 // development bisection (FB_GLM_RUN_DEBUG): 1 no Kᵀp atomics
};

FB_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int C>  // S columns per lane (a.lanes lanes per row)
__global__ void __launch_bounds__(kRunThreads, 2) glm_run_kernel(GlmRunArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double smem[];
  double* sw = smem;                          // w (d)
  double* red = smem + ((a.d + 1 + 1) & ~1);  // [kRunWarps][d + 1] warp partials
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t gwarp = static_cast<int64_t>(blockIdx.x) * kRunWarps + warp;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kRunWarps;
  const int L = a.lanes, sub = lane % L, slot = lane / L, rpw = 32 / L;
  const bool logistic = a.mode == 0;
  const int W = a.d + 1;
  for (int j = tid; j < a.d; j += kRunThreads) sw[j] = a.w[j];
  for (int q = 0; q < a.q; ++q)  // iteration 0's bins
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * kRunThreads + tid; j < a.nr[q];
         j += static_cast<int64_t>(gridDim.x) * kRunThreads)
      a.bins[0][q][j] = 0.0;
  grid.sync();

  for (int it = 0; it < a.iters; ++it) {
    const int b = it & 1;
    // ---- phase 2: the S pass, two row steps in flight per warp
    double gs[C];
#pragma unroll
    for (int m = 0; m < C; ++m) gs[m] = 0.0;
    double lacc = 0.0;
    const int64_t stride = nwarps * rpw;
    for (int64_t base = gwarp * rpw; base < a.n; base += 2 * stride) {
      int64_t ii[2];
      bool live[2];
      double sv[2][C], acc[2], zsum[2], yv[2];
      // labels and K_q z_q first (fk -> z is the longest dependent chain), then the S row
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        ii[h] = base + h * stride + slot;
        live[h] = ii[h] < a.n;
        const int64_t i = live[h] ? ii[h] : 0;
        yv[h] = a.y[i];
        zsum[h] = 0.0;
        for (int q = 0; q < a.q; ++q) {  // Σ_q R_q[fk]·w_q in part order (rewrite.py:186-190)
          const double* rrow = a.r[q] + static_cast<int64_t>(a.fk[q][i]) * a.dr[q];
          const double* wq = sw + a.off[q];
          // all of the lane's R loads issued together (a runtime-bound loop issued them one
          // L2 round trip at a time: ~8 µs per row step at c1)
          const int dr = a.dr[q];
          double zq = 0.0;
          for (int c0 = 0; c0 < dr; c0 += kRunRCols * L) {
            double rv[kRunRCols];
#pragma unroll
            for (int m = 0; m < kRunRCols; ++m) {
              const int c = c0 + sub + m * L;
              rv[m] = c < dr ? rrow[c] : 0.0;
            }
#pragma unroll
            for (int m = 0; m < kRunRCols; ++m) {
              const int c = c0 + sub + m * L;
              if (c < dr) zq = fma(rv[m], wq[c], zq);
            }
          }
          for (int o = L >> 1; o > 0; o >>= 1) zq += __shfl_xor_sync(0xffffffffu, zq, o);
          zsum[h] += zq;
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double* srow = a.s + (live[h] ? ii[h] : 0) * a.ds;
        acc[h] = 0.0;
#pragma unroll
        for (int m = 0; m < C; ++m) {
          const int c = sub + m * L;
          const bool on = c < a.ds;
          sv[h][m] = (on && live[h]) ? srow[c] : 0.0;
          acc[h] = fma(sv[h][m], on ? sw[c] : 0.0, acc[h]);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
        for (int o = L >> 1; o > 0; o >>= 1) acc[h] += __shfl_xor_sync(0xffffffffu, acc[h], o);
      double pv[2] = {0.0, 0.0};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (live[h]) {
          const int64_t i = ii[h];
          const double t = acc[h] + zsum[h];
          if (logistic) {
            const double yt = yv[h] * t;
            pv[h] = yv[h] / (1.0 + exp(t));
            if (sub == 0) lacc += log1p(exp(-fabs(yt))) + fmax(-yt, 0.0);
          } else {
            pv[h] = t - yv[h];
            if (sub == 0) lacc += pv[h] * pv[h];
          }
          if (sub == 0 && !(a.debug & 1))
            for (int q = 0; q < a.q; ++q) red_add(a.bins[b][q] + a.fk[q][i], pv[h]);
        }
      }
#pragma unroll
      for (int m = 0; m < C; ++m) gs[m] = fma(pv[1], sv[1][m], fma(pv[0], sv[0][m], gs[m]));
    }
    // fold the row slots of the warp (fixed xor order); each warp's partials to shared memory
#pragma unroll
    for (int m = 0; m < C; ++m)
      for (int o = 16; o >= L; o >>= 1) gs[m] += __shfl_xor_sync(0xffffffffu, gs[m], o);
    lacc = warp_sum(lacc);
    double* wr = red + warp * W;
    if (slot == 0)
#pragma unroll
      for (int m = 0; m < C; ++m) {
        const int c = sub + m * L;
        if (c < a.ds) wr[c] = gs[m];
      }
    if (lane == 0) wr[a.d] = lacc;

    // ---- phase 3 needs every CTA's bins: barrier, then g_q = bins_qᵀ R_q over this CTA's rows
    if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[it * 5 + 2] = gtimer();
    grid.sync();
    for (int q = 0; q < a.q; ++q)  // the next iteration's bins (its atomics start after the next barrier)
      for (int64_t j = static_cast<int64_t>(blockIdx.x) * kRunThreads + tid; j < a.nr[q];
           j += static_cast<int64_t>(gridDim.x) * kRunThreads)
        a.bins[b ^ 1][q][j] = 0.0;
    for (int q = 0; q < a.q; ++q) {
      const double* R = a.r[q];
      const int dr = a.dr[q];
      double gr[4] = {0.0, 0.0, 0.0, 0.0};
      for (int64_t j = gwarp; j < a.nr[q]; j += nwarps) {
        const double bv = a.bins[b][q][j];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int c = lane + 32 * m;
          if (c < dr) gr[m] = fma(bv, R[j * dr + c], gr[m]);
        }
      }
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int c = lane + 32 * m;
        if (c < dr) wr[a.off[q] + c] = gr[m];
      }
    }
    __syncthreads();
    double* part = a.partials[b] + static_cast<size_t>(blockIdx.x) * W;
    for (int c = tid; c < W; c += kRunThreads) {
      double sum = 0.0;
      for (int v = 0; v < kRunWarps; ++v) sum += red[v * W + c];
      part[c] = sum;
    }
    if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[it * 5 + 3] = gtimer();
    grid.sync();

    // ---- phase 4: g (and the objective) in CTA order, summed by every CTA itself (warp per
    // column, lanes strided over CTAs, fixed butterfly: identical in every CTA), then w ± α·g
    {
      const double* P = a.partials[b];
      double* gsm = red;  // the warp partials are consumed: reuse the space for g
      __syncthreads();
      for (int c = warp; c < W; c += kRunWarps) {
        // the lane's partials loaded together, then summed in CTA order
        double pv[kRunMaxCtas / 32];
#pragma unroll
        for (int k = 0; k < kRunMaxCtas / 32; ++k) {
          const int x = lane + 32 * k;
          pv[k] = x < static_cast<int>(gridDim.x) ? P[static_cast<size_t>(x) * W + c] : 0.0;
        }
        double sum = 0.0;
#pragma unroll
        for (int k = 0; k < kRunMaxCtas / 32; ++k) sum += pv[k];
        sum = warp_sum(sum);
        if (lane == 0) gsm[c] = sum;
      }
      __syncthreads();
      __shared__ int bad;
      if (tid == 0) bad = 0;
      __syncthreads();
      for (int c = tid; c < a.d; c += kRunThreads) {
        const double v = sw[c] + a.alpha * gsm[c];
        sw[c] = v;
        if (!isfinite(v)) bad = 1;
      }
      __syncthreads();
      if (blockIdx.x == 0 && tid == 0) {
        a.trace[it] = gsm[a.d];
        if (bad && *a.diverged < 0) *a.diverged = it;
      }
      if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[it * 5 + 4] = gtimer();
    }
  }
  if (blockIdx.x == 0)
    for (int j = tid; j < a.d; j += kRunThreads) a.w[j] = sw[j];
}

bool glm_run_eligible(int64_t n, int ds, int q, const int* dr, int num_sms) {
  if (ds > 256 || q > kMaxParts) return false;
  for (int i = 0; i < q; ++i)
    if (dr[i] > 128) return false;
  if (2 * num_sms > kRunMaxCtas) return false;  // the phase-4 sum is unrolled for <= kRunMaxCtas CTAs
  // factors small enough to stay in L2 between phases
  return static_cast<double>(n) * (ds + 2) * 8 <= 48.0 * 1024 * 1024;
}

size_t glm_run_workspace_bytes(int d, const int64_t* nr, int q, int num_sms) {
  size_t b = 2 * ((static_cast<size_t>(2 * num_sms) * (d + 1) * 8 + 255) & ~size_t(255));
  for (int i = 0; i < q; ++i) b += 2 * ((static_cast<size_t>(nr[i]) * 8 + 255) & ~size_t(255));
  return b + 256;
}

cudaError_t launch_glm_run(const GlmRunIn& in, void* ws, size_t ws_bytes, cudaStream_t st, int num_sms) {
  GlmRunArgs a{};
  a.s = in.s;
  a.n = in.n;
  a.ds = in.ds;
  a.y = in.y;
  a.mode = in.mode;
  a.alpha = in.mode == 0 ? in.alpha : -in.alpha;
  a.q = in.q;
  int off = in.ds;
  for (int i = 0; i < in.q; ++i) {
    a.fk[i] = in.fk[i];
    a.r[i] = in.r[i];
    a.nr[i] = in.nr[i];
    a.dr[i] = in.dr[i];
    a.off[i] = off;
    off += in.dr[i];
  }
  a.d = off;
  a.w = in.w;
  a.iters = in.iters;
  a.trace = in.trace;
  a.diverged = in.diverged;
  int L = 1;  // lanes per S row: the fewest that keep <= 8 columns per lane
  while (L < 32 && in.ds > 8 * L) L *= 2;
  if (in.ds > 8 * L) return cudaErrorNotSupported;
  a.lanes = L;
  const int C = in.ds > 0 ? (in.ds + L - 1) / L : 1;  // d_S = 0 (M:N: every block keyed) runs the C = 1 kernel
  void* kern = nullptr;
  switch (C) {
#define FB_RUN_CASE(N)                                       \
  case N:                                                    \
    kern = reinterpret_cast<void*>(glm_run_kernel<N>);       \
    break;
    FB_RUN_CASE(1) FB_RUN_CASE(2) FB_RUN_CASE(3) FB_RUN_CASE(4) FB_RUN_CASE(5) FB_RUN_CASE(6) FB_RUN_CASE(7)
    FB_RUN_CASE(8)
#undef FB_RUN_CASE
    default:
      return cudaErrorNotSupported;
  }
  const size_t smem = (static_cast<size_t>((a.d + 2) & ~1) + static_cast<size_t>(kRunWarps) * (a.d + 1)) * 8;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRunThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorNotSupported;
  const int grid = num_sms * (per_sm >= 2 ? 2 : 1);  // co-resident (cooperative launch)
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~size_t(255);
    return reinterpret_cast<double*>(r);
  };
  for (int b = 0; b < 2; ++b) a.partials[b] = take(static_cast<size_t>(grid) * (a.d + 1) * 8);
  for (int i = 0; i < in.q; ++i)
    for (int b = 0; b < 2; ++b) a.bins[b][i] = take(static_cast<size_t>(in.nr[i]) * 8);
  if (static_cast<size_t>(p - static_cast<char*>(ws)) > ws_bytes) return cudaErrorInvalidValue;
  static unsigned long long* prof = nullptr;
  if (getenv("FB_GLM_PROF") && in.iters <= 64) {
    if (!prof) cudaMalloc(&prof, 64 * 5 * 8);
    a.prof = prof;
  }
  if (const char* dbg = getenv("FB_GLM_RUN_DEBUG")) a.debug = atoi(dbg);
  void* args[] = {&a};
  e = cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kRunThreads), args, smem, st);
  FB_LAUNCHED();
  if (a.prof) {
    unsigned long long h[64 * 5];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, a.prof, sizeof(unsigned long long) * 5 * in.iters, cudaMemcpyDeviceToHost);
    for (int it = 1; it + 1 < in.iters && it < 5; ++it)
      fprintf(stderr, "[glm_run] it %d: S phase %.1f us, sync+R+partials %.1f, sync+g+update %.1f\n", it,
              (h[it * 5 + 2] - h[(it - 1) * 5 + 4]) / 1e3, (h[it * 5 + 3] - h[it * 5 + 2]) / 1e3,
              (h[it * 5 + 4] - h[it * 5 + 3]) / 1e3);
  }
  return e;
}

}  // namespace fb
