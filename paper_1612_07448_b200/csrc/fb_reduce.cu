// fb_reduce.cu — weighted column reductions Wᵀ·F with a fused Kᵀ scatter.
//
// Replaces, in one streaming pass over a factor matrix F (n × d):
//   * X·S in rmm (rewrite.py:207-209 -> kernel.matmul, kernel.py:103-129),
//   * colSums(S) and counts·R in col_sums (rewrite.py:131-149; kernel.py:185-193),
//   * binsᵀ·R, the (X·K)·R half of rmm,
//   * and, fused into the S pass, the X·K scatter-add of right_compress
//     (indicator.py:130-141, SciPy csc_matvec in the reference).
// out(j, c) = Σ_i w(i, j) · F(i, c).  Each CTA reduces a contiguous row range into
// registers (threads <-> columns), folds its row groups in shared memory, writes one
// partial, and the last CTA to finish sums the partials in CTA order, so the result
// is deterministic for a fixed grid. The scatter uses warp-aggregated atomics
// (__match_any_sync groups equal keys before one RED per group).
#include "fb_kernels.cuh"

namespace fb {

// weight access modes for the staged tile
enum WMode : int { kWOnes = 0, kWInterleaved = 1, kWColumns = 2, kWGlobal = 3 };

struct ColRedDev {
  ColReduce c;
  int wmode;
  int w_stream0;  // first stream index holding weights
  int fk_stream0;
  int svc_scatter;  // the Kᵀ scatter runs on the (otherwise idle) gatherer warps
};

template <int NX>
FB_DEV double wval(const ColRedDev& p, const TileRing& ring, const StreamSet& ss, int stage,
                   int64_t row0, int r, int j) {
  switch (p.wmode) {
    case kWOnes:
      return 1.0;
    case kWInterleaved:
      return reinterpret_cast<const double*>(ring.stage_ptr(stage, ss, p.w_stream0))[r * NX + j];
    case kWColumns:
      return reinterpret_cast<const double*>(ring.stage_ptr(stage, ss, p.w_stream0 + j))[r];
    default:
      return p.c.w[(row0 + r) * p.c.w_rs + j * p.c.w_cs];
  }
}

// Scatter-add of vals[0:NX] into bins[key*NX + j]. With `aggregate` (skewed keys,
// e.g. Zipf), lanes holding the same key are first combined with __match_any_sync so a
// hot bin receives one RED per warp instead of one per row; uniform keys skip it.
template <int NX>
FB_DEV void scatter_add(double* bins, int key, const double (&vals)[NX], bool active, bool aggregate) {
  const unsigned full = 0xffffffffu;
  if (!aggregate) {
    if (active) {
      double* b = bins + static_cast<int64_t>(key) * NX;
#pragma unroll
      for (int j = 0; j < NX; ++j) red_add(b + j, vals[j]);
    }
    return;
  }
  const int lane = lane_id();
  // inactive lanes use a key no active lane can have
  const int k = active ? key : -1 - lane;
  const unsigned peers = __match_any_sync(full, k);
  const int leader = __ffs(peers) - 1;
  double acc[NX];
#pragma unroll
  for (int j = 0; j < NX; ++j) acc[j] = vals[j];
  unsigned rem = (lane == leader) ? (peers & ~(1u << lane)) : 0u;
  while (__any_sync(full, rem != 0)) {
    const int src = rem ? (__ffs(rem) - 1) : lane;
#pragma unroll
    for (int j = 0; j < NX; ++j) {
      const double t = __shfl_sync(full, vals[j], src);
      if (rem) acc[j] += t;
    }
    if (rem) rem &= rem - 1;
  }
  if (active && lane == leader) {
    double* b = bins + static_cast<int64_t>(key) * NX;
#pragma unroll
    for (int j = 0; j < NX; ++j) red_add(b + j, acc[j]);
  }
}

// Skewed keys: the hottest targets of an indicator (IndicatorMatrix.hot_tables) get a
// slot each; rows that hit a hot slot are combined within the warp (__match_any_sync on
// the slot) and added by the group leader into the warp's private shared-memory bins (no
// atomics, no cross-SM contention on one L2 line), flushed once per CTA; other keys RED
// straight to global.
template <int NX>
FB_DEV void scatter_hot(double* bins, double* whot, int key, int slot, const double (&vals)[NX], bool active) {
  const unsigned full = 0xffffffffu;
  const int lane = lane_id();
  const bool hot = active && slot >= 0;
  if (active && !hot) {
    double* b = bins + static_cast<int64_t>(key) * NX;
#pragma unroll
    for (int j = 0; j < NX; ++j) red_add(b + j, vals[j]);
  }
  if (!__any_sync(full, hot)) return;
  const int k = hot ? slot : -1 - lane;  // non-hot lanes get keys no hot lane has
  const unsigned peers = __match_any_sync(full, k);
  const int leader = __ffs(peers) - 1;
  double acc[NX];
#pragma unroll
  for (int j = 0; j < NX; ++j) acc[j] = vals[j];
  unsigned rem = (hot && lane == leader) ? (peers & ~(1u << lane)) : 0u;
  while (__any_sync(full, rem != 0)) {
    const int src = rem ? (__ffs(rem) - 1) : lane;
#pragma unroll
    for (int j = 0; j < NX; ++j) {
      const double t = __shfl_sync(full, vals[j], src);
      if (rem) acc[j] += t;
    }
    if (rem) rem &= rem - 1;
  }
  if (hot && lane == leader) {
    double* b = whot + slot * NX;  // this warp's private bins: plain read-modify-write
#pragma unroll
    for (int j = 0; j < NX; ++j) b[j] += acc[j];
  }
  __syncwarp();
}

// Uniform-FK scatter on the gatherer warps (no keyed gathers in this ring): they wait for
// each stage like the consumers, RED every row's weights into bins[fk] (fire-and-forget
// REDG: the 8 MB c2 bins stay in L2) and release the stage. The consumers keep only the
// column sums, so the scatter costs no consumer issue slots. Tiles the producer could not
// bulk-copy are filled by the consumers after the "full" wait, so for those the keys and
// weights come from global memory.
template <int NX>
FB_DEV void service_scatter(const ColRedDev& p, const TileRing& ring, const StreamSet& ss) {
  const int lane = lane_id();
  const int gw = (static_cast<int>(threadIdx.x) >> 5) - 1;
  int st = 0;
  uint32_t ph = 0;
  const int64_t n = ring.count();
  for (int64_t k = 0; k < n; ++k) {
    const int64_t tile = ring.tile_begin + k;
    const int rows = ring.rows_of(tile);
    const int64_t r0 = tile * ring.tile_rows;
    mbar_wait(&ring.full[st], ph);
    const bool staged = ring.bulk_ok(ss, tile);
    for (int q = 0; q < p.c.nfk; ++q) {
      const int32_t* fkt = reinterpret_cast<const int32_t*>(ring.stage_ptr(st, ss, p.fk_stream0 + q));
      for (int r = gw * 32 + lane; r < rows; r += 32 * kGatherWarps) {
        const int key = staged ? fkt[r] : p.c.fk[q][r0 + r];
        double v[NX];
#pragma unroll
        for (int j = 0; j < NX; ++j)
          v[j] = (staged || p.wmode == kWOnes || p.wmode == kWGlobal)
                     ? wval<NX>(p, ring, ss, st, r0, r, j)
                     : p.c.w[(r0 + r) * p.c.w_rs + j * p.c.w_cs];
        double* b = p.c.bins[q] + static_cast<int64_t>(key) * NX;
#pragma unroll
        for (int j = 0; j < NX; ++j) red_add(b + j, v[j]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&ring.empty[st]);
    if (++st == ring.stages) {
      st = 0;
      ph ^= 1u;
    }
  }
  // the consumers fold their partials into the ring buffers once every stage is read
  asm volatile("bar.arrive 2, %0;\n" ::"n"(kConsumerThreads + 32 * kGatherWarps) : "memory");
}

template <int NX>
__global__ void __launch_bounds__(kRingThreads, 1) colreduce_kernel(ColRedDev p, StreamSet ss, int stages,
                                                                 int tile_rows) {
  extern __shared__ __align__(128) char smem[];
  const int d = p.c.d;
  // warp-private hot bins after the ring: [warp][Σ_q nhot_q][NX]
  double* hotbins = reinterpret_cast<double*>(smem + kRingHeader + static_cast<size_t>(stages) * ss.stage_bytes);
  int hot_off[kMaxParts + 1];
  hot_off[0] = 0;
#pragma unroll
  for (int q = 0; q < kMaxParts; ++q) hot_off[q + 1] = hot_off[q] + (q < p.c.nfk ? p.c.nhot[q] : 0) * NX;
  const int hot_per_warp = hot_off[kMaxParts];
  for (int i = threadIdx.x; i < hot_per_warp * kConsumerWarps; i += blockDim.x) hotbins[i] = 0.0;
  TileRing ring;
  ring.init(smem, stages, tile_rows, p.c.n);
  ring.start(ss, p.svc_scatter ? kGatherWarps : 0);  // __syncthreads: hot bins zeroed
  if (p.svc_scatter && is_gather_warp()) {
    service_scatter<NX>(p, ring, ss);
    return;
  }
  if (ring.service(ss)) return;
  const int tid = consumer_tid();
  const int groups = d > 0 ? kConsumerThreads / d : 0;
  const int col = d > 0 ? tid % d : 0;
  const int grp = d > 0 ? tid / d : 0;
  const bool colthread = grp < groups;

  double acc[NX];
#pragma unroll
  for (int j = 0; j < NX; ++j) acc[j] = 0.0;

  for (int64_t k = 0; k < ring.count(); ++k) {
    const int stage = ring.acquire(ss, k);
    const int64_t tile = ring.tile_begin + k;
    const int rows = ring.rows_of(tile);
    const int64_t r0 = tile * tile_rows;
    if (colthread) {
      const double* A = reinterpret_cast<const double*>(ring.stage_ptr(stage, ss, 0));
      for (int r = grp; r < rows; r += groups) {
        const double a = A[static_cast<size_t>(r) * d + col];
#pragma unroll
        for (int j = 0; j < NX; ++j) acc[j] = fma(wval<NX>(p, ring, ss, stage, r0, r, j), a, acc[j]);
      }
    }
    // fused Kᵀ scatter of the same weights (row-per-thread)
    for (int q = 0; q < (p.svc_scatter ? 0 : p.c.nfk); ++q) {
      const int32_t* fkt = reinterpret_cast<const int32_t*>(ring.stage_ptr(stage, ss, p.fk_stream0 + q));
      for (int rb = 0; rb < rows; rb += kConsumerThreads) {
        const int r = rb + tid;
        const bool live = r < rows;
        double v[NX];
#pragma unroll
        for (int j = 0; j < NX; ++j) v[j] = live ? wval<NX>(p, ring, ss, stage, r0, r, j) : 0.0;
        const int key = live ? fkt[r] : 0;
        if (p.c.nhot[q] > 0) {
          const int slot = live ? p.c.hot_slot[q][key] : -1;
          scatter_hot<NX>(p.c.bins[q], hotbins + (tid >> 5) * hot_per_warp + hot_off[q], key, slot, v, live);
        } else {
          scatter_add<NX>(p.c.bins[q], key, v, live, p.c.aggregate[q] != 0);
        }
      }
    }
    ring.release();
  }

  // flush the hot bins: Σ over warps in warp order, one RED per (slot, column) per CTA
  consumer_sync();
  for (int i = tid; i < hot_per_warp; i += kConsumerThreads) {
    int q = 0;
    while (q + 1 < kMaxParts && i >= hot_off[q + 1]) ++q;
    const int slot = (i - hot_off[q]) / NX, j = (i - hot_off[q]) % NX;
    double s = 0.0;
    for (int w = 0; w < kConsumerWarps; ++w) s += hotbins[w * hot_per_warp + i];
    red_add(p.c.bins[q] + static_cast<int64_t>(p.c.hot_key[q][slot]) * NX + j, s);
  }
  // fold row groups: red[g][j][c] (the ring buffers are idle now — the scatter warps too)
  double* red = reinterpret_cast<double*>(ring.buf);
  if (p.svc_scatter) asm volatile("bar.sync 2, %0;\n" ::"n"(kConsumerThreads + 32 * kGatherWarps) : "memory");
  consumer_sync();
  if (colthread) {
#pragma unroll
    for (int j = 0; j < NX; ++j) red[(static_cast<size_t>(grp) * NX + j) * d + col] = acc[j];
  }
  consumer_sync();
  double* part = p.c.partials + static_cast<size_t>(blockIdx.x) * NX * d;
  for (int e = tid; e < NX * d; e += kConsumerThreads) {
    double s = 0.0;
    for (int g = 0; g < groups; ++g) s += red[static_cast<size_t>(g) * NX * d + e];
    part[e] = s;
  }
  // the last CTA to finish sums the partials in CTA order (deterministic)
  __threadfence();
  __shared__ unsigned int ticket;
  consumer_sync();
  if (tid == 0) ticket = atomicAdd(p.c.counter, 1u);
  consumer_sync();
  if (ticket != gridDim.x - 1) return;
  __threadfence();
  for (int e = tid >> 5; e < NX * d; e += kConsumerWarps) {  // one warp per output
    const double s = warp_sum_strided(p.c.partials + e, gridDim.x, static_cast<size_t>(NX) * d);
    if ((tid & 31) == 0) {
      const int j = e / d, c = e % d;
      p.c.out[j * p.c.o_js + c * p.c.o_cs] = s;
    }
  }
  if (tid == 0) *p.c.counter = 0u;  // ready for the next launch
}

// X·K over FK-sorted rows (the device analogue of SciPy's CSC scatter at indicator.py:130-141):
// bins(key, j) += Σ_{sorted p with key} w(perm[p], j). Each warp owns a contiguous range of
// sorted positions and walks it 32 at a time: a segmented inclusive scan keyed on the
// (sorted, hence contiguous) keys sums each key run, the run still open at lane 31 is carried
// into the next chunk, and only runs that touch the ends of the warp's range use atomics —
// interior runs are complete and are stored plainly (bins are zeroed first). A hot Zipf key
// costs one atomic per warp range it spans.
template <int NX>
__global__ void segsum_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ keys, int64_t n,
                              const double* __restrict__ w, int64_t w_rs, int64_t w_cs, double* __restrict__ bins) {
  const unsigned full = 0xffffffffu;
  const int lane = lane_id();
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int64_t wid = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t lo = n * wid / nwarps, hi = n * (wid + 1) / nwarps;
  int ckey = -1;        // run open at the end of the previous chunk (valid in every lane)
  bool cfirst = true;   // no run of this warp's range has closed yet: the open / first run may
                        // have started in the previous warp's range (atomics)
  double csum[NX];
#pragma unroll
  for (int j = 0; j < NX; ++j) csum[j] = 0.0;
  for (int64_t base = lo; base < hi; base += 32) {
    const int64_t p = base + lane;
    const bool live = p < hi;
    const int key = live ? keys[p] : -1 - lane;
    const int64_t row = live ? perm[p] : 0;
    double v[NX];
#pragma unroll
    for (int j = 0; j < NX; ++j) v[j] = live ? w[row * w_rs + j * w_cs] : 0.0;
    const int first_key = __shfl_sync(full, key, 0);
    if (ckey >= 0 && first_key != ckey) {
      // the carried run ended exactly at the chunk boundary
      if (lane == 0) {
        double* b = bins + static_cast<int64_t>(ckey) * NX;
#pragma unroll
        for (int j = 0; j < NX; ++j) {
          if (cfirst)
            red_add(b + j, csum[j]);
          else
            b[j] = csum[j];
        }
      }
      cfirst = false;
    } else if (ckey >= 0 && lane == 0) {
#pragma unroll
      for (int j = 0; j < NX; ++j) v[j] += csum[j];  // the carried run continues
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int kk = __shfl_up_sync(full, key, off);
      const bool same = lane >= off && kk == key;
#pragma unroll
      for (int j = 0; j < NX; ++j) {
        const double t = __shfl_up_sync(full, v[j], off);
        if (same) v[j] += t;
      }
    }
    const int last_lane = (hi - 1 - base) < 31 ? static_cast<int>(hi - 1 - base) : 31;
    const int next = __shfl_down_sync(full, key, 1);
    const bool seg_end = live && lane < last_lane && next != key;  // a run that ends inside the chunk
    if (seg_end) {
      double* b = bins + static_cast<int64_t>(key) * NX;
      if (key == first_key && cfirst) {
#pragma unroll
        for (int j = 0; j < NX; ++j) red_add(b + j, v[j]);
      } else {
#pragma unroll
        for (int j = 0; j < NX; ++j) b[j] = v[j];  // complete run inside the range
      }
    }
    if (__any_sync(full, seg_end)) cfirst = false;
    ckey = __shfl_sync(full, key, last_lane);
#pragma unroll
    for (int j = 0; j < NX; ++j) csum[j] = __shfl_sync(full, v[j], last_lane);
  }
  // the last open run may continue into the next warp's range
  if (lane == 0 && ckey >= 0) {
    double* b = bins + static_cast<int64_t>(ckey) * NX;
#pragma unroll
    for (int j = 0; j < NX; ++j) red_add(b + j, csum[j]);
  }
}

cudaError_t launch_segsum(const int32_t* perm, const int32_t* keys, int64_t n, const double* w, int64_t w_rs,
                          int64_t w_cs, int nx, double* bins, int64_t n_bins, cudaStream_t st, int num_sms) {
  cudaError_t e = cudaMemsetAsync(bins, 0, static_cast<size_t>(n_bins) * nx * sizeof(double), st);
  if (e != cudaSuccess || n <= 0) return e;
  const int grid = grid_for((n + 255) / 256, 8, 8, num_sms);  // >= 256 sorted positions per warp
  switch (nx) {
#define FB_SEG_CASE(N)                                                                   \
  case N:                                                                                \
    segsum_kernel<N><<<grid, 256, 0, st>>>(perm, keys, n, w, w_rs, w_cs, bins);          \
    break;
    FB_SEG_CASE(1) FB_SEG_CASE(2) FB_SEG_CASE(3) FB_SEG_CASE(4) FB_SEG_CASE(5) FB_SEG_CASE(6) FB_SEG_CASE(7)
    FB_SEG_CASE(8) FB_SEG_CASE(10) FB_SEG_CASE(12) FB_SEG_CASE(16)
#undef FB_SEG_CASE
    default:
      return cudaErrorNotSupported;
  }
  FB_LAUNCHED();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ host side
static int colred_tile_rows(uint32_t row_bytes) {
  // ~40 KB of staged rows (all streams) per stage, a multiple of 4 rows in [32, 512]
  int rows = row_bytes > 0 ? static_cast<int>((44u * 1024u) / row_bytes) : 512;
  if (rows > 512) rows = 512;
  if (rows < 32) rows = 32;
  return rows & ~3;
}

size_t colreduce_workspace_doubles(int64_t n, int d, int nx, int num_sms) {
  (void)n;
  return static_cast<size_t>(num_sms) * 2 * static_cast<size_t>(nx) * (d > 0 ? d : 1);
}

template <int NX>
static cudaError_t launch_colreduce_nx(const ColReduce& c, cudaStream_t st, int num_sms) {
  ColRedDev p{};
  p.c = c;
  StreamSet ss{};
  int ns = 0;
  ss.base[ns] = reinterpret_cast<const char*>(c.a);
  ss.row_bytes[ns++] = static_cast<uint32_t>(c.d) * 8u;
  if (c.w == nullptr) {
    p.wmode = kWOnes;
  } else if (c.w_cs == 1 && c.w_rs == NX) {
    p.wmode = kWInterleaved;
    p.w_stream0 = ns;
    ss.base[ns] = reinterpret_cast<const char*>(c.w);
    ss.row_bytes[ns++] = NX * 8u;
  } else if (NX + 1 < kMaxStreams && c.w_rs == 1 && NX + 1 + c.nfk <= kMaxStreams) {
    p.wmode = kWColumns;
    p.w_stream0 = ns;
    if constexpr (NX + 1 < kMaxStreams) {
      for (int j = 0; j < NX; ++j) {
        ss.base[ns] = reinterpret_cast<const char*>(c.w + j * c.w_cs);
        ss.row_bytes[ns++] = 8u;
      }
    }
  } else {
    p.wmode = kWGlobal;
  }
  p.fk_stream0 = ns;
  p.svc_scatter = c.nfk > 0 ? 1 : 0;
  for (int q = 0; q < c.nfk; ++q)
    if (c.nhot[q] > 0 || c.aggregate[q]) p.svc_scatter = 0;  // skewed keys: consumer path
  if (const char* e = getenv("FB_SVC_SCATTER")) p.svc_scatter = p.svc_scatter && e[0] == '1';
  for (int q = 0; q < c.nfk; ++q) {
    ss.base[ns] = reinterpret_cast<const char*>(c.fk[q]);
    ss.row_bytes[ns++] = 4u;
  }
  ss.count = ns;
  uint32_t row_bytes = 0;
  for (int i = 0; i < ns; ++i) row_bytes += ss.row_bytes[i];
  const int tile_rows = colred_tile_rows(row_bytes);
  stream_layout(ss, tile_rows, c.n);
  const size_t red_bytes = static_cast<size_t>(kConsumerThreads) * NX * 8;
  int stages = 4;
  size_t smem = kRingHeader + static_cast<size_t>(stages) * ss.stage_bytes;
  if (smem > 200 * 1024) {
    stages = 3;
    smem = kRingHeader + static_cast<size_t>(stages) * ss.stage_bytes;
  }
  if (smem < kRingHeader + red_bytes + 1024) smem = kRingHeader + red_bytes + 1024;
  size_t hot = 0;
  for (int q = 0; q < c.nfk; ++q) hot += static_cast<size_t>(c.nhot[q]) * NX;
  const size_t ring_end = kRingHeader + static_cast<size_t>(stages) * ss.stage_bytes;
  if (smem < ring_end + hot * kConsumerWarps * 8) smem = ring_end + hot * kConsumerWarps * 8;
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  auto kern = colreduce_kernel<NX>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int per_sm = static_cast<int>((227 * 1024) / (smem + 1024));
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 2) per_sm = 2;
  const int64_t ntiles = (c.n + tile_rows - 1) / tile_rows;
  const int grid = grid_for(ntiles, 1, per_sm, num_sms);
  for (int q = 0; q < c.nfk; ++q) {
    e = cudaMemsetAsync(c.bins[q], 0, static_cast<size_t>(c.nbins[q]) * NX * sizeof(double), st);
    if (e != cudaSuccess) return e;
  }
  e = cudaMemsetAsync(c.counter, 0, sizeof(unsigned int), st);
  if (e != cudaSuccess) return e;
  kern<<<grid, kRingThreads, smem, st>>>(p, ss, stages, tile_rows);
  FB_LAUNCHED();
  return cudaGetLastError();
}

cudaError_t launch_colreduce(const ColReduce& c, cudaStream_t st, int num_sms) {
  if (c.d > 256) return cudaErrorNotSupported;
  switch (c.nx) {
#define FB_NX_CASE(N) \
  case N:             \
    return launch_colreduce_nx<N>(c, st, num_sms);
    FB_NX_CASE(1)
    FB_NX_CASE(2)
    FB_NX_CASE(3)
    FB_NX_CASE(4)
    FB_NX_CASE(5)
    FB_NX_CASE(6)
    FB_NX_CASE(7)
    FB_NX_CASE(8)
    FB_NX_CASE(10)
    FB_NX_CASE(12)
    FB_NX_CASE(16)
#undef FB_NX_CASE
    default:
      return cudaErrorNotSupported;
  }
}

}  // namespace fb
