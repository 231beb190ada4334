// fb_crossprod.cu — factorized crossprod TᵀT for T = [S, K·R] (rewrite.py:245-298,
// Algorithm 2 of the paper), on the FP64 tensor cores.
//
//   TᵀT = [[ SᵀS,        (KᵀS)ᵀR       ],
//          [ Rᵀ(KᵀS),    Rᵀ diag(c) R  ]]        c = colSums(K) (indicator.py:61-66)
//
// Two streaming passes, each a DMMA "gram" over row tiles staged by the bulk-copy ring:
//   S pass  rows of S in FK-sorted order (a cached stable permutation; the GPU analogue of
//           the reference's _csr_t, indicator.py:78-86). Every tile feeds (a) the upper-
//           triangle 8×8 tiles of SᵀS and (b) the segmented column sums B = KᵀS: each of d_S
//           threads walks the sorted rows and emits one row of B per key run, so S is read
//           once and KᵀS needs no atomics. Runs cut by a CTA boundary go to a carry table
//           that a one-CTA fixup combines in CTA order (deterministic).
//   R pass  rows of R with B and c alongside: the upper triangle of Rᵀ diag(c) R (W frags
//           scaled by c on the fly) and the full RᵀB block.
// Each warp owns a "job": up to kMaxSlots output tiles over at most two A column blocks
// (block rows i and nb-1-i pair up so every job carries the same DMMA count). Jobs that
// exceed one CTA's eight consumer warps are spread over gridDim.y. Per-CTA partial tiles
// are summed in a fixed order by cp_reduce_kernel, which also writes the exact mirror
// (lower = upperᵀ, rewrite.py:298 / kernel.py:132-135).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "fb_kernels.cuh"

namespace fb {

constexpr int kMaxSlots = 16;
constexpr int kMaxJobGroups = 8;

// slot code: bits 0-7 W column block, bit 8 use A block a1, bit 9 W from region 1,
// bit 10 scale W by the per-row counts
struct GramJob {
  int a0, a1;
  int nslots;
  uint16_t code[kMaxSlots];
  uint16_t tile[kMaxSlots];  // output tile id (partials layout)
};

struct GramJobs {
  GramJob job[kMaxJobGroups][kConsumerWarps];
  int njobs[kMaxJobGroups];
  int row_split;  // warps sharing one job (k-steps interleaved); uniform over jobs
  int ntiles;     // tiles produced by this pass
};

struct GramRegion {
  int pitch;     // doubles per smem row
  int stream;    // ring stream index
  int width;     // valid columns
};

struct GramArgs {
  int64_t n;             // rows streamed
  GramRegion reg[2];     // region 0 = A (and W when bit 9 clear), region 1 = W extra (B)
  int cnt_stream;        // stream holding per-row f64 counts (-1: none)
  double* partials;      // [gridDim.x * row_split][ntiles][64]
  // S pass only: segmented KᵀS
  int seg;               // 1: run the segmented walk (stream 1 = sorted keys, int32)
  int seg_cols;          // d_S
  double* bins;          // n_R × d_S
  int64_t n_bins;
  int* carry_key;        // [gridDim.x][2]
  double* carry_val;     // [gridDim.x][2][d_S]
};

// One tile's worth of DMMA work for this warp's job.
template <int SLOTS>
FB_DEV void gram_tile(const GramJob& jb, const uint32_t (&codes)[SLOTS / 2], const TileRing& ring, const StreamSet& ss,
                      const GramArgs& a, int stage, int rows, int split, int nsplit, double (&acc)[SLOTS][2]) {
  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  const double* R0 = reinterpret_cast<const double*>(ring.stage_ptr(stage, ss, a.reg[0].stream));
  const double* R1 = reinterpret_cast<const double*>(ring.stage_ptr(stage, ss, a.reg[1].stream));
  const double* cnt = a.cnt_stream >= 0 ? reinterpret_cast<const double*>(ring.stage_ptr(stage, ss, a.cnt_stream))
                                        : nullptr;
  const int p0 = a.reg[0].pitch, p1 = a.reg[1].pitch;
  const int ao0 = 8 * jb.a0 + g, ao1 = 8 * jb.a1 + g;
  __syncwarp();  // mma.sync.aligned needs the whole warp converged (after the barrier spin)
  for (int k0 = 4 * split; k0 < rows; k0 += 4 * nsplit) {
    const int k = k0 + t;
    const bool live = k < rows;
    const int kr = live ? k : 0;
    const double a0 = live ? R0[kr * p0 + ao0] : 0.0;
    const double a1 = live ? R0[kr * p0 + ao1] : 0.0;
    const double c = (cnt && live) ? cnt[kr] : 1.0;
    const double* w0 = R0 + kr * p0 + g;
    const double* w1 = R1 + kr * p1 + g;
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      if (s < jb.nslots) {
        const int code = (codes[s / 2] >> (16 * (s & 1))) & 0xffff;
        const int wb = 8 * (code & 0xff);
        double w = (code & 0x200) ? w1[wb] : w0[wb];
        if (code & 0x400) w *= c;
        if (!live) w = 0.0;
        dmma_8x8x4(acc[s][0], acc[s][1], (code & 0x100) ? a1 : a0, w);
      }
    }
  }
}

template <int SLOTS>
FB_DEV void gram_store(const GramJob& jb, const GramArgs& a, int pidx, int ntiles, const double (&acc)[SLOTS][2]) {
  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    if (s < jb.nslots) {
      double* dst = a.partials + (static_cast<size_t>(pidx) * ntiles + jb.tile[s]) * 64 + g * 8 + 2 * t;
      dst[0] = acc[s][0];
      dst[1] = acc[s][1];
    }
  }
}

// Segmented column sums over FK-sorted rows (thread c < d_S owns column c).
struct SegState {
  int key;     // current run key (-1: none yet)
  double sum;
  bool first;  // the current run is this CTA's first (may continue from the previous CTA)
};

FB_DEV void seg_flush(const GramArgs& a, SegState& st, int col, int slot) {
  if (st.key < 0) return;
  if (st.first) {
    a.carry_val[(static_cast<size_t>(blockIdx.x) * 2 + slot) * a.seg_cols + col] = st.sum;
    if (col == 0) a.carry_key[blockIdx.x * 2 + slot] = st.key;
  } else {
    a.bins[static_cast<int64_t>(st.key) * a.seg_cols + col] = st.sum;
  }
}

template <int SLOTS>
__global__ void __launch_bounds__(kRingThreads, 1) cp_gram_kernel(const __grid_constant__ GramJobs jobs, GramArgs a,
                                                               StreamSet ss, int stages, int tile_rows) {
  extern __shared__ __align__(128) char smem[];
  TileRing ring;
  ring.init(smem, stages, tile_rows, a.n);
  ring.start(ss);
  if (ring.service(ss)) return;
  const int warp = consumer_warp();
  const int grp = blockIdx.y;
  const int nsplit = jobs.row_split;
  const int jidx = warp / nsplit, split = warp % nsplit;
  const bool has_job = jidx < jobs.njobs[grp];
  const GramJob& jb = jobs.job[grp][has_job ? jidx : 0];
  double acc[SLOTS][2];
  uint32_t codes[SLOTS / 2];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) acc[s][0] = acc[s][1] = 0.0;
#pragma unroll
  for (int s = 0; s < SLOTS / 2; ++s)
    codes[s] = (2 * s < jb.nslots ? jb.code[2 * s] : 0u) | ((2 * s + 1 < jb.nslots ? jb.code[2 * s + 1] : 0u) << 16);

  const int tid = consumer_tid();
  const bool seg = a.seg && grp == 0 && tid < a.seg_cols;
  SegState sst{-1, 0.0, true};

  for (int64_t kt = 0; kt < ring.count(); ++kt) {
    const int stage = ring.acquire(ss, kt);
    const int rows = ring.rows_of(ring.tile_begin + kt);
    if (has_job) gram_tile<SLOTS>(jb, codes, ring, ss, a, stage, rows, split, nsplit, acc);
    if (seg) {
      const double* S = reinterpret_cast<const double*>(ring.stage_ptr(stage, ss, 0));
      const int32_t* keys = reinterpret_cast<const int32_t*>(ring.stage_ptr(stage, ss, 1));
      const int p = a.reg[0].pitch;
      for (int r = 0; r < rows; ++r) {
        const int key = keys[r];
        const double v = S[r * p + tid];
        if (key != sst.key) {
          seg_flush(a, sst, tid, 0);
          if (sst.key >= 0) {
            sst.first = false;
            for (int z = sst.key + 1; z < key; ++z) a.bins[static_cast<int64_t>(z) * a.seg_cols + tid] = 0.0;
          }
          sst.key = key;
          sst.sum = v;
        } else {
          sst.sum += v;
        }
      }
    }
    ring.release();
  }
  if (seg) {
    // the last run may continue into the next CTA: it goes to carry slot 1 (slot 0 if it
    // is also the first run, in which case slot 1 is marked empty)
    if (sst.first) {
      seg_flush(a, sst, tid, 0);
      if (tid == 0) a.carry_key[blockIdx.x * 2 + 1] = -1;
    } else {
      a.carry_val[(static_cast<size_t>(blockIdx.x) * 2 + 1) * a.seg_cols + tid] = sst.sum;
      if (tid == 0) a.carry_key[blockIdx.x * 2 + 1] = sst.key;
    }
    if (sst.key < 0 && tid == 0) {  // empty CTA
      a.carry_key[blockIdx.x * 2] = -1;
      a.carry_key[blockIdx.x * 2 + 1] = -1;
    }
  }
  if (has_job) gram_store<SLOTS>(jb, a, blockIdx.x * nsplit + split, jobs.ntiles, acc);
}

// Combine the CTA-boundary runs in CTA order and zero the bins no row maps to at the
// CTA seams and at both ends (one CTA; thread c owns column c). Carry slots come in
// (first run, last run) pairs per CTA; interior gaps were zeroed by the walker.
__global__ void cp_carry_fixup_kernel(const int* carry_key, const double* carry_val, int nslots, int cols,
                                      double* bins, int64_t n_bins) {
  const int c = threadIdx.x;
  if (c >= cols) return;
  int cur = -1, prev = -1;
  double sum = 0.0;
  for (int i = 0; i < nslots; ++i) {
    const int k = carry_key[i];
    if (k < 0) continue;
    const double v = carry_val[static_cast<size_t>(i) * cols + c];
    if (k == cur) {
      sum += v;
      continue;
    }
    if (cur >= 0) bins[static_cast<int64_t>(cur) * cols + c] = sum;
    if ((i & 1) == 0)
      for (int z = prev + 1; z < k; ++z) bins[static_cast<int64_t>(z) * cols + c] = 0.0;
    cur = k;
    sum = v;
    prev = k;
  }
  if (cur >= 0) bins[static_cast<int64_t>(cur) * cols + c] = sum;
  for (int64_t z = prev + 1; z < n_bins; ++z) bins[z * cols + c] = 0.0;
}

// Final assembly: out tile element = Σ_p partials[p][tile][e] in p order; written to the
// upper-triangle position and mirrored exactly.
struct TileMap {
  int row0, col0;   // global row/col of the tile's (0,0) element (before mirroring)
  int nrow, ncol;   // valid extent
  int diag;         // 1: a diagonal tile (keep only row <= col, mirror)
};

constexpr int kMaxTiles = 1024;
struct TileMaps {
  TileMap m[kMaxTiles];
};

__global__ void cp_reduce_kernel(const double* partials, int nparts, int ntiles, const __grid_constant__ TileMaps maps,
                                 double* out, int64_t ldo) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e >= static_cast<int64_t>(ntiles) * 64) return;
  const int tile = static_cast<int>(e / 64), el = static_cast<int>(e % 64);
  const TileMap m = maps.m[tile];
  const int a = el / 8, b = el % 8;
  if (a >= m.nrow || b >= m.ncol) return;
  const int r = m.row0 + a, c = m.col0 + b;
  if (m.diag && r > c) return;
  double s = 0.0;
  const double* p = partials + e;
  const size_t stride = static_cast<size_t>(ntiles) * 64;
#pragma unroll 8
  for (int i = 0; i < nparts; ++i) s += p[i * stride];
  out[r * ldo + c] = s;
  out[c * ldo + r] = s;
}

// ------------------------------------------------------------------ host side
namespace {

struct Tile {
  int a, w;  // A block, W block (W blocks >= na refer to region 1 block w - na)
};

// Build jobs: pair A block rows (i, na-1-i); each pair's tiles are the triangle part
// (w in [i, na) when `tri`, else all of [0, na) when region 0 is a full W) plus every
// region-1 block; chunks of at most `slots` tiles.
bool build_jobs(int na, bool tri_region0, bool use_region0, int nb1, bool scale_region0, int slots, int tile_base,
                GramJobs& J, std::vector<TileMap>& maps, int row_off_a, int col_off_w0, int col_off_w1, int da,
                int dw1) {
  std::vector<std::vector<Tile>> jobs;
  for (int i = 0; i <= (na - 1) / 2; ++i) {
    const int j = na - 1 - i;
    std::vector<Tile> tl;
    const int rows_[2] = {i, j};
    const int nrow = (i == j) ? 1 : 2;
    for (int rr = 0; rr < nrow; ++rr) {
      const int ia = rows_[rr];
      if (use_region0)
        for (int w = tri_region0 ? ia : 0; w < na; ++w) tl.push_back({ia, w});
      for (int w = 0; w < nb1; ++w) tl.push_back({ia, na + w});
    }
    for (size_t s0 = 0; s0 < tl.size(); s0 += slots) {
      std::vector<Tile> chunk(tl.begin() + s0, tl.begin() + std::min(tl.size(), s0 + slots));
      jobs.push_back(chunk);
    }
  }
  const int njobs = static_cast<int>(jobs.size());
  const int ngroups = (njobs + kConsumerWarps - 1) / kConsumerWarps;
  if (ngroups > kMaxJobGroups) return false;
  J = GramJobs{};
  J.row_split = njobs >= kConsumerWarps ? 1 : kConsumerWarps / njobs;
  int tid = tile_base;
  for (int gI = 0; gI < ngroups; ++gI) {
    const int in_group = std::min(kConsumerWarps, njobs - gI * kConsumerWarps);
    J.njobs[gI] = in_group;
  }
  for (int q = 0; q < njobs; ++q) {
    GramJob& jb = J.job[q / kConsumerWarps][q % kConsumerWarps];
    const auto& tl = jobs[q];
    jb.a0 = tl[0].a;
    jb.a1 = tl[0].a;
    for (const Tile& t : tl)
      if (t.a != jb.a0) jb.a1 = t.a;
    jb.nslots = static_cast<int>(tl.size());
    for (int s = 0; s < jb.nslots; ++s) {
      const Tile& t = tl[s];
      int code = 0;
      if (t.w < na) {
        code = t.w | (scale_region0 ? 0x400 : 0);
      } else {
        code = (t.w - na) | 0x200;
      }
      if (t.a != jb.a0) code |= 0x100;
      jb.code[s] = static_cast<uint16_t>(code);
      jb.tile[s] = static_cast<uint16_t>(tid - tile_base);
      TileMap m{};
      m.row0 = row_off_a + 8 * t.a;
      m.nrow = std::min(8, da - 8 * t.a);
      if (t.w < na) {
        m.col0 = col_off_w0 + 8 * t.w;
        m.ncol = std::min(8, da - 8 * t.w);
        m.diag = (t.w == t.a) ? 1 : 0;
      } else {
        m.col0 = col_off_w1 + 8 * (t.w - na);
        m.ncol = std::min(8, dw1 - 8 * (t.w - na));
        m.diag = 0;
      }
      maps.push_back(m);
      ++tid;
    }
  }
  J.ntiles = tid - tile_base;
  return true;
}

}  // namespace

size_t fk_sort_workspace_bytes(int64_t n) {
  size_t temp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                  static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                  static_cast<int>(n));
  return ((temp + 255) & ~size_t(255)) + ((static_cast<size_t>(n) * 4 + 255) & ~size_t(255));
}

__global__ void iota_kernel(int32_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = static_cast<int32_t>(i);
}

cudaError_t launch_fk_sort(const int32_t* fk, int64_t n, int64_t n_r, int32_t* perm, int32_t* fk_sorted, void* ws,
                           size_t ws_bytes, cudaStream_t st, int num_sms) {
  if (n <= 0) return cudaSuccess;
  if (n > INT32_MAX) return cudaErrorNotSupported;
  size_t temp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp, fk, fk_sorted, static_cast<const int32_t*>(nullptr), perm,
                                  static_cast<int>(n));
  const size_t tb = (temp + 255) & ~size_t(255);
  if (ws_bytes < tb + static_cast<size_t>(n) * 4) return cudaErrorInvalidValue;
  int32_t* iota = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + tb);
  iota_kernel<<<num_sms * 4, 256, 0, st>>>(iota, n);
  FB_LAUNCHED();
  int end_bit = 1;
  while (end_bit < 31 && (int64_t(1) << end_bit) < n_r) ++end_bit;
  // stable LSD radix sort: ties keep ascending row order (np.argsort kind="stable")
  cudaError_t e = cub::DeviceRadixSort::SortPairs(ws, temp, fk, fk_sorted, iota, perm, static_cast<int>(n), 0,
                                                  end_bit, st);
  FB_LAUNCHED();
  return e;
}

static size_t al(size_t b) { return (b + 255) & ~size_t(255); }

size_t crossprod_workspace_bytes(int64_t n_s, int d_s, int64_t n_r, int d_r, int q, int num_sms) {
  size_t b = 0;
  const int nbs = (d_s + 7) / 8, nbr = (d_r + 7) / 8;
  const size_t st_tiles = static_cast<size_t>(nbs) * (nbs + 1) / 2;
  const size_t rt_tiles = static_cast<size_t>(nbr) * (nbr + 1) / 2 + static_cast<size_t>(nbr) * nbs;
  b += al(static_cast<size_t>(num_sms) * kConsumerWarps * st_tiles * 64 * 8);  // S partials
  b += al(static_cast<size_t>(num_sms) * kConsumerWarps * rt_tiles * 64 * 8);  // R partials
  if (q > 0) {
    b += al(static_cast<size_t>(n_r) * d_s * 8);                   // B = KᵀS
    b += al(static_cast<size_t>(num_sms) * 2 * sizeof(int));       // carry keys
    b += al(static_cast<size_t>(num_sms) * 2 * (d_s > 0 ? d_s : 1) * 8);  // carry values
  }
  (void)n_s;
  return b + 1024;
}

// One wave: job groups share the SMs (each group re-reads its row range).
static int gram_grid(int64_t n, int tile_rows, int ngroups, int num_sms) {
  const int64_t ntiles = (n + tile_rows - 1) / tile_rows;
  const int per = ngroups > 1 ? std::max(1, num_sms / ngroups) : num_sms;
  return grid_for(ntiles, 1, 1, per);
}

static int njob_groups(const GramJobs& J) {
  int ngroups = 0;
  for (int gI = 0; gI < kMaxJobGroups; ++gI)
    if (J.njobs[gI] > 0) ngroups = gI + 1;
  return ngroups;
}

template <class Setup>
static cudaError_t run_gram(GramJobs& J, GramArgs& a, StreamSet& ss, int tile_rows, cudaStream_t st, int num_sms,
                            Setup) {
  stream_layout(ss, tile_rows, a.n);
  int stages = static_cast<int>((200 * 1024 - kRingHeader - 256) / ss.stage_bytes);
  if (stages > 6) stages = 6;
  if (stages < 2) return cudaErrorNotSupported;
  // + slack: fragment loads of the last 8-column block read up to 7 doubles past a row, so
  // the last row of the last stage must not sit at the end of the allocation
  const size_t smem = kRingHeader + static_cast<size_t>(stages) * ss.stage_bytes + 256;
  int ngroups = 0;
  for (int gI = 0; gI < kMaxJobGroups; ++gI)
    if (J.njobs[gI] > 0) ngroups = gI + 1;
  int maxslots = 0;
  for (int gI = 0; gI < ngroups; ++gI)
    for (int w = 0; w < J.njobs[gI]; ++w) maxslots = std::max(maxslots, J.job[gI][w].nslots);
  if (maxslots > kMaxSlots) return cudaErrorNotSupported;
  dim3 gdim(gram_grid(a.n, tile_rows, ngroups, num_sms), ngroups > 0 ? ngroups : 1);
  cudaError_t e =
      cudaFuncSetAttribute(cp_gram_kernel<kMaxSlots>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  if (const char* dbg = getenv("FB_CP_DEBUG")) {  // development bisection switches
    const int bits = atoi(dbg);
    if (bits & 1) a.seg = 0;
    if (bits & 2) ss.bulk_full = ss.bulk_last = false;
    if (bits & 4)
      for (int gI = 0; gI < kMaxJobGroups; ++gI) J.njobs[gI] = 0;
  }
  if (getenv("FB_DEBUG_SYNC"))
    fprintf(stderr, "[fb] gram pass n=%lld tile_rows=%d stages=%d grid=%dx%d split=%d seg=%d bulk=%d/%d gidx=%d\n",
            (long long)a.n, tile_rows, stages, gdim.x, gdim.y, J.row_split, a.seg, (int)ss.bulk_full,
            (int)ss.bulk_last, ss.gidx != nullptr);
  cp_gram_kernel<kMaxSlots><<<gdim, kRingThreads, smem, st>>>(J, a, ss, stages, tile_rows);
  FB_LAUNCHED();
  return cudaGetLastError();
}

static int gram_tile_rows(uint32_t row_bytes, int row_split, bool gather) {
  int rows = static_cast<int>((32u * 1024u) / (row_bytes > 0 ? row_bytes : 1));
  const int unit = 4 * row_split;
  if (rows > (gather ? 128 : 256)) rows = gather ? 128 : 256;
  rows = (rows / unit) * unit;
  if (rows < unit) rows = unit;
  return rows;
}

cudaError_t launch_crossprod(const CrossArgs& c, void* ws, size_t ws_bytes, cudaStream_t st, int num_sms) {
  const int d = c.d_s + c.d_r;
  const int nbs = (c.d_s + 7) / 8, nbr = (c.d_r + 7) / 8;
  const int q = c.r ? 1 : 0;
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t b) {
    char* r = p;
    p += al(b);
    return r;
  };
  const size_t st_tiles = static_cast<size_t>(nbs) * (nbs + 1) / 2;
  const size_t rt_tiles = static_cast<size_t>(nbr) * (nbr + 1) / 2 + static_cast<size_t>(nbr) * nbs;
  double* sp = reinterpret_cast<double*>(take(static_cast<size_t>(num_sms) * kConsumerWarps * st_tiles * 64 * 8));
  double* rp = reinterpret_cast<double*>(take(static_cast<size_t>(num_sms) * kConsumerWarps * rt_tiles * 64 * 8));
  double* bins = nullptr;
  int* ckey = nullptr;
  double* cval = nullptr;
  if (q) {
    bins = reinterpret_cast<double*>(take(static_cast<size_t>(c.n_r) * c.d_s * 8));
    ckey = reinterpret_cast<int*>(take(static_cast<size_t>(num_sms) * 2 * sizeof(int)));
    cval = reinterpret_cast<double*>(take(static_cast<size_t>(num_sms) * 2 * (c.d_s > 0 ? c.d_s : 1) * 8));
  }
  if (static_cast<size_t>(p - static_cast<char*>(ws)) > ws_bytes) return cudaErrorInvalidValue;

  std::vector<TileMap> maps;
  cudaError_t e = cudaMemsetAsync(c.out, 0, static_cast<size_t>(d) * d * 8, st);
  if (e != cudaSuccess) return e;

  // ---- S pass: SᵀS (+ KᵀS when q = 1)
  int s_parts = 0;
  GramJobs JS{};
  if (c.d_s > 0 && c.n_s > 0) {
    if (!build_jobs(nbs, true, true, 0, false, kMaxSlots, 0, JS, maps, 0, 0, 0, c.d_s, 0))
      return cudaErrorNotSupported;
    GramArgs a{};
    a.n = c.n_s;
    a.reg[0] = {c.d_s, 0, c.d_s};
    a.reg[1] = a.reg[0];
    a.cnt_stream = -1;
    a.partials = sp;
    StreamSet ss{};
    ss.base[0] = reinterpret_cast<const char*>(c.s);
    ss.row_bytes[0] = static_cast<uint32_t>(c.d_s) * 8u;
    ss.count = 1;
    if (q) {
      ss.gidx = c.perm;
      ss.base[1] = reinterpret_cast<const char*>(c.fk_sorted);
      ss.row_bytes[1] = 4u;
      ss.count = 2;
      a.seg = 1;
      a.seg_cols = c.d_s;
      a.bins = bins;
      a.n_bins = c.n_r;
      a.carry_key = ckey;
      a.carry_val = cval;
    }
    const int tr = gram_tile_rows(ss.row_bytes[0] + (q ? 4u : 0u), JS.row_split, q != 0);
    const int grid = gram_grid(c.n_s, tr, njob_groups(JS), num_sms);
    e = run_gram(JS, a, ss, tr, st, num_sms, 0);
    if (e != cudaSuccess) return e;
    s_parts = grid * JS.row_split;
    if (q) {
      cp_carry_fixup_kernel<<<1, ((c.d_s + 31) / 32) * 32, 0, st>>>(ckey, cval, 2 * grid, c.d_s, bins, c.n_r);
      FB_LAUNCHED();
    }
  } else if (q && c.d_s > 0) {
    // no rows: KᵀS = 0
    e = cudaMemsetAsync(bins, 0, static_cast<size_t>(c.n_r) * c.d_s * 8, st);
    if (e != cudaSuccess) return e;
  }
  const int s_tiles = static_cast<int>(maps.size());

  // ---- R pass: Rᵀ diag(c) R (upper) and RᵀB
  int r_parts = 0;
  GramJobs JR{};
  if (q && c.d_r > 0 && c.n_r > 0) {
    if (!build_jobs(nbr, true, true, c.d_s > 0 ? nbs : 0, true, kMaxSlots, s_tiles, JR, maps, c.d_s, c.d_s, 0, c.d_r, c.d_s))
      return cudaErrorNotSupported;
    GramArgs a{};
    a.n = c.n_r;
    const int pr = (c.d_r % 8 == 0) ? c.d_r + 4 : c.d_r;
    a.reg[0] = {pr, 0, c.d_r};
    a.reg[1] = {c.d_s > 0 ? c.d_s : 1, 1, c.d_s};
    a.cnt_stream = 2;
    a.partials = rp;
    StreamSet ss{};
    ss.base[0] = reinterpret_cast<const char*>(c.r);
    ss.row_bytes[0] = static_cast<uint32_t>(c.d_r) * 8u;
    ss.pitch[0] = static_cast<uint32_t>(pr) * 8u;
    ss.base[1] = reinterpret_cast<const char*>(bins);
    ss.row_bytes[1] = static_cast<uint32_t>(c.d_s) * 8u;
    ss.base[2] = reinterpret_cast<const char*>(c.counts);
    ss.row_bytes[2] = 8u;
    ss.count = 3;
    const int tr = gram_tile_rows(pr * 8u + c.d_s * 8u + 8u, JR.row_split, false);
    const int grid = gram_grid(c.n_r, tr, njob_groups(JR), num_sms);
    e = run_gram(JR, a, ss, tr, st, num_sms, 0);
    if (e != cudaSuccess) return e;
    r_parts = grid * JR.row_split;
  }
  // ---- assemble (fixed-order sums + exact mirror)
  const int ntot = static_cast<int>(maps.size());
  const int passes[2][3] = {{0, s_tiles, s_parts}, {s_tiles, ntot, r_parts}};
  for (const auto& ps : passes) {
    const int t0 = ps[0], t1 = ps[1];
    if (t1 <= t0) continue;
    if (t1 - t0 > kMaxTiles) return cudaErrorNotSupported;
    TileMaps tm;
    for (int i = t0; i < t1; ++i) tm.m[i - t0] = maps[i];
    const int n = (t1 - t0) * 64;
    cp_reduce_kernel<<<(n + 255) / 256, 256, 0, st>>>(t0 == 0 ? sp : rp, ps[2], t1 - t0, tm, c.out, d);
    FB_LAUNCHED();
  }
  return cudaGetLastError();
}

}  // namespace fb
