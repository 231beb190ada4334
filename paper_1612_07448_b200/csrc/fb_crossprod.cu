// fb_crossprod.cu — factorized crossprod TᵀT for T = [S, K·R] (rewrite.py:245-298,
// Algorithm 2 of the paper).
//
//   TᵀT = [[ SᵀS,        (KᵀS)ᵀR       ],
//          [ Rᵀ(KᵀS),    Rᵀ diag(c) R  ]]        c = colSums(K) (indicator.py:61-66)
//
//   KᵀS     kts_walk_kernel: a segmented reduction over the cached FK-sorted order (the GPU
//           analogue of the reference's _csr_t, indicator.py:78-86) on the side stream.
//   S pass  cp_gram_kernel over S in storage order (bulk copies): the upper triangle of SᵀS.
//   R pass  cp_gram_kernel over R with B = KᵀS and c alongside: the upper triangle of
//           Rᵀ diag(c) R (W fragments scaled by c) and the full RᵀB block.
//
// Gram work unit: an 8·BS × 8·BS "block tile" of BS × BS DMMA accumulators (mma.sync m8n8k4
// f64 → DMMA.8x8x4; tcgen05 has no f64 kind); BS = 2 costs 4 shared loads per 4 DMMAs. The
// (block tile, k-step) units of a tile are cut by a host-built table into one contiguous range
// per consumer warp, balanced across the 4 SM sub-partitions (one DMMA pipe each); a warp's
// accumulators stay in registers for the whole pass. Each (CTA, warp) writes its block tiles
// into a dense partial; cp_reduce_kernel sums the writers of every element in a fixed order
// and writes the exact mirror (lower = upperᵀ, rewrite.py:298 / kernel.py:132-135).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "fb_kernels.cuh"

namespace fb {

constexpr int kNB = 4;          // block tiles one warp may touch (BS = 2: 4 × 16 accumulator registers)
constexpr int kMaxGroups = 16;  // gridDim.y job groups
constexpr int kMaxBT = 256;     // block tiles per pass
constexpr int kWalkers = 3;     // KᵀS walker warps of the fused S pass (416 + 96 threads: 128 registers each;
                                // a fourth walker caps registers at 96 and the consumers spill; a gatherer
                                // warp traded for a fourth walker (512 threads kept): no gain, round 2)
constexpr int kWalkNB = kNB;    // block tiles per consumer warp in the fused pass

// block tile code: bits 0-5 A block bi, bits 6-11 W block bj, bit 12 W from region 1.
// Host-built assignment (build_block_jobs): the (block tile, k-step) units of a tile are
// laid out block-tile major and cut into one contiguous range per consumer warp, sized so
// every SM sub-partition (warp slot mod 4: one DMMA pipe each) gets the same share; warps
// that run the KᵀS walk get none. A warp's range covers <= kNB block tiles, each with a
// k-step interval [ka, kb) of every full tile.
struct WarpJob {
  uint16_t code[kNB];
  uint8_t ka[kNB], kb[kNB];
  uint8_t nb;
};
struct BlockJobs {
  WarpJob w[kMaxGroups][kConsumerWarps];
  int ngroups;
  int per_group;  // block tiles per group (the last may hold fewer)
  int total;      // block tiles of the pass
};

struct GramArgs {
  int64_t n;            // rows streamed
  int p0, p1;           // smem row pitch (doubles) of region 0 (A, and W when bit 12 clear) / region 1
  int s1;               // ring stream of region 1 (-1: none)
  int cnt_stream;       // stream holding per-row f64 counts that scale region-0 W frags (-1: none)
  int ra, cw;           // partial matrix: ra rows (8·BS·T2a) × cw cols (8·BS·(T2a + T2b))
  int w1_col0;          // first partial column of region 1 (8·BS·T2a)
  double* partials;     // [gridDim.x · 8 warps][ra][cw] (a warp writes only its block tiles)
  int debug;            // development bisection bits (FB_CP_DEBUG): 1 no walk, 2 no DMMA
  // fused KᵀS walk (S pass in FK-sorted order; cp_gram_kernel<BS, false, CJ > 0>)
  const int32_t* perm;       // sorted position -> S row
  const int32_t* keys;       // FK-sorted keys (ring stream `key_stream` carries the tile's keys)
  const double* s;           // S in global memory (rows of a tile the ring could not bulk-copy)
  int d;                     // S width
  int key_stream;
  double* bins;              // n_r × d, B = KᵀS
  int* carry_key;            // 2 slots per CTA (first run, last run)
  double* carry_val;
};

// KᵀS (B = group-by-key column sums of S, rewrite.py:260-270 via indicator.py:130-141) as
// a segmented reduction over the FK-sorted rows, in its own pass on a side stream beside the
// S gram (which then streams S in storage order with bulk copies). Warp w owns a contiguous
// range of sorted positions; lanes own columns (lane + 32 j); rows are gathered through the
// cached permutation 8 at a time (loads in flight together) and walked in order: a key
// change closes the run (its bins row written once, keys without rows in between zeroed).
// The first and last run of a warp's range may continue in the neighbouring ranges: they go
// to a carry table that cp_carry_fixup_kernel combines in order (deterministic, no atomics).
// Many resident warps hide the walk's dependency chains (a walker inside the gram CTA had
// two warps for the whole SM and bounded the S pass).
template <int CJ>
__global__ void __launch_bounds__(256, CJ <= 2 ? 4 : 2) kts_walk_kernel(const int32_t* __restrict__ perm,
                                                       const int32_t* __restrict__ keys, int64_t n,
                                                       const double* __restrict__ S, int d, double* __restrict__ bins,
                                                       int* __restrict__ carry_key, double* __restrict__ carry_val) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int64_t wid = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t lo = n * wid / nwarps, hi = n * (wid + 1) / nwarps;
  int key = -1;
  bool first = true;  // the open run is this range's first
  double sum[CJ];
#pragma unroll
  for (int j = 0; j < CJ; ++j) sum[j] = 0.0;
  auto close_open = [&](int next) {  // close the open run (if any) before key `next`
    if (key >= 0) {
      if (first) {
#pragma unroll
        for (int j = 0; j < CJ; ++j)
          if (lane + 32 * j < d) carry_val[static_cast<size_t>(2 * wid) * d + lane + 32 * j] = sum[j];
        if (lane == 0) carry_key[2 * wid] = key;
        first = false;
      } else {
#pragma unroll
        for (int j = 0; j < CJ; ++j)
          if (lane + 32 * j < d) bins[static_cast<int64_t>(key) * d + lane + 32 * j] = sum[j];
      }
      for (int z = key + 1; z < next; ++z)
#pragma unroll
        for (int j = 0; j < CJ; ++j)
          if (lane + 32 * j < d) bins[static_cast<int64_t>(z) * d + lane + 32 * j] = 0.0;
    }
    key = next;
#pragma unroll
    for (int j = 0; j < CJ; ++j) sum[j] = 0.0;
  };
  for (int64_t b0 = lo; b0 < hi; b0 += 32) {
    const int cnt = static_cast<int>(hi - b0 < 32 ? hi - b0 : 32);
    const int kl = lane < cnt ? keys[b0 + lane] : 0;
    const int rl = lane < cnt ? perm[b0 + lane] : 0;
    for (int j0 = 0; j0 < cnt; j0 += 8) {
      int kk[8];
      double vv[8][CJ];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int r = j0 + u;
        kk[u] = __shfl_sync(full, kl, r & 31);
        const int row = __shfl_sync(full, rl, r & 31);
#pragma unroll
        for (int j = 0; j < CJ; ++j)
          vv[u][j] = (r < cnt && lane + 32 * j < d) ? __ldcs(S + static_cast<int64_t>(row) * d + lane + 32 * j) : 0.0;
      }
      if (j0 + 8 <= cnt && kk[7] == key) {  // the batch continues the open run (keys are sorted)
#pragma unroll
        for (int j = 0; j < CJ; ++j)
          sum[j] += ((vv[0][j] + vv[1][j]) + (vv[2][j] + vv[3][j])) + ((vv[4][j] + vv[5][j]) + (vv[6][j] + vv[7][j]));
        continue;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (j0 + u < cnt) {
          if (kk[u] != key) close_open(kk[u]);
#pragma unroll
          for (int j = 0; j < CJ; ++j) sum[j] += vv[u][j];
        }
      }
    }
  }
  // the open run may continue in the next range: slot 1 (slot 0 if it is also the first run)
  const int slot = first ? 0 : 1;
  if (key >= 0) {
#pragma unroll
    for (int j = 0; j < CJ; ++j)
      if (lane + 32 * j < d) carry_val[static_cast<size_t>(2 * wid + slot) * d + lane + 32 * j] = sum[j];
  }
  if (lane == 0) {
    carry_key[2 * wid + slot] = key;  // -1: an empty range
    if (first) carry_key[2 * wid + 1] = -1;
  }
}

// KᵀS walker warps of the fused S pass. The ring streams S in FK-sorted order (rows gathered
// through the cached permutation) with the sorted keys alongside, so the walk reads every
// tile from shared memory while the consumer warps run the SᵀS DMMAs on the same tile: S
// crosses HBM once for both products. NW walker warps take whole tiles round-robin (tile kt
// of the CTA -> walker kt mod NW), lanes own columns (lane + 32 j). Within a tile, a key change
// closes the run: interior runs write their bins row once (keys without rows in between are
// zeroed); the tile's first and last runs, which may continue in the neighbouring tiles, go to
// the tile's two carry slots, combined in tile order by cp_carry_fixup_kernel — deterministic,
// no atomics (the contract of kts_walk_kernel, with tiles for warp ranges). A single walker
// per CTA walking every tile in order was the pass's bottleneck (one warp's dependent DADD
// and loop chains at IPC ~0.15 against ~4 spinning warps per SM sub-partition), hence several
// walkers on independent tiles. The walker of a tile releases its stage with one extra arrival
// on the stage's "empty" barrier.
template <int CJ>
FB_DEV void kts_walk_tiles(TileRing& ring, const StreamSet& ss, const GramArgs& a, int w, int nw) {
  const unsigned full = 0xffffffffu;
  const int lane = lane_id();
  const int d = a.d;
  const int pitch = static_cast<int>(ss.pitch[0] >> 3);
  bool on[CJ];  // this lane's columns lane + 32 j
  int lcol[CJ];  // lanes past the last column read a valid column (never stored): loads carry no predicate
#pragma unroll
  for (int j = 0; j < CJ; ++j) {
    on[j] = lane + 32 * j < d;
    lcol[j] = on[j] ? lane + 32 * j : d - 1;
  }
  int key;
  bool first;
  int64_t slot0;  // carry slots of the current tile
  double sum[CJ];
  auto close_open = [&](int next) {
    if (key >= 0) {
      double* dst = first ? a.carry_val + slot0 * d : a.bins + static_cast<int64_t>(key) * d;
#pragma unroll
      for (int j = 0; j < CJ; ++j)
        if (on[j]) dst[lane + 32 * j] = sum[j];
      if (first && lane == 0) a.carry_key[slot0] = key;
      first = false;
      for (int z = key + 1; z < next; ++z)
#pragma unroll
        for (int j = 0; j < CJ; ++j)
          if (on[j]) a.bins[static_cast<int64_t>(z) * d + lane + 32 * j] = 0.0;
    }
    key = next;
#pragma unroll
    for (int j = 0; j < CJ; ++j) sum[j] = 0.0;
  };
  auto add_rows = [&](const double* base, int stride, int lo, int hi) {  // rows [lo, hi)
    int u = lo;
    // 8-row blocks: independent loads, a pairwise tree, one add on the run's chain
    for (; u + 8 <= hi; u += 8) {
      double t[8][CJ];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < CJ; ++j) t[i][j] = base[(u + i) * stride + lcol[j]];
#pragma unroll
      for (int j = 0; j < CJ; ++j)
        sum[j] += ((t[0][j] + t[1][j]) + (t[2][j] + t[3][j])) + ((t[4][j] + t[5][j]) + (t[6][j] + t[7][j]));
    }
    if (u + 4 <= hi) {
      double t[4][CJ];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < CJ; ++j) t[i][j] = base[(u + i) * stride + lcol[j]];
#pragma unroll
      for (int j = 0; j < CJ; ++j) sum[j] += (t[0][j] + t[1][j]) + (t[2][j] + t[3][j]);
      u += 4;
    }
    for (; u < hi; ++u)
#pragma unroll
      for (int j = 0; j < CJ; ++j) sum[j] += base[u * stride + lcol[j]];
  };
  // A chunk of up to 32 rows: lane u < cnt holds the key of row u (kl); starts = rows whose key
  // differs from the previous row's (row 0: from the open run). Each run's rows are summed in
  // row order straight from shared memory; a run boundary closes the open run.
  auto fold = [&](const double* base, int stride, int kl, int cnt) {
    const int kprev0 = __shfl_up_sync(full, kl, 1);
    const int kprev = lane == 0 ? key : kprev0;
    unsigned starts = __ballot_sync(full, lane < cnt && kl != kprev);
    int pos = 0;
    while (starts) {
      const int b = __ffs(starts) - 1;
      starts &= starts - 1;
      add_rows(base, stride, pos, b);
      close_open(__shfl_sync(full, kl, b));
      pos = b;
    }
    add_rows(base, stride, pos, cnt);
  };
  const bool active = blockIdx.y == 0 && !(a.debug & 1);  // job groups > 0 stream the same rows: release only
  int st = w % ring.stages;
  uint32_t ph = (w / ring.stages) & 1u;
  for (int64_t kt = w; kt < ring.count(); kt += nw) {
    const int64_t tile = ring.tile_begin + kt;
    const int rows = active ? ring.rows_of(tile) : 0;
    mbar_wait(&ring.full[st], ph);
    mbar_wait(&ring.gfull[st], ph);
    key = -1;
    first = true;
    slot0 = 2 * tile;
#pragma unroll
    for (int j = 0; j < CJ; ++j) sum[j] = 0.0;
    if (ring.bulk_ok(ss, tile)) {
      const double* A = reinterpret_cast<const double*>(ring.stage_ptr(st, ss, 0));
      const int32_t* K = reinterpret_cast<const int32_t*>(ring.stage_ptr(st, ss, a.key_stream));
      for (int r0 = 0; r0 < rows; r0 += 32) {
        const int cnt = rows - r0 < 32 ? rows - r0 : 32;
        fold(A + r0 * pitch, pitch, lane < cnt ? K[r0 + lane] : -1, cnt);
      }
    } else {
      // a tile the ring could not bulk-copy is filled by the consumers: read it from global,
      // one row at a time
      const int64_t p0 = tile * ring.tile_rows;
      for (int r = 0; r < rows; ++r) {
        const double* row = a.s + static_cast<int64_t>(a.perm[p0 + r]) * d;
        fold(row, 0, lane == 0 ? a.keys[p0 + r] : -1, 1);
      }
    }
    __syncwarp(full);
    if (lane == 0) mbar_arrive(&ring.empty[st]);
    if (active) {
      // the open run may continue in the next tile: slot 1 (slot 0 if it is also the first run)
      const int64_t slot = slot0 + (first ? 0 : 1);
      if (key >= 0) {
#pragma unroll
        for (int j = 0; j < CJ; ++j)
          if (on[j]) a.carry_val[slot * d + lane + 32 * j] = sum[j];
      }
      if (lane == 0) {
        a.carry_key[slot] = key;  // -1: an empty tile
        if (first) a.carry_key[slot0 + 1] = -1;
      }
    }
    st += nw;
    while (st >= ring.stages) {
      st -= ring.stages;
      ph ^= 1u;
    }
  }
}

// NW > 0: fused KᵀS walk (see kts_walk_tiles) on NW extra warps, CJ = ceil(d_S / 32) columns
// per lane.
template <int BS, bool SCALE, int NW = 0, int CJ = 1, int NB = kNB>
__global__ void __launch_bounds__(kRingThreads + 32 * NW, 1)
    cp_gram_kernel(const __grid_constant__ BlockJobs jobs, GramArgs a, StreamSet ss, int stages, int tile_rows) {
  extern __shared__ __align__(128) char smem[];
  TileRing ring;
  ring.init(smem, stages, tile_rows, a.n);
  ring.start(ss, NW > 0 ? 1 : 0);  // one walker releases each stage
  if constexpr (NW > 0) {
    if (threadIdx.x >= kRingThreads) {
      kts_walk_tiles<CJ>(ring, ss, a, (static_cast<int>(threadIdx.x) - kRingThreads) >> 5, NW);
      return;
    }
  }
  if (ring.template service<(NW > 0)>(ss)) return;
  const int warp = consumer_warp();
  const int grp = blockIdx.y;
  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;

  const WarpJob& wj = jobs.w[grp][warp];
  const int nb = (a.debug & 2) ? 0 : wj.nb;
  int ka[NB], kb[NB], code[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    code[b] = wj.code[b];
    ka[b] = wj.ka[b];
    kb[b] = wj.kb[b];
  }
  // per block tile: A column offset and W column offset (this lane's row of the fragments)
  int aoff[NB], woff[NB];
  bool reg1[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    aoff[b] = 8 * BS * (code[b] & 63) + g;
    woff[b] = 8 * BS * ((code[b] >> 6) & 63) + g;
    reg1[b] = (code[b] >> 12) & 1;
  }
  double acc[NB][BS * BS][2];
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int u = 0; u < BS * BS; ++u) acc[b][u][0] = acc[b][u][1] = 0.0;

  for (int64_t kt = 0; kt < ring.count(); ++kt) {
    const int stage = ring.acquire(ss, kt);
    const int rows = ring.rows_of(ring.tile_begin + kt);
    const double* R0 = reinterpret_cast<const double*>(ring.stage_ptr(stage, ss, 0));
    const double* R1 = a.s1 >= 0 ? reinterpret_cast<const double*>(ring.stage_ptr(stage, ss, a.s1)) : R0;
    const double* cnt =
        a.cnt_stream >= 0 ? reinterpret_cast<const double*>(ring.stage_ptr(stage, ss, a.cnt_stream)) : nullptr;
    __syncwarp();  // mma.sync.aligned needs the whole warp converged (after the barrier spin)
    const int full = rows >> 2;  // k-steps whose four rows all exist
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      if (b < nb) {
        // one k-step of block tile b: rows k0..k0+3 (lane t takes row k0 + t)
        // one k-step of block tile b: rows k0..k0+3 (lane t takes row k0 + t). Operands of
        // step k+1 are loaded before the DMMAs of step k are issued (a lone warp on an SM
        // sub-partition otherwise waits out the shared-memory latency every step); the
        // count scaling is applied at use so it does not force that wait early.
        const double* wbase = reg1[b] ? R1 : R0;
        const int wp = reg1[b] ? a.p1 : a.p0;
        auto load = [&](int kr, bool live, double (&av)[BS], double (&wv)[BS], double& c) {
#pragma unroll
          for (int u = 0; u < BS; ++u) {
            av[u] = live ? R0[kr * a.p0 + aoff[b] + 8 * u] : 0.0;
            wv[u] = wbase[kr * wp + woff[b] + 8 * u];
          }
          c = SCALE && !reg1[b] ? cnt[kr] : 1.0;
        };
        auto mma = [&](const double (&av)[BS], const double (&wv)[BS], double c) {
#pragma unroll
          for (int v = 0; v < BS; ++v) {
            const double w = SCALE ? wv[v] * c : wv[v];
#pragma unroll
            for (int u = 0; u < BS; ++u) dmma_8x8x4(acc[b][u * BS + v][0], acc[b][u * BS + v][1], av[u], w);
          }
        };
        const int kend = min(kb[b], full);
        if (ka[b] < kend) {
          // operand pointers advanced by one k-step (4 rows) per iteration instead of an index
          // product per load (the R pass issued 1.5 IMAD per DMMA; ncu source view)
          const int kr0 = 4 * ka[b] + t;
          const double* pa = R0 + kr0 * a.p0 + aoff[b];
          const double* pw = wbase + kr0 * wp + woff[b];
          const double* pc = SCALE ? cnt + kr0 : nullptr;
          const int sa = 4 * a.p0, sw = 4 * wp;
          auto loadp = [&](double (&av)[BS], double (&wv)[BS], double& c) {
#pragma unroll
            for (int u = 0; u < BS; ++u) {
              av[u] = pa[8 * u];
              wv[u] = pw[8 * u];
            }
            c = SCALE && !reg1[b] ? *pc : 1.0;
            pa += sa;
            pw += sw;
            if (SCALE) pc += 4;
          };
          double av[BS], wv[BS], c;
          loadp(av, wv, c);
#pragma unroll 2
          for (int k = ka[b] + 1; k < kend; ++k) {
            double an[BS], wn[BS], cn;
            loadp(an, wn, cn);
            mma(av, wv, c);
#pragma unroll
            for (int u = 0; u < BS; ++u) {
              av[u] = an[u];
              wv[u] = wn[u];
            }
            c = cn;
          }
          mma(av, wv, c);
        }
        if ((rows & 3) && full >= ka[b] && full < kb[b]) {  // ragged last k-step of the last tile
          const bool live = 4 * full + t < rows;
          double av[BS], wv[BS], c;
          load(live ? 4 * full + t : 0, live, av, wv, c);
          mma(av, wv, c);
        }
      }
    }
    ring.release();
  }
  // this (CTA, warp) partial: block tile b covers rows 8·BS·bi + 8u + g, cols 8·BS·bj + 8v + 2t
  double* part = a.partials + static_cast<size_t>(blockIdx.x * kConsumerWarps + warp) * a.ra * a.cw;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    if (b < nb) {
      const int row0 = aoff[b] - g;
      const int col0 = (woff[b] - g) + (reg1[b] ? a.w1_col0 : 0);
#pragma unroll
      for (int u = 0; u < BS; ++u)
#pragma unroll
        for (int v = 0; v < BS; ++v) {
          double* dst = part + static_cast<size_t>(row0 + 8 * u + g) * a.cw + col0 + 8 * v + 2 * t;
          dst[0] = acc[b][BS * u + v][0];
          dst[1] = acc[b][BS * u + v][1];
        }
    }
  }
}

// Combine the boundary runs in slot order and zero the bins no row maps to at the seams and
// at both ends. Carry slots come in (first run, last run) pairs per walker range / per fused
// tile; interior gaps were zeroed by the walkers. One warp per slot (lanes over columns): the
// slot that starts a key's run of slots sums that run in slot order and writes the bins row;
// an even slot (a range's first run) also zeroes the keys between the previous run and its
// own (a seam), the last run the tail. (One CTA per slot cost ~160 us at c3's 312k slots.)
__global__ void cp_carry_fixup_kernel(const int* __restrict__ carry_key, const double* __restrict__ carry_val,
                                      int nslots, int cols, double* __restrict__ bins, int64_t n_bins) {
  const int i = static_cast<int>((blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= nslots) return;
  const int k = carry_key[i];
  if (k < 0) return;
  int prev = -1;  // key of the previous valid slot
  for (int j = i - 1; j >= 0; --j)
    if (carry_key[j] >= 0) {
      prev = carry_key[j];
      break;
    }
  if (prev == k) return;  // not the head of its run of slots
  int last = i;
  for (int j = i + 1; j < nslots; ++j) {
    const int kj = carry_key[j];
    if (kj < 0) continue;
    if (kj != k) break;
    last = j;
  }
  bool tail = true;  // no valid slot after this run: zero the keys above it
  for (int j = last + 1; j < nslots; ++j)
    if (carry_key[j] >= 0) {
      tail = false;
      break;
    }
  for (int c = lane; c < cols; c += 32) {
    double sum = 0.0;
    for (int j = i; j <= last; ++j)
      if (carry_key[j] >= 0) sum += carry_val[static_cast<size_t>(j) * cols + c];
    bins[static_cast<int64_t>(k) * cols + c] = sum;
    if ((i & 1) == 0)
      for (int z = prev + 1; z < k; ++z) bins[static_cast<int64_t>(z) * cols + c] = 0.0;
    if (tail)
      for (int64_t z = k + 1; z < n_bins; ++z) bins[z * cols + c] = 0.0;
  }
}

static void launch_carry_fixup(const int* ckey, const double* cval, int nslots, int cols, double* bins,
                               int64_t n_bins, cudaStream_t st) {
  if (nslots <= 0) return;
  cp_carry_fixup_kernel<<<(nslots + 7) / 8, 256, 0, st>>>(ckey, cval, nslots, cols, bins, n_bins);
  FB_LAUNCHED();
}

// Final assembly of one pass: element (i, j) of the pass = Σ over CTAs x, then over the
// warps w that hold units of its block tile, of partials[x·8 + w][i][j] (fixed order).
//   region 0 (j < w1_col0): the upper triangle (i <= j < da) of a gram block at (off0, off0)
//   region 1: a full da × db block at (off0, off1)
// Written at its position of the d × d output and mirrored exactly.
struct ReduceArgs {
  const double* partials;
  int gridx, ra, cw, w1_col0;
  int da, db;       // valid widths of region 0 / region 1
  int off0, off1;   // output offsets
  double* out;
  int64_t ldo;
  int bsz, t2a, t2b;  // block layout of the pass (build_block_jobs enumeration order)
  uint8_t wmask[kMaxBT];  // per block tile: the consumer warps that wrote it
  int r1only;         // 1: region 1 only (Rᵀ·X, launch_rtx): no gram triangle, no mirror
  int64_t o_cs;       // r1only: output column stride (element (i, j) at out[(off0+i)·ldo + (off1+j)·o_cs])
};

// Partial element (i, pc) -> its block tile -> the mask of consumer warps that wrote it.
FB_DEV uint32_t tile_writers(const ReduceArgs& r, int i, int pc) {
  const int bi = i / r.bsz;
  if (r.r1only) return r.wmask[bi * r.t2b + (pc - r.w1_col0) / r.bsz];
  int idx = bi * (r.t2a + r.t2b) - bi * (bi - 1) / 2;
  idx += pc < r.w1_col0 ? pc / r.bsz - bi : (r.t2a - bi) + (pc - r.w1_col0) / r.bsz;
  return r.wmask[idx];
}

FB_DEV bool reduce_coords(const ReduceArgs& r, int64_t e, int& i, int& pc, int& orow, int& ocol) {
  const int n0 = r.r1only ? 0 : r.da * r.da;
  int j;
  if (e < n0) {
    i = static_cast<int>(e / r.da);
    j = static_cast<int>(e % r.da);
    if (i > j) return false;
    pc = j;
    orow = r.off0 + i;
    ocol = r.off0 + j;
  } else {
    const int64_t f = e - n0;
    i = static_cast<int>(f / r.db);
    j = static_cast<int>(f % r.db);
    pc = r.w1_col0 + j;
    orow = r.off0 + i;
    ocol = r.off1 + j;
  }
  return true;
}

// One warp per output element: lanes stride over the CTAs, then a fixed butterfly
// (deterministic); the per-element serial loop was latency bound (~100 us per pass).
__global__ void cp_reduce_kernel(ReduceArgs r) {
  const int64_t e = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  // r1only passes (launch_rtx) have da·db elements: the gram bound let the last CTA's spare warps
  // reduce and store up to 7 elements of a row past the block (found by tests/test_fuzz_gpu.py:
  // K-Means with an even k > 16 not a multiple of 8 had its first cluster sizes overwritten)
  if (e >= static_cast<int64_t>(r.da) * ((r.r1only ? 0 : r.da) + r.db)) return;
  int i, pc, orow, ocol;
  if (!reduce_coords(r, e, i, pc, orow, ocol)) return;
  const uint32_t mask = tile_writers(r, i, pc);
  const size_t stride = static_cast<size_t>(r.ra) * r.cw;
  const double* p = r.partials + static_cast<size_t>(i) * r.cw + pc;
  double s = 0.0;
  for (int x = lane; x < r.gridx; x += 32)
    for (uint32_t m = mask; m; m &= m - 1) s += p[(static_cast<size_t>(x) * kConsumerWarps + __ffs(m) - 1) * stride];
  s = warp_sum(s);
  if (lane == 0) {
    if (r.r1only) {
      r.out[orow * r.ldo + ocol * r.o_cs] = s;
    } else {
      r.out[orow * r.ldo + ocol] = s;
      r.out[ocol * r.ldo + orow] = s;
    }
  }
}

static void launch_reduce(const ReduceArgs& r, cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(r.da) * ((r.r1only ? 0 : r.da) + r.db);
  cp_reduce_kernel<<<static_cast<unsigned>((n * 32 + 255) / 256), 256, 0, st>>>(r);
  FB_LAUNCHED();
}

// ------------------------------------------------------------------ host side
namespace {

// Upper-triangle block tiles of a T2a × T2a gram, plus a full T2a × T2b rectangle (region 1),
// in row-major order (tile_writers depends on it), cut into ngroups equal groups; in each
// group the units are split over the consumer warps as described at WarpJob. The first
// `walkers` consumer warps of group 0 run the KᵀS walk and get no units. wmask receives,
// per block tile, the warps that hold units of it.
bool build_block_jobs(int T2a, int T2b, int nks, int walkers, BlockJobs& J, uint8_t* wmask, bool r1only = false,
                      int nb_max = kNB) {
  std::vector<uint16_t> list;
  for (int bi = 0; bi < T2a; ++bi) {
    if (!r1only)
      for (int bj = bi; bj < T2a; ++bj) list.push_back(static_cast<uint16_t>(bi | (bj << 6)));
    for (int bj = 0; bj < T2b; ++bj) list.push_back(static_cast<uint16_t>(bi | (bj << 6) | (1 << 12)));
  }
  const int bt = static_cast<int>(list.size());
  J = BlockJobs{};
  J.ngroups = 1;
  J.per_group = 1;
  J.total = bt;
  if (bt == 0) return true;
  if (T2a > 63 || T2b > 63 || bt > kMaxBT || nks > 255) return false;
  for (int ng = 1; ng <= kMaxGroups; ++ng) {
    J = BlockJobs{};
    J.ngroups = ng;
    J.per_group = (bt + ng - 1) / ng;
    J.total = bt;
    std::fill(wmask, wmask + kMaxBT, 0);
    bool ok = true;
    for (int gi = 0; gi < ng && ok; ++gi) {
      const int b0 = gi * J.per_group, nbtg = std::min(J.per_group, bt - b0);
      if (nbtg <= 0) break;
      const int first = gi == 0 ? walkers : 0;
      // sub-partition of consumer warp w: its hardware warp slot mod 4
      int m[4] = {0, 0, 0, 0};
      for (int w = first; w < kConsumerWarps; ++w) ++m[(kServiceWarps + w) % 4];
      int nsp = 0;
      for (int q = 0; q < 4; ++q) nsp += m[q] > 0;
      const int64_t U = static_cast<int64_t>(nbtg) * nks;
      double cum = 0.0;
      int64_t u0 = 0;
      for (int w = first; w < kConsumerWarps && ok; ++w) {
        cum += 1.0 / (m[(kServiceWarps + w) % 4] * nsp);
        int64_t u1 = w == kConsumerWarps - 1 ? U : static_cast<int64_t>(cum * U + 0.5);
        if (u1 > U) u1 = U;
        WarpJob& wj = J.w[gi][w];
        while (u0 < u1) {
          const int b = static_cast<int>(u0 / nks);
          const int64_t e = std::min<int64_t>(u1, static_cast<int64_t>(b + 1) * nks);
          if (wj.nb == nb_max) {
            ok = false;
            break;
          }
          wj.code[wj.nb] = list[b0 + b];
          wj.ka[wj.nb] = static_cast<uint8_t>(u0 - static_cast<int64_t>(b) * nks);
          wj.kb[wj.nb] = static_cast<uint8_t>(e - static_cast<int64_t>(b) * nks);
          ++wj.nb;
          wmask[b0 + b] |= static_cast<uint8_t>(1u << w);
          u0 = e;
        }
      }
    }
    if (ok) return true;
  }
  return false;
}

size_t al(size_t b) { return (b + 255) & ~size_t(255); }

int gram_grid(int64_t n, int tile_rows, int ngroups, int num_sms) {
  const int64_t ntiles = (n + tile_rows - 1) / tile_rows;
  const int per = ngroups > 1 ? std::max(1, num_sms / ngroups) : num_sms;
  return grid_for(ntiles, 1, 1, per);
}

int gram_tile_rows(uint32_t row_bytes, bool gather) {
  int rows = static_cast<int>((48u * 1024u) / (row_bytes > 0 ? row_bytes : 1));
  const int unit = 32;  // 8 k-steps: one per consumer warp
  if (rows > (gather ? 128 : 256)) rows = gather ? 128 : 256;
  rows = (rows / unit) * unit;
  if (rows < unit) rows = unit;
  // long rows (the c3 R pass: 1480 B): 64-row tiles in two ~95 KB stages beat 32-row tiles in
  // four — a warp's per-tile overhead (ring wait, job loop, pipeline prologue) is paid over 16
  // k-steps instead of 8 (R pass 0.83 -> 0.74 ms)
  if (!gather && rows < 64 && 2u * 64u * row_bytes + 2048u <= 200u * 1024u) rows = 64;
  return rows;
}

// Launch one pass; *gridx = CTAs per group (each wrote kConsumerWarps partial slots).
cudaError_t run_gram(const BlockJobs& J, GramArgs& a, StreamSet& ss, int tile_rows, cudaStream_t st, int num_sms,
                     int* gridx, int bs, int walk_cj = 0, int walk_nb = kWalkNB) {
  stream_layout(ss, tile_rows, a.n);
  int stages = static_cast<int>((200 * 1024 - kRingHeader - 256) / ss.stage_bytes);
  if (stages > 6) stages = 6;
  if (const char* e = getenv("FB_CP_STAGES")) stages = std::min(stages, atoi(e));  // development override
  // fused walk: walker w takes tiles w, w + kWalkers, ...; with a stage count that is a multiple
  // of kWalkers, the previous tile on a walker's stage is its own, so its parity wait can never
  // see a fill one round old as the one it wants (mbarrier parity aliases phases two apart)
  if (walk_cj > 0) stages = (stages / kWalkers) * kWalkers;
  if (stages < 2) return cudaErrorNotSupported;
  // + slack: fragment loads of a padded block read up to 8·BS - 1 doubles past a row,
  // so the last row of the last stage must not sit at the end of the allocation
  const size_t smem = kRingHeader + static_cast<size_t>(stages) * ss.stage_bytes + 256;
  if (const char* dbg = getenv("FB_CP_DEBUG")) a.debug = atoi(dbg);
  dim3 gdim(gram_grid(a.n, tile_rows, J.ngroups, num_sms), J.ngroups);
  *gridx = static_cast<int>(gdim.x);
  if (getenv("FB_DEBUG_SYNC"))
    fprintf(stderr, "[fb] gram pass n=%lld tile_rows=%d stages=%d grid=%dx%d bt=%d/group bs=%d\n", (long long)a.n,
            tile_rows, stages, gdim.x, gdim.y, J.per_group, bs);
  cudaError_t e;
#define FB_WALK_CASE(S, CJ)                                                                                     \
  if (bs == S && walk_cj == CJ) {                                                                               \
    auto kern = walk_nb == 2 ? cp_gram_kernel<S, false, kWalkers, CJ, 2> : cp_gram_kernel<S, false, kWalkers, CJ, kWalkNB>; \
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));        \
    if (e != cudaSuccess) return e;                                                                             \
    kern<<<gdim, kRingThreads + 32 * kWalkers, smem, st>>>(J, a, ss, stages, tile_rows);                         \
    FB_LAUNCHED();                                                                                              \
    return cudaGetLastError();                                                                                  \
  }
  if (walk_cj > 0) {
    FB_WALK_CASE(1, 1)
    FB_WALK_CASE(2, 1)
    FB_WALK_CASE(2, 2)
    FB_WALK_CASE(2, 3)
    FB_WALK_CASE(2, 4)
    return cudaErrorNotSupported;
  }
#undef FB_WALK_CASE
#define FB_GRAM_CASE(S)                                                                                         \
  if (bs == S) {                                                                                                \
    auto kern = a.cnt_stream >= 0 ? cp_gram_kernel<S, true> : cp_gram_kernel<S, false>;                        \
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));        \
    if (e != cudaSuccess) return e;                                                                             \
    kern<<<gdim, kRingThreads, smem, st>>>(J, a, ss, stages, tile_rows);                                        \
    FB_LAUNCHED();                                                                                              \
    return cudaGetLastError();                                                                                  \
  }
  FB_GRAM_CASE(1)
  FB_GRAM_CASE(2)
#undef FB_GRAM_CASE
  return cudaErrorNotSupported;
}

size_t partial_doubles(int T2a, int T2b, int num_sms, int bs) {
  // one slot per (CTA, consumer warp); all groups together use at most num_sms CTAs per row
  return static_cast<size_t>(num_sms) * kConsumerWarps * (8 * bs * T2a) * (8 * bs * (T2a + T2b));
}

// Block size (8-column blocks per side) of a pass over widths da (A) and db (region 1): large
// blocks reuse fragments (4 + 4 loads per 16 DMMAs) at the cost of triangle padding.
// KᵀS walk: warps (8 per CTA, 4 CTAs per SM) and the launch (+ the ordered carry fixup).
int kts_warps(int num_sms) { return num_sms * 4 * 8; }

cudaError_t launch_kts(const CrossArgs& c, double* bins, int* ckey, double* cval, cudaStream_t st, int num_sms) {
  const int grid = num_sms * 4;
  const int cj = (c.d_s + 31) / 32;
#define FB_KTS_CASE(J)                                                                                        \
  case J:                                                                                                     \
    kts_walk_kernel<J><<<grid, 256, 0, st>>>(c.perm, c.fk_sorted, c.n_s, c.s, c.d_s, bins, ckey, cval);      \
    break;
  switch (cj) {
    FB_KTS_CASE(1)
    FB_KTS_CASE(2)
    FB_KTS_CASE(3)
    FB_KTS_CASE(4)
    default:
      return cudaErrorNotSupported;
  }
#undef FB_KTS_CASE
  FB_LAUNCHED();
  const int slots = 2 * kts_warps(num_sms);
  launch_carry_fixup(ckey, cval, slots, c.d_s, bins, c.n_r, st);
  return cudaGetLastError();
}

// Fused S pass tiles: ~32 KB stages (6 in flight). A stage stays busy for its gather latency
// plus the walk of that tile (a walker's per-tile latency exceeds the DMMA time of a tile), so
// the ring needs more, smaller stages than a pass whose stages turn over at consumer speed.
int fused_tile_rows(int d_s) {
  if (const char* e = getenv("FB_CP_FUSED_ROWS")) return atoi(e);  // development override
  int rows = static_cast<int>((32u * 1024u) / (static_cast<uint32_t>(d_s) * 8u + 4u));
  rows = (rows / 32) * 32;
  if (rows > 128) rows = 128;
  return rows < 32 ? 32 : rows;
}

// Carry slots: two per walker warp range (kts_walk_kernel) or per tile of the fused S pass.
size_t carry_slots(int64_t n_s, int d_s, int num_sms) {
  const int64_t tr = 32;  // the smallest fused tile (FB_CP_FUSED_ROWS may pick any multiple of 32)
  return std::max<size_t>(2 * static_cast<size_t>(kts_warps(num_sms)), 2 * static_cast<size_t>((n_s + tr - 1) / tr));
}

// Shared-memory row pitch (doubles) for the DMMA fragment loads of a gram pass: a half-warp
// of an LDS.64 covers rows t = 0..3 × 4 consecutive doubles g, i.e. banks 2(t·p + g) (+1) mod 32;
// they are distinct for p ≡ 4 or 12 (mod 16). Even widths are padded up to the next such
// pitch (the padded rows stream with one bulk copy per row, StreamSet::row_bulk); odd widths
// (whose rows cannot be bulk-copied) keep their width. d_r = 120 (≡ 8): 2-way conflicts on
// every fragment load held the c3 R pass at ~55% of the DMMA rate.
int frag_pitch(int d) {
  if (d & 1) return d;
  int p = d;
  while (p % 16 != 4 && p % 16 != 12) p += 2;
  return p;
}

int block_size(int da) {
  if (const char* e = getenv("FB_CP_BS")) return atoi(e);  // development override (1, 2 or 4)
  return da <= 8 ? 1 : 2;
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

size_t crossprod_workspace_bytes(int64_t n_s, int d_s, int64_t n_r, int d_r, int q, int num_sms) {
  const int bs_s = block_size(d_s), bs_r = block_size(d_r);
  const int t2s = (d_s + 8 * bs_s - 1) / (8 * bs_s), t2r = (d_r + 8 * bs_r - 1) / (8 * bs_r);
  const int t2b = q ? (d_s + 8 * bs_r - 1) / (8 * bs_r) : 0;
  size_t b = al(partial_doubles(t2s, 0, num_sms, bs_s) * 8);
  b += al(partial_doubles(t2r, t2b, num_sms, bs_r) * 8);
  if (q > 0) {
    const size_t slots = carry_slots(n_s, d_s, num_sms);
    b += al(static_cast<size_t>(n_r) * d_s * 8);               // B = KᵀS
    b += al(slots * sizeof(int));                               // carry keys
    b += al(slots * static_cast<size_t>(d_s > 0 ? d_s : 1) * 8);  // carry values
  }
  return b + 1024;
}

// SᵀS of a narrow plain matrix (q = 0, d <= 8: GNMF's WᵀW, 5M × 5 at c5): a thread per row
// (a warp reads 32 consecutive rows), the d(d+1)/2 upper products in registers, warp
// butterflies, per-CTA partials in warp order, the last CTA sums the partials in CTA order and
// writes both triangles (exactly symmetric). The DMMA gram pass costs ~100 µs of tile and job
// overhead for these 200 MB; this one streams them.
template <int R>
__global__ void __launch_bounds__(256) narrow_gram_kernel(const double* __restrict__ f, int64_t n,
                                                          double* __restrict__ partials, unsigned* counter,
                                                          double* __restrict__ out, int64_t ldo) {
  constexpr int P = R * (R + 1) / 2;
  double acc[P];
#pragma unroll
  for (int i = 0; i < P; ++i) acc[i] = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    double v[R];
#pragma unroll
    for (int a = 0; a < R; ++a) v[a] = __ldcs(f + i * R + a);
    int k = 0;
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = a; b < R; ++b, ++k) acc[k] = fma(v[a], v[b], acc[k]);
  }
  __shared__ double wpart[8][P];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const double v = warp_sum(acc[k]);
    if (lane == 0) wpart[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < P) {
    double v = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) v += wpart[w][threadIdx.x];
    partials[static_cast<size_t>(blockIdx.x) * P + threadIdx.x] = v;
  }
  __threadfence();
  __shared__ unsigned ticket;
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(counter, 1u);
  __syncthreads();
  if (ticket != gridDim.x - 1) return;
  __threadfence();
  for (int k = warp; k < P; k += blockDim.x >> 5) {
    const double v = warp_sum_strided(partials + k, gridDim.x, P);
    if (lane == 0) {
      int a = 0, rem = k;
      while (rem >= R - a) {
        rem -= R - a;
        ++a;
      }
      const int b = a + rem;
      out[a * ldo + b] = v;
      out[b * ldo + a] = v;
    }
  }
  if (threadIdx.x == 0) *counter = 0u;
}

static cudaError_t launch_narrow_gram(const double* f, int64_t n, int d, double* partials, unsigned* counter,
                                      double* out, cudaStream_t st, int num_sms) {
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  const int grid = grid_for(n, 256 * 4, 4, num_sms);
  switch (d) {
#define FB_NG_CASE(R)                                                                       \
  case R:                                                                                   \
    narrow_gram_kernel<R><<<grid, 256, 0, st>>>(f, n, partials, counter, out, d);           \
    break;
    FB_NG_CASE(1) FB_NG_CASE(2) FB_NG_CASE(3) FB_NG_CASE(4) FB_NG_CASE(5) FB_NG_CASE(6) FB_NG_CASE(7) FB_NG_CASE(8)
#undef FB_NG_CASE
    default:
      return cudaErrorNotSupported;
  }
  FB_LAUNCHED();
  return cudaGetLastError();
}

cudaError_t launch_crossprod(const CrossArgs& c, void* ws, size_t ws_bytes, cudaStream_t st, int num_sms) {
  const int d = c.d_s + c.d_r;
  const int q = c.r ? 1 : 0;
  if (!q && c.d_s >= 1 && c.d_s <= 8 && c.n_s > 0 && !getenv("FB_CP_NO_NARROW")) {
    // partials (grid × d(d+1)/2 doubles) + counter inside the workspace's first partial slot
    double* partials = static_cast<double*>(ws);
    unsigned* counter = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + al(static_cast<size_t>(num_sms) * 4 * 36 * 8));
    if (al(static_cast<size_t>(num_sms) * 4 * 36 * 8) + 256 > ws_bytes) return cudaErrorInvalidValue;
    return launch_narrow_gram(c.s, c.n_s, c.d_s, partials, counter, c.out, st, num_sms);
  }
  const int bs_s = block_size(c.d_s), bs_r = block_size(c.d_r);
  const int t2s = (c.d_s + 8 * bs_s - 1) / (8 * bs_s), t2r = (c.d_r + 8 * bs_r - 1) / (8 * bs_r);
  const int t2b = q && c.d_s > 0 ? (c.d_s + 8 * bs_r - 1) / (8 * bs_r) : 0;
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t b) {
    char* r = p;
    p += al(b);
    return r;
  };
  double* sp = reinterpret_cast<double*>(take(partial_doubles(t2s, 0, num_sms, bs_s) * 8));
  double* rp = reinterpret_cast<double*>(take(partial_doubles(t2r, t2b, num_sms, bs_r) * 8));
  double* bins = nullptr;
  int* ckey = nullptr;
  double* cval = nullptr;
  const size_t slots = carry_slots(c.n_s, c.d_s, num_sms);
  if (q) {
    bins = reinterpret_cast<double*>(take(static_cast<size_t>(c.n_r) * c.d_s * 8));
    ckey = reinterpret_cast<int*>(take(slots * sizeof(int)));
    cval = reinterpret_cast<double*>(take(slots * (c.d_s > 0 ? c.d_s : 1) * 8));
    if (c.kts) bins = c.kts;  // split passes: KᵀS lives in the caller's buffer
  }
  if (static_cast<size_t>(p - static_cast<char*>(ws)) > ws_bytes) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(c.out, 0, static_cast<size_t>(d) * d * 8, st);
  if (e != cudaSuccess) return e;
  const bool do_s = c.mode != 2, do_r = c.mode != 1;
  if (do_s) {

  // ---- S pass. Fused (q = 1, even d_S <= 128): one pass over S in FK-sorted order computes
  // SᵀS on the consumer warps and KᵀS on the walker warp. Otherwise SᵀS streams S in storage
  // order on the main stream and kts_walk_kernel runs KᵀS on the side stream.
  const bool fused = q && c.d_s > 0 && c.n_s > 0 && c.d_s <= 128 && (c.d_s % 2) == 0 && c.n_s <= INT32_MAX &&
                     !getenv("FB_CP_UNFUSED");
  if (fused) {
    GramArgs a{};
    a.n = c.n_s;
    a.p0 = a.p1 = c.d_s;
    a.s1 = -1;
    a.cnt_stream = -1;
    a.ra = 8 * bs_s * t2s;
    a.cw = 8 * bs_s * t2s;
    a.w1_col0 = 8 * bs_s * t2s;
    a.partials = sp;
    a.perm = c.perm;
    a.keys = c.fk_sorted;
    a.s = c.s;
    a.d = c.d_s;
    a.key_stream = 1;
    a.bins = bins;
    a.carry_key = ckey;
    a.carry_val = cval;
    StreamSet ss{};
    ss.base[0] = reinterpret_cast<const char*>(c.s);
    ss.row_bytes[0] = static_cast<uint32_t>(c.d_s) * 8u;
    ss.gidx = c.perm;
    ss.base[1] = reinterpret_cast<const char*>(c.fk_sorted);
    ss.row_bytes[1] = 4u;
    ss.count = 2;
    ss.gidx_bulk = !getenv("FB_CP_GIDX_CHUNKS");
    const int tr = fused_tile_rows(c.d_s);
    ReduceArgs r{sp, 0, a.ra, a.cw, a.w1_col0, c.d_s, 0, 0, 0, c.out, d, 8 * bs_s, t2s, 0, {}};
    BlockJobs JS;
    if (!build_block_jobs(t2s, 0, tr / 4, 0, JS, r.wmask, false, kWalkNB)) return cudaErrorNotSupported;
    // Opt-in (FB_CP_NB2=1, measurement): when no warp's range touches more than two block tiles
    // (c3: 10 block tiles over 8 warps), the two-tile instantiation halves the accumulator
    // registers and the freed registers keep each range's bounds and offsets live across tiles
    // instead of re-deriving them from the constant bank at every range (an S2R -> LDC -> LDC ->
    // LDS chain per range per tile). The consumers alone get faster (c3 op 2.79 -> 2.61 ms with the
    // walkers idle), but the walkers' DADDs share the FP64 datapath with the DMMAs and then cost
    // what the idle slots used to hide: 3.00 vs 2.93 ms with everything on, so it is not the default.
    int walk_nb = kWalkNB;
    {
      BlockJobs J2;
      uint8_t wm2[kMaxBT];
      if (getenv("FB_CP_NB2") && build_block_jobs(t2s, 0, tr / 4, 0, J2, wm2, false, 2) && J2.ngroups == JS.ngroups) {
        JS = J2;
        std::copy(wm2, wm2 + kMaxBT, r.wmask);
        walk_nb = 2;
      }
    }
    int gridx = 0;
    e = run_gram(JS, a, ss, tr, st, num_sms, &gridx, bs_s, (c.d_s + 31) / 32, walk_nb);
    if (e != cudaSuccess) return e;
    r.gridx = gridx;
    launch_reduce(r, st);
    const int nslots = static_cast<int>(2 * ((c.n_s + tr - 1) / tr));  // two carry slots per tile
    launch_carry_fixup(ckey, cval, nslots, c.d_s, bins, c.n_r, st);
  }
  bool forked = false;
  if (!fused && q && c.d_s > 0 && c.n_s > 0) {
    cudaStream_t side = nullptr;
    e = side_fork(st, &side);
    if (e != cudaSuccess) return e;
    forked = true;
    e = launch_kts(c, bins, ckey, cval, side, num_sms);
    if (e != cudaSuccess) return e;
  }
  if (!fused && c.d_s > 0 && c.n_s > 0) {
    GramArgs a{};
    a.n = c.n_s;
    a.p0 = a.p1 = c.d_s;
    a.s1 = -1;
    a.cnt_stream = -1;
    a.ra = 8 * bs_s * t2s;
    a.cw = 8 * bs_s * t2s;
    a.w1_col0 = 8 * bs_s * t2s;
    a.partials = sp;
    StreamSet ss{};
    ss.base[0] = reinterpret_cast<const char*>(c.s);
    ss.row_bytes[0] = static_cast<uint32_t>(c.d_s) * 8u;
    ss.count = 1;
    const int tr = gram_tile_rows(ss.row_bytes[0], false);
    ReduceArgs r{sp, 0, a.ra, a.cw, a.w1_col0, c.d_s, 0, 0, 0, c.out, d, 8 * bs_s, t2s, 0, {}};
    BlockJobs JS;
    if (!build_block_jobs(t2s, 0, tr / 4, 0, JS, r.wmask)) return cudaErrorNotSupported;
    int gridx = 0;
    e = run_gram(JS, a, ss, tr, st, num_sms, &gridx, bs_s);
    r.gridx = gridx;
    if (e != cudaSuccess) return e;
    launch_reduce(r, st);
  } else if (!fused && q && c.d_s > 0) {
    e = cudaMemsetAsync(bins, 0, static_cast<size_t>(c.n_r) * c.d_s * 8, st);  // no rows: KᵀS = 0
    if (e != cudaSuccess) return e;
  }
  if (forked) {
    e = side_join(st);  // the R pass reads B
    if (e != cudaSuccess) return e;
  }

  }  // do_s

  // ---- R pass: Rᵀ diag(c) R (upper) and RᵀB
  if (do_r && q && c.d_r > 0 && c.n_r > 0) {
    GramArgs a{};
    a.n = c.n_r;
    // R rows padded to a bank-conflict-free pitch (frag_pitch), one bulk copy per row
    const int pr = frag_pitch(c.d_r);
    a.p0 = pr;
    a.p1 = c.d_s > 0 ? c.d_s : 1;
    a.s1 = c.d_s > 0 ? 1 : -1;
    a.cnt_stream = 2;
    a.ra = 8 * bs_r * t2r;
    a.cw = 8 * bs_r * (t2r + t2b);
    a.w1_col0 = 8 * bs_r * t2r;
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
    ss.row_bulk = true;
    const int tr = gram_tile_rows(pr * 8u + c.d_s * 8u + 8u, false);
    ReduceArgs r{rp, 0, a.ra, a.cw, a.w1_col0, c.d_r, c.d_s, c.d_s, 0, c.out, d, 8 * bs_r, t2r, t2b, {}};
    BlockJobs JR;
    if (!build_block_jobs(t2r, t2b, tr / 4, 0, JR, r.wmask)) return cudaErrorNotSupported;
    int gridx = 0;
    e = run_gram(JR, a, ss, tr, st, num_sms, &gridx, bs_r);
    r.gridx = gridx;
    if (e != cudaSuccess) return e;
    launch_reduce(r, st);
  }
  return cudaGetLastError();
}


// ------------------------------------------------------------------ Rᵀ·X on the tensor cores
// out(c, j) = Σ_r R(r, c)·X(r, j): the R-side contraction of Tᵀ·X-shaped products (K-Means
// R_qᵀ(AᵀK_q)ᵀ, RMM/Tᵀ·X bins passes) as the crossprod R pass restricted to its region 1.
// X rows must be 16-byte multiples (even nx) so both streams move with bulk copies.
static void rtx_layout(int d_r, int nx, int& bs, int& t2a, int& t2b) {
  bs = block_size(d_r > nx ? d_r : nx);
  t2a = (d_r + 8 * bs - 1) / (8 * bs);
  t2b = (nx + 8 * bs - 1) / (8 * bs);
}

size_t rtx_workspace_bytes(int d_r, int nx, int num_sms) {
  int bs, t2a, t2b;
  rtx_layout(d_r, nx, bs, t2a, t2b);
  return static_cast<size_t>(num_sms) * kConsumerWarps * (8 * bs * t2a) * (8 * bs * t2b) * 8 + 256;
}

bool rtx_supported(int d_r, int nx) { return d_r > 0 && nx >= 2 && nx % 2 == 0 && nx <= 128 && d_r <= 512; }

cudaError_t launch_rtx(const double* r, int64_t n_r, int d_r, const double* x, int nx, double* out, int64_t o_rs,
                       int64_t o_cs, void* ws, size_t ws_bytes, cudaStream_t st, int num_sms) {
  if (!rtx_supported(d_r, nx)) return cudaErrorNotSupported;
  if (ws_bytes < rtx_workspace_bytes(d_r, nx, num_sms)) return cudaErrorInvalidValue;
  if (n_r <= 0) {
    for (int c = 0; c < d_r; ++c) {
      cudaError_t e = cudaMemset2DAsync(out + c * o_rs, static_cast<size_t>(o_cs) * 8, 0, 8, nx, st);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  int bs, t2a, t2b;
  rtx_layout(d_r, nx, bs, t2a, t2b);
  GramArgs a{};
  a.n = n_r;
  const int pr = frag_pitch(d_r);  // see the crossprod R pass
  a.p0 = pr;
  a.p1 = nx;
  a.s1 = 1;
  a.cnt_stream = -1;
  a.ra = 8 * bs * t2a;
  a.cw = 8 * bs * t2b;
  a.w1_col0 = 0;
  a.partials = static_cast<double*>(ws);
  StreamSet ss{};
  ss.base[0] = reinterpret_cast<const char*>(r);
  ss.row_bytes[0] = static_cast<uint32_t>(d_r) * 8u;
  ss.pitch[0] = static_cast<uint32_t>(pr) * 8u;
  ss.base[1] = reinterpret_cast<const char*>(x);
  ss.row_bytes[1] = static_cast<uint32_t>(nx) * 8u;
  ss.count = 2;
  ss.row_bulk = true;
  const int tr = gram_tile_rows(pr * 8u + nx * 8u, false);
  ReduceArgs ra{};
  ra.partials = a.partials;
  ra.ra = a.ra;
  ra.cw = a.cw;
  ra.w1_col0 = 0;
  ra.da = d_r;
  ra.db = nx;
  ra.out = out;
  ra.ldo = o_rs;
  ra.o_cs = o_cs;
  ra.bsz = 8 * bs;
  ra.t2a = t2a;
  ra.t2b = t2b;
  ra.r1only = 1;
  BlockJobs J;
  if (!build_block_jobs(t2a, t2b, tr / 4, 0, J, ra.wmask, true)) return cudaErrorNotSupported;
  int gridx = 0;
  cudaError_t e = run_gram(J, a, ss, tr, st, num_sms, &gridx, bs);
  if (e != cudaSuccess) return e;
  ra.gridx = gridx;
  launch_reduce(ra, st);
  return cudaGetLastError();
}
}  // namespace fb
