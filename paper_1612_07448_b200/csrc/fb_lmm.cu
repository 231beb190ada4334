// fb_lmm.cu — factorized left multiplication T·X and its row-wise relatives.
//
// Replaces the reference's LMM rewrite (rewrite.py:172-191): for every column block
// out += F·X[slice], with indicator blocks applied as a gather *after* the factor
// product (rewrite.py:187-189, "R·X before K"). On B200 that is two streaming passes:
//   1. z_q = R_q · X[slice_q]          (one pass over each attribute table)
//   2. out_i = S_i · X[0:d_S] + Σ_q z_q[fk_q[i]]   (one pass over S and the FK columns)
// rowSums (rewrite.py:118-128) is the same pass with X = ones.
//
// Factor rows stream through the warp-specialised bulk-copy ring (fb_stream.cuh). Two
// consumer bodies:
//   * rowdot (d_x <= 4): FP64 FMAs. L lanes share a row (L = the largest power of two
//     dividing the width, so the 8-byte shared loads of a half-warp hit distinct banks),
//     a butterfly shuffle finishes the dot product, and lane k ends up owning row k of
//     its 32-row group for a coalesced epilogue.
//   * DMMA (5 <= d_x <= 16): mma.sync m8n8k4 f64 (SASS DMMA; tcgen05 has no f64 kind),
//     each warp owning MT m-tiles of 8 rows against X zero-padded to NT·8 columns.
// The z[fk] rows are keyed gathers of the ring (fb_stream.cuh): the gatherer warp bulk-
// copies them into the stage as soon as the FK column lands, so they arrive as many
// stages ahead as the S rows and the consumers only read shared memory. z rows are
// padded to an even number of doubles (16-byte bulk copies) and read with an L2
// evict_last policy; the streamed output is written evict_first; the z-pass (no FK)
// stores z evict_last so it stays L2-resident for the S pass.
#include "fb_kernels.cuh"

namespace fb {

struct LmmArgs {
  const double* a;  // factor rows, row-major n × d
  int64_t n;
  int d;
  const double* x;  // d × dx, leading dimension ldx (this block's slice of X)
  int dx;
  int64_t ldx;
  int nfk;
  const int32_t* fk[kMaxParts];
  const double* z[kMaxParts];  // n_R,q × dx row-major
  double* out;                 // n × dx, leading dimension ldo
  int64_t ldo;
  int pitch;                   // shared-memory row pitch of the factor tile (doubles)
  int zstride;                 // doubles per z row (even: gathered rows are 16-byte bulk copies)
  int lanes;                   // rowdot: lanes per row (power of two)
  int cols;                    // rowdot: columns per lane (d / lanes)
  float zfrac;                 // z-pass (nfk == 0): evict_last fraction of the stored z rows
  int debug;                   // FB_LMM_DEBUG (measurement only): 1 skip stores, 4 plain stores
  int zcol0;                   // rowdot: first column of the gathered z rows this launch adds (sub-chunks)
  size_t ztable_bytes[kMaxParts];  // bytes of each z table (host side: gather cache choice)
};

// ------------------------------------------------------------------ rowdot (d_x <= 4)
// IT = rows each lane group handles per tile; their dot products run interleaved (IT
// independent FMA chains and shuffle trees) so the per-tile latency is one chain, not IT.
template <int NX, int IT>
__global__ void __launch_bounds__(kRingThreads, 1) lmm_rowdot_kernel(LmmArgs p, StreamSet ss, int stages,
                                                                     int tile_rows) {
  extern __shared__ __align__(128) char smem[];
  const int d = p.d;
  double* xs = reinterpret_cast<double*>(smem);  // X slice, d × NX row-major
  const size_t xs_bytes = (static_cast<size_t>(d > 0 ? d : 1) * NX * sizeof(double) + 127) & ~size_t(127);
  char* buf = smem + xs_bytes;
  for (int i = threadIdx.x; i < d * NX; i += blockDim.x) xs[i] = p.x[(i / NX) * p.ldx + (i % NX)];

  TileRing ring;
  ring.init(buf, stages, tile_rows, p.n);
  ring.start(ss);  // __syncthreads: xs visible
  if (ring.service(ss)) return;

  const int lane = lane_id();
  const int warp = consumer_warp();
  const int rw = tile_rows / kConsumerWarps;  // rows per warp per tile (<= 32)
  const int wrow = warp * rw;
  const int L = p.lanes, C = p.cols;
  const int rpi = 32 / L;                     // rows per instruction
  const int sub = lane % L, rsub = lane / L;
  const int src = (lane % rpi) * L;           // lane k takes row k: iteration k / rpi, group k % rpi
  const int myit = lane / rpi;
  const uint64_t pol = p.nfk == 0 ? policy_evict_last_frac(p.zfrac) : policy_evict_first();  // z stays in L2
  const double* xc = xs + sub * NX;

  for (int64_t kt = 0; kt < ring.count(); ++kt) {
    const int cur = ring.acquire(ss, kt);
    const int64_t tile = ring.tile_begin + kt;
    const int rows = ring.rows_of(tile);
    const int64_t r0 = tile * tile_rows;
    const double* A = reinterpret_cast<const double*>(ring.stage_ptr(cur, ss, 0));

    double acc[IT][NX];
    const double* arow[IT];
    bool live[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int rl = it * rpi + rsub;  // row within the warp's share
      live[it] = rl < rw && wrow + rl < rows;
      arow[it] = A + static_cast<size_t>(live[it] ? wrow + rl : 0) * p.pitch + sub;
#pragma unroll
      for (int j = 0; j < NX; ++j) acc[it][j] = 0.0;
    }
#pragma unroll 2
    for (int m = 0; m < C; ++m) {
      double xv[NX];
#pragma unroll
      for (int j = 0; j < NX; ++j) xv[j] = xc[m * L * NX + j];
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const double a = arow[it][m * L];
#pragma unroll
        for (int j = 0; j < NX; ++j) acc[it][j] = fma(a, xv[j], acc[it][j]);
      }
    }
    for (int o = L >> 1; o > 0; o >>= 1)
#pragma unroll
      for (int it = 0; it < IT; ++it)
#pragma unroll
        for (int j = 0; j < NX; ++j) acc[it][j] += __shfl_xor_sync(0xffffffffu, acc[it][j], o);
    double res[NX];
#pragma unroll
    for (int j = 0; j < NX; ++j) res[j] = 0.0;
#pragma unroll
    for (int it = 0; it < IT; ++it)
#pragma unroll
      for (int j = 0; j < NX; ++j) {
        const double v = __shfl_sync(0xffffffffu, acc[it][j], src);
        if (myit == it) res[j] = v;
      }
    const int r = wrow + lane;
    if (lane < rw && r < rows) {
      // + z_0[fk_0] + z_1[fk_1] ... in part order (rewrite.py:186-190), gathered into smem
      for (int q = 0; q < p.nfk; ++q) {
        const double* zr = reinterpret_cast<const double*>(ring.gather_ptr(cur, ss, q)) + r * p.zstride;
#pragma unroll
        for (int j = 0; j < NX; ++j) res[j] += zr[p.zcol0 + j];
      }
      double* o = p.out + (r0 + r) * p.ldo;
#pragma unroll
      for (int j = 0; j < NX; ++j) st_hint(o + j, res[j], pol);
    }
    ring.release();
  }
}

// ------------------------------------------------------------------ DMMA (5 <= d_x <= 16)
// KS = number of 4-wide k-steps when known at compile time (narrow factors: the whole
// k-loop unrolls into KS·MT·NT DMMAs with constant shared-memory offsets), 0 = runtime.
// The ncu source view of the runtime-loop version at c2 (d = 20, d_x = 16) showed ~480
// issued instructions per warp per 128-row tile for 20 DMMAs (row/k predicates, per-column
// bounds checks, address arithmetic): the SM issue slots, not HBM, bounded the pass.
// Rows past the end of a partial tile are computed on stale shared memory and simply not
// stored (DMMA row g of C depends only on row g of A), so the k-loop carries no row
// predicate; only the last k-step of a width that is not a multiple of 4 masks k >= d.
template <int NT, int MT, int KS, bool CG>
__global__ void __launch_bounds__(kRingThreads, 1) lmm_dmma_kernel(LmmArgs p, StreamSet ss, int stages,
                                                               int tile_rows) {
  extern __shared__ __align__(128) char smem[];
  const int d = p.d;
  const int dpad = KS > 0 ? 4 * KS : (d + 3) & ~3;
  constexpr int ldxs = 8 * NT + 4;  // bank skew for the B-fragment loads (see conflict_free_pitch)
  double* xs = reinterpret_cast<double*>(smem);
  const size_t xs_bytes = (static_cast<size_t>(dpad > 0 ? dpad : 4) * ldxs * sizeof(double) + 127) & ~size_t(127);
  char* buf = smem + xs_bytes;

  for (int i = threadIdx.x; i < dpad * ldxs; i += blockDim.x) {
    const int k = i / ldxs, n = i % ldxs;
    xs[i] = (k < d && n < p.dx) ? p.x[k * p.ldx + n] : 0.0;
  }

  TileRing ring;
  ring.init(buf, stages, tile_rows, p.n);
  ring.start(ss);  // contains __syncthreads (xs visible after it)
  if (ring.service<false, CG>(ss)) return;

  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  const int warp = consumer_warp();
  const int pitch = p.pitch;
  const int wrow = warp * (8 * MT);
  const uint64_t pol = p.nfk == 0 ? policy_evict_last_frac(p.zfrac) : policy_evict_first();
  const bool ragged_k = (d & 3) != 0;
  // every output column pair present and 16-byte aligned: one v2 store per pair
  const bool full_cols = p.dx == 8 * NT && (p.ldo & 1) == 0 && (reinterpret_cast<uintptr_t>(p.out) & 15u) == 0;
  const double* xb = xs + t * ldxs + g;  // this lane's B-fragment column
  const int zst = p.zstride;

  for (int64_t kt = 0; kt < ring.count(); ++kt) {
    const int cur = ring.acquire(ss, kt);
    const int64_t tile = ring.tile_begin + kt;
    const int rows = ring.rows_of(tile);
    const int64_t r0 = tile * tile_rows;
    const double* A = reinterpret_cast<const double*>(ring.stage_ptr(cur, ss, 0)) + (wrow + g) * pitch + t;

    __syncwarp();  // mma.sync.aligned needs the whole warp converged (after the barrier spin)
    if (wrow < rows) {
      double acc[MT][NT][2];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;

      auto kstep = [&](int k0, bool mask) {
        double b[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) b[nt] = xb[k0 * ldxs + 8 * nt];
        const bool on = !mask || k0 + t < d;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const double a = on ? A[8 * mt * pitch + k0] : 0.0;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], a, b[nt]);
        }
      };
      if constexpr (KS > 0) {
#pragma unroll
        for (int s = 0; s < KS - 1; ++s) kstep(4 * s, false);
        kstep(4 * (KS - 1), ragged_k);
      } else {
        for (int k0 = 0; k0 < dpad; k0 += 4) kstep(k0, ragged_k && k0 + 4 > d);
      }

      // epilogue: + z_0 + z_1 ... in part order (rewrite.py:186-190), then store
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int r = wrow + 8 * mt + g;
        if (r >= rows) continue;
        double* o = p.out + (r0 + r) * p.ldo;
        if (full_cols) {
          for (int q = 0; q < p.nfk; ++q) {
            const double* zr = reinterpret_cast<const double*>(ring.gather_ptr(cur, ss, q)) + r * zst + 2 * t;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const double2 zv = *reinterpret_cast<const double2*>(zr + 8 * nt);
              acc[mt][nt][0] += zv.x;
              acc[mt][nt][1] += zv.y;
            }
          }
          if (p.debug & 1) continue;
          if (p.debug & 4) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
              *reinterpret_cast<double2*>(o + 8 * nt + 2 * t) = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
            continue;
          }
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) st_hint2(o + 8 * nt + 2 * t, acc[mt][nt][0], acc[mt][nt][1], pol);
          continue;
        }
        for (int q = 0; q < p.nfk; ++q) {
          const double* zr = reinterpret_cast<const double*>(ring.gather_ptr(cur, ss, q)) + r * zst;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const int c = 8 * nt + 2 * t;
            if (c < p.dx) acc[mt][nt][0] += zr[c];
            if (c + 1 < p.dx) acc[mt][nt][1] += zr[c + 1];
          }
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int c = 8 * nt + 2 * t;
          if (c + 1 < p.dx && ((reinterpret_cast<uintptr_t>(o + c) & 15u) == 0)) {
            st_hint2(o + c, acc[mt][nt][0], acc[mt][nt][1], pol);
          } else {
            if (c < p.dx) st_hint(o + c, acc[mt][nt][0], pol);
            if (c + 1 < p.dx) st_hint(o + c + 1, acc[mt][nt][1], pol);
          }
        }
      }
    }
    ring.release();
  }
}

// ------------------------------------------------------------------ DMMA, z-initialised accumulators
// The common case of the S pass (every output column present and 16-byte aligned, d_x = 8·NT,
// at least one keyed part, narrow S so the k-loop is unrolled): the accumulators start from the
// gathered z rows (the C-fragment layout of m8n8k4 — lane (g, t) owns C[g][2t, 2t+1] — is
// exactly a double2 of a z row), so the epilogue is the stores alone; the X fragments are
// loaded once per CTA into registers; full tiles store without row predicates. ncu of the
// generic body at c2 X100x16: ~420 issued instructions per warp per 256-row tile (z adds,
// part loop, per-row bounds, debug switches) for 40 DMMAs, and the consumers' DADD chains on
// the z loads sat on the critical path of every tile.
// Parts after the first are added before the DMMAs (sum order z_0 + z_1 + ... then + S·X).
template <int NT, int MT, int KS, bool CG>
__global__ void __launch_bounds__(kRingThreads, 1) lmm_dmma_zinit_kernel(LmmArgs p, StreamSet ss, int stages,
                                                                     int tile_rows) {
  static_assert(KS > 0, "the z-initialised body needs a compile-time k-loop");
  extern __shared__ __align__(128) char smem[];
  const int d = p.d;
  constexpr int dpad = 4 * KS;
  constexpr int ldxs = 8 * NT + 4;
  double* xs = reinterpret_cast<double*>(smem);
  const size_t xs_bytes = (static_cast<size_t>(dpad) * ldxs * sizeof(double) + 127) & ~size_t(127);
  char* buf = smem + xs_bytes;
  for (int i = threadIdx.x; i < dpad * ldxs; i += blockDim.x) {
    const int k = i / ldxs, n = i % ldxs;
    xs[i] = (k < d && n < p.dx) ? p.x[k * p.ldx + n] : 0.0;
  }

  TileRing ring;
  ring.init(buf, stages, tile_rows, p.n);
  ring.start(ss);  // contains __syncthreads (xs visible after it)
  if (ring.service<false, CG>(ss)) return;

  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  const int warp = consumer_warp();
  const int pitch = p.pitch;
  const int wrow = warp * (8 * MT);
  const uint64_t pol = policy_evict_first();
  const bool ragged_k = (d & 3) != 0;
  const int zst = p.zstride;
  const int nfk = p.nfk;
  double bf[KS][NT];  // B fragments: X[4s + t][8nt + g], zero past d
#pragma unroll
  for (int s = 0; s < KS; ++s)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) bf[s][nt] = xs[(4 * s + t) * ldxs + 8 * nt + g];
  const int a_off = (wrow + g) * pitch + t;
  const int z_off = (wrow + g) * zst + 2 * t;

  for (int64_t kt = 0; kt < ring.count(); ++kt) {
    const int cur = ring.acquire(ss, kt);
    const int64_t tile = ring.tile_begin + kt;
    const int rows = ring.rows_of(tile);
    const double* A = reinterpret_cast<const double*>(ring.stage_ptr(cur, ss, 0)) + a_off;
    __syncwarp();  // mma.sync.aligned needs the whole warp converged (after the barrier spin)
    if (wrow < rows) {
      double acc[MT][NT][2];
      {
        const double* z0 = reinterpret_cast<const double*>(ring.gather_ptr(cur, ss, 0)) + z_off;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const double2 zv = *reinterpret_cast<const double2*>(z0 + 8 * mt * zst + 8 * nt);
            acc[mt][nt][0] = zv.x;
            acc[mt][nt][1] = zv.y;
          }
      }
      for (int q = 1; q < nfk; ++q) {
        const double* zq = reinterpret_cast<const double*>(ring.gather_ptr(cur, ss, q)) + z_off;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const double2 zv = *reinterpret_cast<const double2*>(zq + 8 * mt * zst + 8 * nt);
            acc[mt][nt][0] += zv.x;
            acc[mt][nt][1] += zv.y;
          }
      }
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        const bool on = !(s == KS - 1 && ragged_k) || 4 * s + t < d;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const double a = on ? A[8 * mt * pitch + 4 * s] : 0.0;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], a, bf[s][nt]);
        }
      }
      double* o = p.out + (tile * tile_rows + wrow + g) * p.ldo + 2 * t;
      if (rows == tile_rows) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
            st_hint2(o + 8 * mt * p.ldo + 8 * nt, acc[mt][nt][0], acc[mt][nt][1], pol);
      } else {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          if (wrow + 8 * mt + g >= rows) continue;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
            st_hint2(o + 8 * mt * p.ldo + 8 * nt, acc[mt][nt][0], acc[mt][nt][1], pol);
        }
      }
    }
    ring.release();
  }
}

// ------------------------------------------------------------------ host launchers
static size_t ring_budget() {
  static size_t b = [] {
    const char* e = getenv("FB_RING_BUDGET_KB");
    return static_cast<size_t>(e ? atoi(e) : 200) * 1024;
  }();
  return b;
}

static int stages_for(size_t fixed, uint32_t stage_bytes, int max_stages, size_t budget) {
  if (fixed + kRingHeader + 2 * static_cast<size_t>(stage_bytes) > budget) return 0;
  int st = static_cast<int>((budget - fixed - kRingHeader) / stage_bytes);
  return st > max_stages ? max_stages : st;
}

template <class K>
static cudaError_t launch_ring(K kern, const LmmArgs& p, StreamSet& ss, size_t fixed, int tile_rows,
                               cudaStream_t st, int num_sms, size_t budget = 0) {
  stream_layout(ss, tile_rows, p.n);
  const int stages = stages_for(fixed, ss.stage_bytes, 8, budget ? budget : ring_budget());
  if (stages < 2) return cudaErrorNotSupported;
  const size_t smem = fixed + kRingHeader + static_cast<size_t>(stages) * ss.stage_bytes;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int per_sm = static_cast<int>((228 * 1024) / (smem + 1024));
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 4) per_sm = 4;
  const int64_t ntiles = (p.n + tile_rows - 1) / tile_rows;
  const int grid = grid_for(ntiles, 1, per_sm, num_sms);
  kern<<<grid, kRingThreads, smem, st>>>(p, ss, stages, tile_rows);
  FB_LAUNCHED();
  return cudaGetLastError();
}

// z-pass stores: evict_last for this fraction of the z lines (FB_ZSTORE_FRAC overrides it,
// measurement only: fractions 0.5-1.0, with or without evict_last gathers, all timed the c2
// X100x16 S pass within 2% of each other)
static float z_store_frac() {
  static float f = [] {
    const char* e = getenv("FB_ZSTORE_FRAC");
    return e ? static_cast<float>(atof(e)) : 1.0f;
  }();
  return f;
}

// The ring carries the factor rows; the FK columns are read by the gatherer warps only
// (keys straight from global memory), which copy z[fk] rows into the stage.
static void fill_streams(const LmmArgs& p, StreamSet& ss, int pitch) {
  ss = StreamSet{};
  ss.count = 1;
  ss.base[0] = reinterpret_cast<const char*>(p.a);
  ss.row_bytes[0] = static_cast<uint32_t>(p.d) * 8u;
  ss.pitch[0] = static_cast<uint32_t>(pitch) * 8u;
  for (int q = 0; q < p.nfk; ++q) {
    ss.gkeys[q] = p.fk[q];
    ss.gbase[q] = reinterpret_cast<const char*>(p.z[q]);
    ss.grow_bytes[q] = static_cast<uint32_t>(p.zstride) * 8u;
  }
  ss.ngather = (p.debug & 2) ? 0 : p.nfk;
}

template <int NX>
static cudaError_t launch_rowdot(LmmArgs p, cudaStream_t st, int num_sms) {
  // lanes per row: largest power of two dividing d (<= 32), so half-warp loads are conflict-free
  int L = 1;
  while (p.d > 0 && L < 32 && (p.d % (2 * L)) == 0) L *= 2;
  p.lanes = L;
  p.cols = p.d / L;
  p.pitch = p.d;
  const uint32_t row_bytes = static_cast<uint32_t>(p.d) * 8u + 8u * p.zstride * p.nfk;
  // rows per warp per tile: 32, fewer for wide rows (stage <= ~44 KB)
  int rw = 32;
  while (rw > 4 && static_cast<size_t>(row_bytes) * rw * kConsumerWarps > 48 * 1024) rw >>= 1;
  // a lane group takes at most 8 interleaved rows per tile (the widest instantiation below): widths
  // 16 and 32 (L = 16 / 32 with rows short enough for rw = 32) would need 16 / 32 — their rows past
  // the eighth were never computed (found by tests/test_fuzz_gpu.py, round 2)
  while (rw > 1 && rw * L > 8 * 32) rw >>= 1;
  StreamSet ss;
  fill_streams(p, ss, p.d);
  const size_t fixed = (static_cast<size_t>(p.d > 0 ? p.d : 1) * NX * 8 + 127) & ~size_t(127);
  const int it = (rw * L + 31) / 32;  // rows per lane group per tile
  if (it <= 1) return launch_ring(lmm_rowdot_kernel<NX, 1>, p, ss, fixed, rw * kConsumerWarps, st, num_sms);
  if (it <= 2) return launch_ring(lmm_rowdot_kernel<NX, 2>, p, ss, fixed, rw * kConsumerWarps, st, num_sms);
  if (it <= 4) return launch_ring(lmm_rowdot_kernel<NX, 4>, p, ss, fixed, rw * kConsumerWarps, st, num_sms);
  return launch_ring(lmm_rowdot_kernel<NX, 8>, p, ss, fixed, rw * kConsumerWarps, st, num_sms);
}

template <int NT, int MT, int KS>
static cudaError_t launch_dmma_cfg(LmmArgs p, cudaStream_t st, int num_sms, size_t budget = 0) {
  // uniform keys into a table far beyond L1 (largest z > 32 MB): L1-bypassing gathers
  size_t zmax = 0;
  for (int q = 0; q < p.nfk; ++q) zmax = p.ztable_bytes[q] > zmax ? p.ztable_bytes[q] : zmax;
  const bool cg = zmax > (32u << 20);
  const int tile_rows = kConsumerWarps * 8 * MT;
  // dense rows (one bulk copy per tile): a padded pitch needs one copy per row, which costs
  // more than the 8-way A-fragment bank conflicts of a width ≡ 0 (mod 16)
  p.pitch = p.d;
  StreamSet ss;
  fill_streams(p, ss, p.pitch);
  const int dpad = (p.d + 3) & ~3;
  const size_t fixed = (static_cast<size_t>(dpad > 0 ? dpad : 4) * (8 * NT + 4) * 8 + 127) & ~size_t(127);
  static const bool zinit_on = [] { const char* e = getenv("FB_LMM_ZINIT"); return !(e && atoi(e) == 0); }();
  if constexpr (KS > 0) {
    const bool zinit = zinit_on && p.nfk > 0 && p.dx == 8 * NT && p.zstride >= 8 * NT && (p.ldo & 1) == 0 &&
                       (reinterpret_cast<uintptr_t>(p.out) & 15u) == 0 && p.debug == 0;
    if (zinit && cg) return launch_ring(lmm_dmma_zinit_kernel<NT, MT, KS, true>, p, ss, fixed, tile_rows, st, num_sms, budget);
    if (zinit) return launch_ring(lmm_dmma_zinit_kernel<NT, MT, KS, false>, p, ss, fixed, tile_rows, st, num_sms, budget);
  }
  if (cg) return launch_ring(lmm_dmma_kernel<NT, MT, KS, true>, p, ss, fixed, tile_rows, st, num_sms, budget);
  return launch_ring(lmm_dmma_kernel<NT, MT, KS, false>, p, ss, fixed, tile_rows, st, num_sms, budget);
}

// narrow factors (d <= 32, the multi-row tile configurations): the k-step count is a
// template parameter so the k-loop unrolls completely
template <int NT, int MT>
static cudaError_t launch_dmma_ks(const LmmArgs& p, cudaStream_t st, int num_sms, size_t budget = 0) {
  switch ((p.d + 3) / 4) {
    case 1: return launch_dmma_cfg<NT, MT, 1>(p, st, num_sms, budget);
    case 2: return launch_dmma_cfg<NT, MT, 2>(p, st, num_sms, budget);
    case 3: return launch_dmma_cfg<NT, MT, 3>(p, st, num_sms, budget);
    case 4: return launch_dmma_cfg<NT, MT, 4>(p, st, num_sms, budget);
    case 5: return launch_dmma_cfg<NT, MT, 5>(p, st, num_sms, budget);
    case 6: return launch_dmma_cfg<NT, MT, 6>(p, st, num_sms, budget);
    case 7: return launch_dmma_cfg<NT, MT, 7>(p, st, num_sms, budget);
    case 8: return launch_dmma_cfg<NT, MT, 8>(p, st, num_sms, budget);
    default: return launch_dmma_cfg<NT, MT, 0>(p, st, num_sms, budget);
  }
}

template <int NT>
static cudaError_t launch_dmma(const LmmArgs& p, cudaStream_t st, int num_sms) {
  const size_t row_bytes = static_cast<size_t>(p.d) * 8 + 8 * static_cast<size_t>(p.zstride) * p.nfk;
  // The consumers are latency-bound on the DMMA chains (c2 X100x16 with z L2-resident: 1.24 ms
  // with 2 m-tiles per warp, 1.10 ms with 4; ncu: 'wait' / 'math' stalls in the k-loop), so
  // prefer 4 m-tiles (8 independent accumulators per warp) even when that makes a stage
  // ~74 KB (S rows + gathered z rows): three stages in a 224 KB ring.
  static int mt = [] { const char* e = getenv("FB_LMM_MT"); return e ? atoi(e) : 0; }();
  const size_t big = 224 * 1024;
  if (mt == 4 && p.nfk > 0) return launch_dmma_ks<NT, 4>(p, st, num_sms, big);
  if (mt == 2 && p.nfk > 0 && row_bytes * 128 <= 48 * 1024) return launch_dmma_ks<NT, 2>(p, st, num_sms);
  if (mt == 1 && p.nfk > 0) return launch_dmma_ks<NT, 1>(p, st, num_sms);
  if (row_bytes * 256 <= 48 * 1024) return launch_dmma_ks<NT, 4>(p, st, num_sms);
  if (mt == 0 && p.nfk > 0 && row_bytes * 256 <= 76 * 1024) return launch_dmma_ks<NT, 4>(p, st, num_sms, big);
  if (row_bytes * 128 <= 48 * 1024) return launch_dmma_ks<NT, 2>(p, st, num_sms);
  return launch_dmma_cfg<NT, 1, 0>(p, st, num_sms);
}

cudaError_t launch_lmm_rows(const double* a, int64_t n, int d, const double* x, int dx, int64_t ldx,
                            int nfk, const int32_t* const* fk, const double* const* z, int zstride, double* out,
                            int64_t ldo, cudaStream_t st, int num_sms, const int64_t* z_rows) {
  if (n <= 0) return cudaSuccess;
  if (dx < 1 || dx > 16) return cudaErrorNotSupported;
  LmmArgs p{};
  p.a = a;
  p.n = n;
  p.d = d;
  p.x = x;
  p.dx = dx;
  p.ldx = ldx;
  p.nfk = nfk;
  for (int q = 0; q < nfk; ++q) {
    p.fk[q] = fk[q];
    p.z[q] = z[q];
    p.ztable_bytes[q] = z_rows ? static_cast<size_t>(z_rows[q]) * zstride * sizeof(double) : 0;
  }
  p.zstride = zstride;
  if (nfk > 0 && (zstride < dx || (zstride & 1))) return cudaErrorInvalidValue;
  p.out = out;
  p.ldo = ldo;
  p.zfrac = z_store_frac();
  static int dbg = [] { const char* e = getenv("FB_LMM_DEBUG"); return e ? atoi(e) : 0; }();
  p.debug = nfk > 0 ? dbg : 0;
  switch (dx) {
    case 1:
      return launch_rowdot<1>(p, st, num_sms);
    case 2:
      return launch_rowdot<2>(p, st, num_sms);
    case 3:
      return launch_rowdot<3>(p, st, num_sms);
    case 4:
      return launch_rowdot<4>(p, st, num_sms);
    default:
      break;
  }
  cudaError_t e = dx <= 8 ? launch_dmma<1>(p, st, num_sms) : launch_dmma<2>(p, st, num_sms);
  if (e != cudaErrorNotSupported) return e;
  // Two 64-row DMMA stages of a wide factor (d above ~170, less with gathered z rows) do not fit
  // the ring: the same product in column sub-chunks of <= 4 on the rowdot kernel, whose tiles
  // shrink to 4 rows per warp (found by the wide fixtures of tests/test_fuzz_gpu.py)
  for (int c0 = 0; c0 < dx; c0 += 4) {
    LmmArgs q = p;
    q.x = p.x + c0;
    q.out = p.out + c0;
    q.dx = dx - c0 < 4 ? dx - c0 : 4;
    q.zcol0 = c0;
    switch (q.dx) {
      case 1: e = launch_rowdot<1>(q, st, num_sms); break;
      case 2: e = launch_rowdot<2>(q, st, num_sms); break;
      case 3: e = launch_rowdot<3>(q, st, num_sms); break;
      default: e = launch_rowdot<4>(q, st, num_sms); break;
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace fb
