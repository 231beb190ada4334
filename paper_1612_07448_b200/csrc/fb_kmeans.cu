// fb_kmeans.cu — one fused pass over S per K-Means iteration.
//
// Replaces, for the rows of S, the body of the reference's K-Means loop (ml.py:275-283):
//   dist = d_t + Σ_r c² − (2T)·C ;  a = row_min_mask(dist) ;  trace += Σ dist·a ;
//   sizes = Σ a ;  TᵀA = [SᵀA ; R_qᵀ (K_qᵀ A)]
// The reference evaluates it as four whole-matrix steps (an n × k product written out, the
// mask, the objective, the transposed product). Here a single ring pass over S (fb_stream.cuh)
// does, per 8-row m-tile of a consumer warp:
//   1. T·(2C) on the FP64 tensor cores: the accumulators start from the gathered z_q[fk_q]
//      rows (z_q = R_q·(2C)_q from the z-pass, the LMM's "R·X before K" order,
//      rewrite.py:187-189), then S·(2C)_S by DMMA;
//   2. the argmin in registers: the 4 lanes holding a row's columns reduce (value, index)
//      with two xor shuffles, ties to the lowest index (kernel.py:327-339); a NaN distance
//      latches (iteration, row) as the first NaN row (kernel.py:332-334);
//   3. the objective (Σ of the row minima), the cluster sizes (shared-memory counters), and
//      the integer histograms K_qᵀA (one fire-and-forget REDG per row and part, exact);
//   4. SᵀA on the tensor cores from the same shared-memory S tile: the one-hot assignment
//      (k × rows) times the S rows (rows × d_S), accumulated per warp across its tiles.
// Nothing of size n × k touches HBM (the unfused path wrote and re-read T·(2C): 800 MB per
// c4 iteration, and read S a second time for SᵀA). The per-warp objective and SᵀA partials
// are summed in a fixed (CTA, warp) order by the last CTA, so the pass is deterministic.
// The R side (R_qᵀ H_q on the tensor cores) and the centroid update stay in fb_capi.cu.
#include "fb_kernels.cuh"

namespace fb {

namespace {
constexpr int kKmMaxK = 16;   // k <= 16: two 8-column DMMA n-tiles of T·C, two m-tiles of SᵀA
constexpr int kKmStaCols = 32;  // d_S <= 32 (KS <= 8)
constexpr int kKmPitch = 17;    // per-warp T·C tile row pitch (doubles): conflict-free column reads
}  // namespace

// shared memory ahead of the ring: (2C)_S fragments, Σc², the per-warp T·C tiles, sizes
__host__ __device__ inline size_t km_head_bytes(int ks, int mt) {
  const int dpad = ks > 0 ? 4 * ks : 4;
  return (static_cast<size_t>(dpad * 20 + kKmMaxK + kConsumerWarps * 8 * mt * kKmPitch) * 8 + kKmMaxK * 4 + 127) &
         ~size_t(127);
}

size_t kmeans_pass_partials_doubles(int num_sms) {
  return static_cast<size_t>(num_sms) * kConsumerWarps * (1 + kKmMaxK * kKmStaCols);
}

// RR: the rows come from an FK-band layout (fb_band_layout: S, d_t and the FK columns in band
// order) and the tiles are dealt round-robin, so all CTAs gather z_0 from one L2-resident band
// at a time; every result of the pass is a sum over rows or a per-row value stored in band
// order (the caller un-permutes the final assignment once).
template <int KS, int MT, bool CG, bool RR = false>
__global__ void __launch_bounds__(kRingThreads, 1) kmeans_pass_kernel(KmPass p, StreamSet ss, int stages,
                                                                  int tile_rows) {
  constexpr int NT2 = (4 * KS + 7) / 8;  // 8-column n-tiles of SᵀA over d_S
  constexpr int ldxs = 2 * 8 + 4;        // (2C)_S in shared memory, bank-skewed like the LMM
  constexpr int dpad = KS > 0 ? 4 * KS : 4;
  extern __shared__ __align__(128) char smem[];
  double* xs = reinterpret_cast<double*>(smem);
  double* ccs = xs + dpad * ldxs;
  double* wbuf_all = ccs + kKmMaxK;  // [8 warps][8·MT rows][kKmPitch]
  int* ssz = reinterpret_cast<int*>(wbuf_all + kConsumerWarps * 8 * MT * kKmPitch);
  const size_t head = km_head_bytes(KS, MT);
  char* buf = smem + head;
  const int d = p.d, k = p.k;
  for (int i = threadIdx.x; i < dpad * ldxs; i += blockDim.x) {
    const int r = i / ldxs, c = i % ldxs;
    xs[i] = (r < d && c < k) ? p.c2s[r * k + c] : 0.0;
  }
  for (int j = threadIdx.x; j < kKmMaxK; j += blockDim.x) {
    ccs[j] = j < k ? p.cc[j] : 0.0;
    ssz[j] = 0;
  }

  TileRingT<RR> ring;
  ring.init(buf, stages, tile_rows, p.n);
  ring.start(ss);  // __syncthreads: xs / ccs / ssz visible
  if (ring.template service<false, CG>(ss)) return;

  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  const int warp = consumer_warp();
  const int wrow = warp * (8 * MT);
  constexpr int ROWS = 8 * MT;        // rows per warp per tile
  constexpr int LPR = 32 / ROWS;      // lanes per row in the argmin scan
  const int my_row = lane % ROWS, my_part = lane / ROWS;
  double* wbuf = wbuf_all + warp * ROWS * kKmPitch;
  const int pitch = d;
  const int zst = p.zst;
  const bool ragged_k = (d & 3) != 0;
  double bf[KS > 0 ? KS : 1][2];
#pragma unroll
  for (int s = 0; s < KS; ++s)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) bf[s][nt] = xs[(4 * s + t) * ldxs + 8 * nt + g];
  double sta[2][NT2 > 0 ? NT2 : 1][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < (NT2 > 0 ? NT2 : 1); ++b) sta[a][b][0] = sta[a][b][1] = 0.0;
  double obj = 0.0;
  unsigned long long nan_first = ~0ull;
  const unsigned long long it_tag = static_cast<unsigned long long>(p.it) << 40;

  for (int64_t kt = 0; kt < ring.count(); ++kt) {
    const int cur = ring.acquire(ss, kt);
    const int64_t tile = ring.tile_of(kt);
    const int rows = ring.rows_of(tile);
    const int64_t r0 = tile * tile_rows;
    const double* S = reinterpret_cast<const double*>(ring.stage_ptr(cur, ss, 0));
    const double* dts = reinterpret_cast<const double*>(ring.stage_ptr(cur, ss, 1));
    __syncwarp();
    if (wrow < rows) {
      // 1. T·(2C): the accumulators start from z_0[fk_0] + z_1[fk_1] ... (parts in order), then
      // + S·(2C)_S on the tensor cores. (Running the S DMMAs before waiting for the gathered z
      // rows, with or without handing the z rows back to the gatherers early, measured 2-5%
      // slower at c4.)
      double acc[MT][2][2];
      {  // part 0 initialises (0 + z_0 = z_0), the others add: every load of a part issues before its adds
        const double* z0 = reinterpret_cast<const double*>(ring.gather_ptr(cur, ss, 0)) + (wrow + g) * zst;
        const bool has0 = p.nfk > 0;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            const int c = 8 * nt + 2 * t;
            double2 zv = make_double2(0.0, 0.0);
            if (has0 && c < zst) zv = *reinterpret_cast<const double2*>(z0 + 8 * mt * zst + c);
            acc[mt][nt][0] = zv.x;
            acc[mt][nt][1] = zv.y;
          }
      }
#pragma unroll
      for (int q = 1; q < kMaxParts; ++q) {
        if (q >= p.nfk) break;
        const double* zq = reinterpret_cast<const double*>(ring.gather_ptr(cur, ss, q)) + (wrow + g) * zst;
        double2 zv[MT][2];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            const int c = 8 * nt + 2 * t;
            zv[mt][nt] = c < zst ? *reinterpret_cast<const double2*>(zq + 8 * mt * zst + c) : make_double2(0.0, 0.0);
          }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            acc[mt][nt][0] += zv[mt][nt].x;
            acc[mt][nt][1] += zv[mt][nt].y;
          }
      }
      if constexpr (KS > 0) {
        const double* A = S + (wrow + g) * pitch + t;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          const bool on = !(s == KS - 1 && ragged_k) || 4 * s + t < d;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const double a = on ? A[8 * mt * pitch + 4 * s] : 0.0;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], a, bf[s][nt]);
          }
        }
      }
      // 2. + 3. argmin, objective, sizes, histograms: the C fragments go through a per-warp
      // shared-memory tile (row pitch 17: conflict-free column reads) so each row's k
      // distances are scanned by LPR lanes holding that row — no per-m-tile shuffle trees,
      // every lane busy, one coalesced store / REDG per row group
      __syncwarp();
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          double* w = wbuf + (8 * mt + g) * kKmPitch + 8 * nt + 2 * t;
          w[0] = acc[mt][nt][0];
          w[1] = acc[mt][nt][1];
        }
      __syncwarp();
      const int r = wrow + my_row;
      const bool live = r < rows;
      const double dt = live ? dts[r] : 0.0;
      const double* wr = wbuf + my_row * kKmPitch;
      double bv = __longlong_as_double(0x7ff0000000000000ll);  // +inf
      int bj = 1 << 30;
      bool nan = false;
      if constexpr (LPR == 1) {
        // the lane scans all k distances of its row. A running minimum is a chain of k dependent
        // compare + select pairs (ncu source view at c4: 41% of the consumers' stall samples sat
        // on these lines, two warps per scheduler cannot hide it): load every distance first,
        // then a pairwise tournament of depth 4 — the left entry of a pair holds the lower
        // indices and wins ties, so the result is np.argmin's (lowest index of the minimum)
        double v[kKmMaxK];
        int ix[kKmMaxK];
#pragma unroll
        for (int j = 0; j < kKmMaxK; ++j) {
          const double x = (dt + ccs[j]) - wr[j];  // (d_t + Σc²) − (2T)·C, ml.py:276
          nan |= j < k && x != x;
          v[j] = j < k ? x : bv;
          ix[j] = j;
        }
#pragma unroll
        for (int w = 1; w < kKmMaxK; w <<= 1)
#pragma unroll
          for (int j = 0; j + w < kKmMaxK; j += 2 * w) {
            const bool right = v[j + w] < v[j];
            v[j] = right ? v[j + w] : v[j];
            ix[j] = right ? ix[j + w] : ix[j];
          }
        bv = v[0];
        bj = ix[0];
      } else {
#pragma unroll
        for (int j0 = 0; j0 < kKmMaxK; j0 += LPR) {
          const int j = j0 + my_part;
          if (j < k) {
            const double v = (dt + ccs[j]) - wr[j];  // (d_t + Σc²) − (2T)·C, ml.py:276
            nan |= isnan(v);
            if (v < bv) {  // increasing j: ties keep the lowest index (np.argmin)
              bv = v;
              bj = j;
            }
          }
        }
      }
      if constexpr (LPR == 2) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, ROWS);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, ROWS);
        nan |= __shfl_xor_sync(0xffffffffu, static_cast<int>(nan), ROWS) != 0;
        if (ov < bv || (ov == bv && oj < bj)) {
          bv = ov;
          bj = oj;
        }
      }
      bj = bj < k ? bj : 0;  // a row of NaN distances compares false everywhere: keep the indices in range
      const int best = live ? bj : -1;  // lane my_row (part 0) owns row my_row's result
      if (live && my_part == 0) {
        const int64_t gr = r0 + r;
        if (nan) nan_first = min(nan_first, it_tag | static_cast<unsigned long long>(gr));
        p.assign[gr] = bj;
        obj += bv;
        atomicAdd(&ssz[bj], 1);
#pragma unroll
        for (int q = 0; q < kMaxParts; ++q) {
          if (q >= p.nfk) break;
          const int32_t key = reinterpret_cast<const int32_t*>(ring.stage_ptr(cur, ss, 2 + q))[r];
          red_add(p.bins[q] + static_cast<int64_t>(key) * k + bj, 1);
        }
      }
      // 4. SᵀA += onehot(a)ᵀ · S_tile on the tensor cores (k = 4 rows per step)
      if constexpr (KS > 0) {
#pragma unroll
        for (int s = 0; s < 2 * MT; ++s) {
          const int ar = __shfl_sync(0xffffffffu, best, 4 * s + t);  // row 4s+t's owner lane
          const int rl = wrow + 4 * s + t;
          const bool live = rl < rows;
          double b[NT2];
#pragma unroll
          for (int nt = 0; nt < NT2; ++nt) b[nt] = live ? S[rl * pitch + 8 * nt + g] : 0.0;
#pragma unroll
          for (int mt2 = 0; mt2 < 2; ++mt2) {
            const double a = ar == g + 8 * mt2 ? 1.0 : 0.0;
#pragma unroll
            for (int nt = 0; nt < NT2; ++nt) dmma_8x8x4(sta[mt2][nt][0], sta[mt2][nt][1], a, b[nt]);
          }
        }
      }
    }
    ring.release();
  }

  // per-warp partials -> shared memory (the ring is idle once every consumer left its loop),
  // summed over the 8 warps in order into one partial per CTA; the last CTA sums those in CTA
  // order (deterministic). Slot 0: objective; 1 + m·32 + n: SᵀA (cluster m, column n).
  constexpr int kSlots = 1 + kKmMaxK * kKmStaCols;
  double* red = reinterpret_cast<double*>(buf + kRingHeader);  // past the ring's mbarriers
  const int tid = consumer_tid();
  obj = warp_sum(obj);
  consumer_sync();
  double* mine = red + warp * kSlots;
  if (lane == 0) mine[0] = obj;
  if constexpr (KS > 0) {
#pragma unroll
    for (int mt2 = 0; mt2 < 2; ++mt2)
#pragma unroll
      for (int nt = 0; nt < NT2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) mine[1 + (8 * mt2 + g) * kKmStaCols + 8 * nt + 2 * t + e] = sta[mt2][nt][e];
  }
  if (nan_first != ~0ull) atomicMin(p.nan_row, nan_first);
  consumer_sync();
  const int used = KS > 0 ? kSlots : 1;
  for (int i = tid; i < used; i += kConsumerThreads) {
    double v = 0.0;
    for (int w = 0; w < kConsumerWarps; ++w) v += red[w * kSlots + i];
    p.partials[static_cast<size_t>(blockIdx.x) * used + i] = v;
  }
  for (int j = tid; j < k; j += kConsumerThreads)
    if (ssz[j]) red_add(p.sizes + j, ssz[j]);
  __threadfence();
  __shared__ unsigned ticket;
  consumer_sync();
  if (tid == 0) ticket = atomicAdd(p.counter, 1u);
  consumer_sync();
  if (ticket != gridDim.x - 1) return;
  __threadfence();
  // one thread per output, CTA partials added in CTA order (coalesced rows of the [CTA][slot] table)
  const int nout = KS > 0 ? 1 + d * k : 1;
  for (int o = tid; o < nout; o += kConsumerThreads) {
    const int slot = o == 0 ? 0 : 1 + ((o - 1) % k) * kKmStaCols + (o - 1) / k;  // o-1 = c·k + j
    double v = 0.0;
#pragma unroll 8
    for (int b = 0; b < static_cast<int>(gridDim.x); ++b) v += __ldcg(p.partials + static_cast<size_t>(b) * used + slot);
    if (o == 0)
      p.trace[p.it] = v;
    else
      p.sta[o - 1] = v;
  }
  if (tid == 0) *p.counter = 0u;
}

template <int KS, int MT, bool CG, bool RR = false>
static cudaError_t launch_km(const KmPass& p, cudaStream_t st, int num_sms) {
  const int tile_rows = kConsumerWarps * 8 * MT;
  StreamSet ss{};
  ss.count = 2 + p.nfk;
  ss.base[0] = reinterpret_cast<const char*>(p.s);
  ss.row_bytes[0] = static_cast<uint32_t>(p.d) * 8u;
  ss.base[1] = reinterpret_cast<const char*>(p.d_t);
  ss.row_bytes[1] = 8u;
  for (int q = 0; q < p.nfk; ++q) {
    ss.base[2 + q] = reinterpret_cast<const char*>(p.fk[q]);
    ss.row_bytes[2 + q] = 4u;
    ss.gkeys[q] = p.fk[q];
    ss.gbase[q] = reinterpret_cast<const char*>(p.z[q]);
    ss.grow_bytes[q] = static_cast<uint32_t>(p.zst) * 8u;
  }
  ss.ngather = p.nfk;
  for (int i = 0; i < ss.count; ++i) ss.pitch[i] = ss.row_bytes[i];
  stream_layout(ss, tile_rows, p.n);
  const size_t head = km_head_bytes(KS, MT);
  const size_t budget = 224 * 1024;
  int stages = static_cast<int>((budget - head - kRingHeader) / ss.stage_bytes);
  if (stages > 8) stages = 8;
  if (stages < 2) return cudaErrorNotSupported;
  const size_t smem = head + kRingHeader + static_cast<size_t>(stages) * ss.stage_bytes;
  auto kern = kmeans_pass_kernel<KS, MT, CG, RR>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int64_t ntiles = (p.n + tile_rows - 1) / tile_rows;
  const int grid = grid_for(ntiles, 1, 1, num_sms);
  kern<<<grid, kRingThreads, smem, st>>>(p, ss, stages, tile_rows);
  FB_LAUNCHED();
  return cudaGetLastError();
}

template <int MT, bool CG, bool RR = false>
static cudaError_t launch_km_ks(const KmPass& p, cudaStream_t st, int num_sms) {
  {
    switch ((p.d + 3) / 4) {
      case 0: return launch_km<0, MT, CG, RR>(p, st, num_sms);
      case 1: return launch_km<1, MT, CG, RR>(p, st, num_sms);
      case 2: return launch_km<2, MT, CG, RR>(p, st, num_sms);
      case 3: return launch_km<3, MT, CG, RR>(p, st, num_sms);
      case 4: return launch_km<4, MT, CG, RR>(p, st, num_sms);
      case 5: return launch_km<5, MT, CG, RR>(p, st, num_sms);
      case 6: return launch_km<6, MT, CG, RR>(p, st, num_sms);
      case 7: return launch_km<7, MT, CG, RR>(p, st, num_sms);
      case 8: return launch_km<8, MT, CG, RR>(p, st, num_sms);
      default: return cudaErrorNotSupported;
    }
  }
}

// 32 rows per consumer warp (256-row tiles, two stages at c4): measured 1.36 ms per c4
// iteration against 1.50 / 1.58 ms with 16 / 24 rows (fewer rows leave the per-tile argmin and
// barrier latency exposed)
template <bool CG>
static cudaError_t launch_km_cg(const KmPass& p, cudaStream_t st, int num_sms) {
  return launch_km_ks<4, CG>(p, st, num_sms);
}

// Shape limits of the fused pass and room for two ring stages of 256 rows (S, d_t, the FK columns and
// the gathered z rows of every part): wide stars (three parts at k > 8, two parts with a wide S)
// do not fit and take the operator-by-operator step. (Until the randomised-fixture suite of round 2
// this tested the shape limits only and the launch then failed with "unsupported size".)
bool kmeans_pass_supported(int d_s, int k, int nfk) {
  if (!(k >= 1 && k <= kKmMaxK && d_s >= 0 && d_s <= kKmStaCols && nfk >= 0 && nfk <= kMaxParts)) return false;
  constexpr int MT = 4;
  StreamSet ss{};
  ss.count = 2 + nfk;
  ss.row_bytes[0] = static_cast<uint32_t>(d_s) * 8u;
  ss.row_bytes[1] = 8u;
  for (int q = 0; q < nfk; ++q) {
    ss.row_bytes[2 + q] = 4u;
    ss.grow_bytes[q] = static_cast<uint32_t>(z_stride(k)) * 8u;
  }
  ss.ngather = nfk;
  for (int i = 0; i < ss.count; ++i) ss.pitch[i] = ss.row_bytes[i];
  stream_layout(ss, kConsumerWarps * 8 * MT, kConsumerWarps * 8 * MT);
  const size_t head = km_head_bytes((d_s + 3) / 4, MT);
  const size_t budget = 224 * 1024;
  return ss.stage_bytes > 0 && head + kRingHeader + 2 * static_cast<size_t>(ss.stage_bytes) <= budget;
}

cudaError_t launch_kmeans_pass(const KmPass& p, cudaStream_t st, int num_sms) {
  if (!kmeans_pass_supported(p.d, p.k, p.nfk) || p.n <= 0) return cudaErrorNotSupported;
  size_t zmax = 0;
  for (int q = 0; q < p.nfk; ++q) zmax = p.ztable_bytes[q] > zmax ? p.ztable_bytes[q] : zmax;
  cudaError_t e = cudaMemsetAsync(p.counter, 0, sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  if (p.rr) return launch_km_ks<4, true, true>(p, st, num_sms);  // band layouts exist only for big z tables
  // uniform keys into a table far beyond L1: L1-bypassing gathers (as the LMM S pass)
  return zmax > (32u << 20) ? launch_km_cg<true>(p, st, num_sms) : launch_km_cg<false>(p, st, num_sms);
}

// ------------------------------------------------------------------ R_qᵀ H_q (K-Means R side)
// out(c, j) = Σ_r R[r, c] · H[r, j] for the integer histograms H_q = K_qᵀA (n_R × k int32):
// ml.py:279's TᵀA for an attribute block, R_qᵀ(K_qᵀA). One ring pass over R and H on the FP64
// tensor cores (rows are the DMMA k dimension: A = Rᵀ fragments, B = H fragments converted
// from int32 in registers), per-warp accumulators summed in a fixed order by the last CTA.
// The generic Gram engine (launch_rtx) spent 249 µs on c4's R1 (1M × 40, k = 10): one bulk
// copy per padded row; this reads both streams densely.
size_t rth_partials_doubles(int num_sms) { return static_cast<size_t>(num_sms) * kConsumerWarps * 64 * 16; }
bool rth_supported(int d_r, int nx) { return d_r >= 1 && d_r <= 64 && nx >= 1 && nx <= 16; }

template <int MTR, int RPW, typename WT>
__global__ void __launch_bounds__(kRingThreads, 1) rth_kernel(const double* __restrict__ rr, int64_t n, int d_r,
                                                          const WT* __restrict__ h, int nx, double* out,
                                                          int64_t o_rs, int64_t o_cs, double* partials,
                                                          StreamSet ss, int stages, int tile_rows) {
  extern __shared__ __align__(128) char smem[];
  TileRing ring;
  ring.init(smem, stages, tile_rows, n);
  ring.start(ss);
  if (ring.service(ss)) return;
  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  const int warp = consumer_warp();
  const int wrow = warp * RPW;
  double acc[MTR][2][2];
#pragma unroll
  for (int mt = 0; mt < MTR; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  for (int64_t kt = 0; kt < ring.count(); ++kt) {
    const int cur = ring.acquire(ss, kt);
    const int rows = ring.rows_of(ring.tile_begin + kt);
    const double* R = reinterpret_cast<const double*>(ring.stage_ptr(cur, ss, 0));
    const WT* H = reinterpret_cast<const WT*>(ring.stage_ptr(cur, ss, 1));
    __syncwarp();
    if (wrow < rows) {
      const bool full = wrow + RPW <= rows;
#pragma unroll
      for (int s = 0; s < RPW / 4; ++s) {
        const int rl = wrow + 4 * s + t;
        const bool live = full || rl < rows;  // dead rows: zero both operands (stale smem may be NaN)
        double b[2];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const int j = 8 * nt + g;
          b[nt] = (live && j < nx) ? static_cast<double>(H[rl * nx + j]) : 0.0;
        }
#pragma unroll
        for (int mt = 0; mt < MTR; ++mt) {
          const double a = live ? R[rl * d_r + 8 * mt + g] : 0.0;  // columns >= d_r only feed discarded rows
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], a, b[nt]);
        }
      }
    }
    ring.release();
  }
  // per-warp partials -> shared memory -> one partial per CTA (warps in order); the CTA
  // partials are summed in CTA order by rth_reduce_kernel
  double* red = reinterpret_cast<double*>(smem + kRingHeader);  // past the ring's mbarriers
  const int tid = consumer_tid();
  consumer_sync();
#pragma unroll
  for (int mt = 0; mt < MTR; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) red[warp * (8 * MTR * 16) + (8 * mt + g) * 16 + 8 * nt + 2 * t + e] = acc[mt][nt][e];
  consumer_sync();
  for (int i = tid; i < 8 * MTR * 16; i += kConsumerThreads) {
    double v = 0.0;
    for (int w = 0; w < kConsumerWarps; ++w) v += red[w * (8 * MTR * 16) + i];
    partials[static_cast<size_t>(blockIdx.x) * (8 * MTR * 16) + i] = v;
  }
}

// out(c, j) = Σ_b partials[b][c·16 + j] in CTA order b = 0, 1, ...: a warp per output (lanes
// take CTAs b ≡ lane mod 32 in order, then a fixed xor tree) — a single last CTA summing the
// 600 outputs of c4's R2 one thread each took ~40 µs of dependent L2 round trips.
__global__ void rth_reduce_kernel(const double* __restrict__ partials, int nb, int stride, int d_r, int nx,
                                  double* out, int64_t o_rs, int64_t o_cs) {
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (e >= d_r * nx) return;
  const int c = e / nx, j = e % nx;
  const double v = warp_sum_strided(partials + c * 16 + j, nb, static_cast<size_t>(stride));
  if ((threadIdx.x & 31) == 0) out[c * o_rs + j * o_cs] = v;
}

template <int MTR, int RPW, typename WT>
static cudaError_t launch_rth_rpw(const double* r, int64_t n, int d_r, const WT* h, int nx, double* out,
                                 int64_t o_rs, int64_t o_cs, double* partials, unsigned* counter, cudaStream_t st,
                                 int num_sms) {
  const int tile_rows = kConsumerWarps * RPW;
  StreamSet ss{};
  ss.count = 2;
  ss.base[0] = reinterpret_cast<const char*>(r);
  ss.row_bytes[0] = ss.pitch[0] = static_cast<uint32_t>(d_r) * 8u;
  ss.base[1] = reinterpret_cast<const char*>(h);
  ss.row_bytes[1] = ss.pitch[1] = static_cast<uint32_t>(nx * sizeof(WT));
  stream_layout(ss, tile_rows, n);
  const size_t budget = 200 * 1024;
  int stages = static_cast<int>((budget - kRingHeader) / ss.stage_bytes);
  if (stages > 8) stages = 8;
  if (stages < 2) return cudaErrorNotSupported;
  const size_t smem = kRingHeader + static_cast<size_t>(stages) * ss.stage_bytes;
  auto kern = rth_kernel<MTR, RPW, WT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  (void)counter;
  const int64_t ntiles = (n + tile_rows - 1) / tile_rows;
  const int grid = grid_for(ntiles, 1, 1, num_sms);
  kern<<<grid, kRingThreads, smem, st>>>(r, n, d_r, h, nx, out, o_rs, o_cs, partials, ss, stages, tile_rows);
  FB_LAUNCHED();
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int nout = d_r * nx;
  rth_reduce_kernel<<<(nout + 7) / 8, 256, 0, st>>>(partials, grid, 8 * MTR * 16, d_r, nx, out, o_rs, o_cs);
  FB_LAUNCHED();
  return cudaGetLastError();
}

// 32 rows per warp while a 256-row stage stays <= 64 KB (three stages in flight), else 16
template <int MTR, typename WT>
static cudaError_t launch_rth_mt(const double* r, int64_t n, int d_r, const WT* h, int nx, double* out,
                                 int64_t o_rs, int64_t o_cs, double* partials, unsigned* counter, cudaStream_t st,
                                 int num_sms) {
  if (256 * (8 * d_r + static_cast<int>(sizeof(WT)) * nx) <= 64 * 1024)
    return launch_rth_rpw<MTR, 32, WT>(r, n, d_r, h, nx, out, o_rs, o_cs, partials, counter, st, num_sms);
  return launch_rth_rpw<MTR, 16, WT>(r, n, d_r, h, nx, out, o_rs, o_cs, partials, counter, st, num_sms);
}

template <typename WT>
static cudaError_t launch_rth_t(const double* r, int64_t n, int d_r, const WT* h, int nx, double* out, int64_t o_rs,
                                int64_t o_cs, double* partials, unsigned* counter, cudaStream_t st, int num_sms) {
  if (!rth_supported(d_r, nx)) return cudaErrorNotSupported;
  if (n <= 0) {
    for (int c = 0; c < d_r; ++c)
      for (int j = 0; j < nx; ++j) {
        cudaError_t e = cudaMemsetAsync(out + c * o_rs + j * o_cs, 0, 8, st);
        if (e != cudaSuccess) return e;
      }
    return cudaSuccess;
  }
  switch ((d_r + 7) / 8) {
    case 1: return launch_rth_mt<1, WT>(r, n, d_r, h, nx, out, o_rs, o_cs, partials, counter, st, num_sms);
    case 2: return launch_rth_mt<2, WT>(r, n, d_r, h, nx, out, o_rs, o_cs, partials, counter, st, num_sms);
    case 3: return launch_rth_mt<3, WT>(r, n, d_r, h, nx, out, o_rs, o_cs, partials, counter, st, num_sms);
    case 4: return launch_rth_mt<4, WT>(r, n, d_r, h, nx, out, o_rs, o_cs, partials, counter, st, num_sms);
    case 5: return launch_rth_mt<5, WT>(r, n, d_r, h, nx, out, o_rs, o_cs, partials, counter, st, num_sms);
    case 6: return launch_rth_mt<6, WT>(r, n, d_r, h, nx, out, o_rs, o_cs, partials, counter, st, num_sms);
    case 7: return launch_rth_mt<7, WT>(r, n, d_r, h, nx, out, o_rs, o_cs, partials, counter, st, num_sms);
    case 8: return launch_rth_mt<8, WT>(r, n, d_r, h, nx, out, o_rs, o_cs, partials, counter, st, num_sms);
    default: return cudaErrorNotSupported;
  }
}

cudaError_t launch_rth(const double* r, int64_t n, int d_r, const int32_t* h, int nx, double* out, int64_t o_rs,
                       int64_t o_cs, double* partials, unsigned* counter, cudaStream_t st, int num_sms) {
  return launch_rth_t(r, n, d_r, h, nx, out, o_rs, o_cs, partials, counter, st, num_sms);
}

cudaError_t launch_rth(const double* r, int64_t n, int d_r, const double* h, int nx, double* out, int64_t o_rs,
                       int64_t o_cs, double* partials, unsigned* counter, cudaStream_t st, int num_sms) {
  return launch_rth_t(r, n, d_r, h, nx, out, o_rs, o_cs, partials, counter, st, num_sms);
}

}  // namespace fb
