// fb_lmm_band.cu — the wide-X LMM S pass over an FK-band layout (fb_band_layout).
//
// c2 X100x16 in storage order (fb_lmm.cu): z = R·X (n_R × 16 doubles = 128 MB) does not stay in
// the 126 MB L2 beside the S stream, two of three z gathers miss and the op moves 8.2 GB for
// 6.5 GB algorithmic (profiles/r01_ncu_full_v5.txt, r02_lmm16_experiments.txt). This pass reads a
// cached copy of S and FK whose rows are grouped into FK bands (band b = keys
// [b·n_R/B, (b+1)·n_R/B), storage order kept inside a band) with the tiles dealt round-robin
// (TileRingT<true>), so at any moment all CTAs gather from one ~16 MB slice of z, which stays
// L2-resident: every z row is read from DRAM once (ncu: 6.1 GB per S pass instead of 7.6). The band
// permutation rides along as a second ring stream and each finished row is stored to its own
// output row. For d_x = 16 the two 8-column DMMA tiles take interleaved column pairs (tile nt
// owns columns 4j + 2nt, 4j + 2nt + 1), so lane (g, t) ends with columns 4t..4t+3 of row g and
// one 256-bit store per lane writes a whole 128-byte row per four lanes. Each output element is
// the same chain of DMMA sums as in lmm_dmma_zinit_kernel (z first, then the k-steps in order):
// results are bitwise equal to the storage-order pass.
#include "fb_kernels.cuh"

namespace fb {

struct BandArgs {
  const double* x;  // d × dx, leading dimension ldx
  int d, dx;
  int64_t ldx;
  int64_t n;
  double* out;  // n × dx, leading dimension ldo (even, base 32-byte aligned)
  int64_t ldo;
  int zstride;  // doubles per gathered z row
  int debug;    // FB_LMM_DEBUG (measurement only): 8 = store rows in band order (wrong rows)
};

FB_DEV void st_hint4(double* p, double a, double b, double c, double d, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;\n" ::"l"(p), "d"(a), "d"(b), "d"(c),
               "d"(d), "l"(policy)
               : "memory");
}

// output column of local column j of DMMA tile nt
template <int NT>
FB_DEV constexpr int band_col(int nt, int j) {
  return NT == 2 ? 4 * (j >> 1) + 2 * nt + (j & 1) : j;
}

template <int NT, int MT, int KS>
__global__ void __launch_bounds__(kRingThreads, 1) lmm_dmma_band_kernel(BandArgs p, StreamSet ss, int stages,
                                                                    int tile_rows) {
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

  TileRingT<true> ring;
  ring.init(buf, stages, tile_rows, p.n);
  ring.start(ss);  // contains __syncthreads (xs visible after it)
  if (ring.service<false, true>(ss)) return;

  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  const int warp = consumer_warp();
  const int pitch = d;
  const int wrow = warp * (8 * MT);
  const uint64_t pol = policy_evict_first();
  const bool ragged_k = (d & 3) != 0;
  const int zst = p.zstride;
  double bf[KS][NT];  // B fragments: X[4s + t][column of (nt, g)], zero past d
#pragma unroll
  for (int s = 0; s < KS; ++s)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) bf[s][nt] = xs[(4 * s + t) * ldxs + band_col<NT>(nt, g)];
  const int a_off = (wrow + g) * pitch + t;
  const int z_off = (wrow + g) * zst + 2 * NT * t;  // this lane's 2·NT consecutive columns
  const int64_t nt_local = ring.count();

  for (int64_t kt = 0; kt < nt_local; ++kt) {
    const int cur = ring.acquire(ss, kt);
    const int64_t tile = ring.tile_of(kt);
    const int rows = ring.rows_of(tile);
    const double* A = reinterpret_cast<const double*>(ring.stage_ptr(cur, ss, 0)) + a_off;
    const int32_t* pm = reinterpret_cast<const int32_t*>(ring.stage_ptr(cur, ss, 1)) + wrow + g;
    __syncwarp();  // mma.sync.aligned needs the whole warp converged (after the barrier spin)
    if (wrow < rows) {
      double acc[MT][NT][2];
      int32_t orow[MT];
      const double* z0 = reinterpret_cast<const double*>(ring.gather_ptr(cur, ss, 0)) + z_off;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        orow[mt] = pm[8 * mt];
        if (p.debug & 8) orow[mt] = static_cast<int32_t>(tile * tile_rows + wrow + 8 * mt + g);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double2 zv = *reinterpret_cast<const double2*>(z0 + 8 * mt * zst + 2 * nt);
          acc[mt][nt][0] = zv.x;
          acc[mt][nt][1] = zv.y;
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
      double* o = p.out + 2 * NT * t;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        if (rows != tile_rows && wrow + 8 * mt + g >= rows) continue;
        double* orp = o + static_cast<int64_t>(orow[mt]) * p.ldo;
        if constexpr (NT == 2)
          st_hint4(orp, acc[mt][0][0], acc[mt][0][1], acc[mt][1][0], acc[mt][1][1], pol);
        else
          st_hint2(orp, acc[mt][0][0], acc[mt][0][1], pol);
      }
    }
    ring.release();
  }
}

template <int NT, int KS>
static cudaError_t launch_band_ks(const BandArgs& p, StreamSet& ss, cudaStream_t st, int num_sms) {
  constexpr int MT = 4;
  const int tile_rows = kConsumerWarps * 8 * MT;
  stream_layout(ss, tile_rows, p.n);
  const size_t fixed = (static_cast<size_t>(4 * KS) * (8 * NT + 4) * 8 + 127) & ~size_t(127);
  const size_t budget = 224 * 1024;
  if (fixed + kRingHeader + 2 * static_cast<size_t>(ss.stage_bytes) > budget) return cudaErrorNotSupported;
  int stages = static_cast<int>((budget - fixed - kRingHeader) / ss.stage_bytes);
  if (stages > 8) stages = 8;
  const size_t smem = fixed + kRingHeader + static_cast<size_t>(stages) * ss.stage_bytes;
  auto kern = lmm_dmma_band_kernel<NT, MT, KS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int64_t ntiles = (p.n + tile_rows - 1) / tile_rows;
  kern<<<grid_for(ntiles, 1, 1, num_sms), kRingThreads, smem, st>>>(p, ss, stages, tile_rows);
  FB_LAUNCHED();
  return cudaGetLastError();
}

template <int NT>
static cudaError_t launch_band_nt(const BandArgs& p, StreamSet& ss, cudaStream_t st, int num_sms) {
  switch ((p.d + 3) / 4) {
    case 1: return launch_band_ks<NT, 1>(p, ss, st, num_sms);
    case 2: return launch_band_ks<NT, 2>(p, ss, st, num_sms);
    case 3: return launch_band_ks<NT, 3>(p, ss, st, num_sms);
    case 4: return launch_band_ks<NT, 4>(p, ss, st, num_sms);
    case 5: return launch_band_ks<NT, 5>(p, ss, st, num_sms);
    case 6: return launch_band_ks<NT, 6>(p, ss, st, num_sms);
    case 7: return launch_band_ks<NT, 7>(p, ss, st, num_sms);
    case 8: return launch_band_ks<NT, 8>(p, ss, st, num_sms);
    default: return cudaErrorNotSupported;
  }
}

bool lmm_band_supported(int d, int dx, int64_t ldo, const double* out) {
  const uintptr_t al = dx == 16 ? 31u : 15u;
  const int64_t lm = dx == 16 ? 3 : 1;
  return d >= 1 && d <= 32 && (dx == 8 || dx == 16) && (ldo & lm) == 0 && (reinterpret_cast<uintptr_t>(out) & al) == 0;
}

cudaError_t launch_lmm_band(const double* a_band, const int32_t* fk_band, const int32_t* perm, int64_t n, int d,
                            const double* x, int dx, int64_t ldx, const double* z, int zstride, int64_t z_rows,
                            double* out, int64_t ldo, cudaStream_t st, int num_sms) {
  (void)z_rows;
  if (n <= 0) return cudaSuccess;
  if (!lmm_band_supported(d, dx, ldo, out) || zstride < dx || (zstride & 1)) return cudaErrorNotSupported;
  BandArgs p{};
  p.x = x;
  p.d = d;
  p.dx = dx;
  p.ldx = ldx;
  p.n = n;
  p.out = out;
  p.ldo = ldo;
  p.zstride = zstride;
  static int dbg = [] { const char* e = getenv("FB_LMM_DEBUG"); return e ? atoi(e) : 0; }();
  p.debug = dbg & 8;
  StreamSet ss{};
  ss.count = 2;  // S rows in band order + the band permutation (row-aligned int32)
  ss.base[0] = reinterpret_cast<const char*>(a_band);
  ss.row_bytes[0] = ss.pitch[0] = static_cast<uint32_t>(d) * 8u;
  ss.base[1] = reinterpret_cast<const char*>(perm);
  ss.row_bytes[1] = ss.pitch[1] = 4u;
  ss.ngather = 1;  // z[fk] rows, keys in band order
  ss.gkeys[0] = fk_band;
  ss.gbase[0] = reinterpret_cast<const char*>(z);
  ss.grow_bytes[0] = static_cast<uint32_t>(zstride) * 8u;
  return dx == 8 ? launch_band_nt<1>(p, ss, st, num_sms) : launch_band_nt<2>(p, ss, st, num_sms);
}

}  // namespace fb
