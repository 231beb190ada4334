// fb_lmm.cu — factorized left multiplication T·X and its row-wise relatives.
//
// Replaces the reference's LMM rewrite (rewrite.py:172-191): for every column block
// out += F·X[slice], with indicator blocks applied as a gather *after* the factor
// product (rewrite.py:187-189, "R·X before K"). On B200 that is two streaming passes:
//   1. z_q = R_q · X[slice_q]          (one pass over each attribute table)
//   2. out_i = S_i · X[0:d_S] + Σ_q z_q[fk_q[i]]   (one pass over S and the FK columns)
// rowSums (rewrite.py:118-128) is the same pass with X = ones.
//
// Both passes are the same kernel: factor rows stream through a shared-memory
// bulk-copy ring (fb_stream.cuh) and the per-tile product runs on the FP64 tensor
// cores (mma.sync m8n8k4 f64 -> DMMA; tcgen05 has no f64 kind). Each warp owns MT
// m-tiles of 8 rows; X (d × d_x, zero-padded to NT·8 columns) is the B operand read
// from a bank-skewed shared copy. The gathered z values are loaded before the k-loop
// so their L2 latency overlaps the tensor-core work, then added in the reference's
// order (S·X first, then each part in turn).
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
};

template <int NT>
FB_DEV int xs_ld() {
  return 8 * NT + 4;  // bank skew for the B-fragment loads (see conflict_free_pitch)
}

template <int NT, int MT>
__global__ void __launch_bounds__(kRingThreads) lmm_dmma_kernel(LmmArgs p, StreamSet ss, int stages,
                                                       int tile_rows) {
  extern __shared__ __align__(128) char smem[];
  const int d = p.d;
  const int dpad = (d + 3) & ~3;
  const int ldxs = xs_ld<NT>();
  double* xs = reinterpret_cast<double*>(smem);
  const size_t xs_bytes = (static_cast<size_t>(dpad > 0 ? dpad : 4) * ldxs * sizeof(double) + 127) & ~size_t(127);
  char* buf = smem + xs_bytes;

  for (int i = threadIdx.x; i < dpad * ldxs; i += blockDim.x) {
    const int k = i / ldxs, n = i % ldxs;
    xs[i] = (k < d && n < p.dx) ? p.x[k * p.ldx + n] : 0.0;
  }

  TileRing ring;
  ring.init(buf, stages, tile_rows, p.n);
  ring.start();  // contains __syncthreads (xs visible after it)
  if (is_producer_warp()) {
    ring.produce(ss);
    return;
  }

  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  const int warp = (threadIdx.x >> 5) - 1;  // consumer warp index
  const int pitch = p.pitch;

  for (int64_t kt = 0; kt < ring.count(); ++kt) {
    const int stage = ring.acquire(ss, kt);
    const int64_t tile = ring.tile_begin + kt;
    const int rows = ring.rows_of(tile);
    const int64_t r0 = tile * tile_rows;
    const double* A = reinterpret_cast<const double*>(ring.stage_ptr(stage, ss, 0));
    const int wrow = warp * (8 * MT);

    if (wrow < rows) {
      // prefetch the first part's gathered z values (they are added after the product)
      double zpre[MT][NT][2];
      if (p.nfk > 0) {
        const int32_t* fkt = reinterpret_cast<const int32_t*>(ring.stage_ptr(stage, ss, 1));
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int r = wrow + 8 * mt + g;
          const bool live = r < rows;
          const double* zr = p.z[0] + static_cast<int64_t>(live ? fkt[r] : 0) * p.dx;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const int c = 8 * nt + 2 * t;
            zpre[mt][nt][0] = (live && c < p.dx) ? __ldg(zr + c) : 0.0;
            zpre[mt][nt][1] = (live && c + 1 < p.dx) ? __ldg(zr + c + 1) : 0.0;
          }
        }
      }

      double acc[MT][NT][2];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;

      const double* arow[MT];
      bool rlive[MT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int r = wrow + 8 * mt + g;
        rlive[mt] = r < rows;
        arow[mt] = A + static_cast<size_t>(rlive[mt] ? r : 0) * pitch;
      }
      for (int k0 = 0; k0 < dpad; k0 += 4) {
        const int k = k0 + t;
        double b[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) b[nt] = xs[k * ldxs + 8 * nt + g];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const double a = (rlive[mt] && k < d) ? arow[mt][k] : 0.0;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], a, b[nt]);
        }
      }

      // epilogue: + z_0 (prefetched) + z_1 ... in part order, then store
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int r = wrow + 8 * mt + g;
        if (r >= rows) continue;
        if (p.nfk > 0) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            acc[mt][nt][0] += zpre[mt][nt][0];
            acc[mt][nt][1] += zpre[mt][nt][1];
          }
          for (int q = 1; q < p.nfk; ++q) {
            const int32_t* fkt = reinterpret_cast<const int32_t*>(ring.stage_ptr(stage, ss, 1 + q));
            const double* zr = p.z[q] + static_cast<int64_t>(fkt[r]) * p.dx;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const int c = 8 * nt + 2 * t;
              if (c < p.dx) acc[mt][nt][0] += __ldg(zr + c);
              if (c + 1 < p.dx) acc[mt][nt][1] += __ldg(zr + c + 1);
            }
          }
        }
        double* o = p.out + (r0 + r) * p.ldo;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int c = 8 * nt + 2 * t;
          if (c + 1 < p.dx && ((reinterpret_cast<uintptr_t>(o + c) & 15u) == 0)) {
            *reinterpret_cast<double2*>(o + c) = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
          } else {
            if (c < p.dx) o[c] = acc[mt][nt][0];
            if (c + 1 < p.dx) o[c + 1] = acc[mt][nt][1];
          }
        }
      }
    }
    ring.release();
  }
}

// ------------------------------------------------------------------ host launcher
template <int NT, int MT>
static cudaError_t launch_lmm_cfg(const LmmArgs& a, cudaStream_t st, int num_sms) {
  LmmArgs p = a;
  const int tile_rows = kConsumerWarps * 8 * MT;
  StreamSet ss{};
  ss.count = 1 + p.nfk;
  ss.base[0] = reinterpret_cast<const char*>(p.a);
  ss.row_bytes[0] = static_cast<uint32_t>(p.d) * 8u;
  p.pitch = (p.d % 2 == 0) ? conflict_free_pitch(p.d) : p.d;
  ss.pitch[0] = static_cast<uint32_t>(p.pitch) * 8u;
  for (int q = 0; q < p.nfk; ++q) {
    ss.base[1 + q] = reinterpret_cast<const char*>(p.fk[q]);
    ss.row_bytes[1 + q] = 4u;
  }
  stream_layout(ss, tile_rows, p.n);
  const int dpad = (p.d + 3) & ~3;
  const size_t xs_bytes = (static_cast<size_t>(dpad > 0 ? dpad : 4) * (8 * NT + 4) * 8 + 127) & ~size_t(127);
  const size_t budget = 200 * 1024;
  int stages = static_cast<int>((budget - xs_bytes - 256) / ss.stage_bytes);
  if (stages > 4) stages = 4;
  if (stages < 2) return cudaErrorNotSupported;
  const size_t smem = xs_bytes + 256 + static_cast<size_t>(stages) * ss.stage_bytes;
  auto kern = lmm_dmma_kernel<NT, MT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
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

template <int NT>
static cudaError_t launch_lmm_nt(const LmmArgs& p, cudaStream_t st, int num_sms) {
  // rows per warp: 32 when a 256-row tile of this width fits 4 stages comfortably
  const int pitch = (p.d % 2 == 0) ? conflict_free_pitch(p.d) : p.d;
  const size_t row_bytes = static_cast<size_t>(pitch) * 8 + 4 * p.nfk;
  if (row_bytes * 256 <= 48 * 1024) return launch_lmm_cfg<NT, 4>(p, st, num_sms);
  if (row_bytes * 128 <= 48 * 1024) return launch_lmm_cfg<NT, 2>(p, st, num_sms);
  return launch_lmm_cfg<NT, 1>(p, st, num_sms);
}

cudaError_t launch_lmm_rows(const double* a, int64_t n, int d, const double* x, int dx, int64_t ldx,
                            int nfk, const int32_t* const* fk, const double* const* z, double* out,
                            int64_t ldo, cudaStream_t st, int num_sms) {
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
  }
  p.out = out;
  p.ldo = ldo;
  if (dx <= 8) return launch_lmm_nt<1>(p, st, num_sms);
  return launch_lmm_nt<2>(p, st, num_sms);
}

}  // namespace fb
