// fb_lmm.cu — factorized left multiplication T·X and its row-wise relatives.
//
// Replaces the reference's LMM rewrite (rewrite.py:172-191): for every column block
// out += F·X[slice], with indicator blocks applied as a gather *after* the factor
// product (rewrite.py:187-189, "R·X before K"). On B200 that is two streaming passes:
//   1. z_q = R_q · X[slice_q]          (one pass over each attribute table)
//   2. out_i = S_i · X[0:d_S] + Σ_q z_q[fk_q[i]]   (one pass over S and the FK columns)
// Pass 2 streams S and the FK columns through a shared-memory bulk-copy ring and
// gathers z from L2 (z is n_R × d_X, L2-resident at the BASELINE shapes).
// rowSums (rewrite.py:118-128) is the same pass with X = ones.
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
  int tpr;  // threads cooperating on one row (1, 2, 4, 8)
};

template <int DX>
__global__ void __launch_bounds__(256) lmm_rows_kernel(LmmArgs p, StreamSet ss, int stages,
                                                       int tile_rows) {
  extern __shared__ __align__(128) char smem[];
  const int d = p.d;
  double* xs = reinterpret_cast<double*>(smem);
  const size_t xs_bytes = (static_cast<size_t>(d) * DX * sizeof(double) + 127) & ~size_t(127);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + xs_bytes);
  char* buf = smem + xs_bytes + 128;

  for (int i = threadIdx.x; i < d * DX; i += blockDim.x) xs[i] = p.x[(i / DX) * p.ldx + (i % DX)];

  TileRing ring;
  ring.buf = buf;
  ring.bar = bars;
  ring.stages = stages;
  ring.tile_rows = tile_rows;
  ring.n_rows = p.n;
  ring.policy = policy_evict_first();
  const int64_t ntiles = (p.n + tile_rows - 1) / tile_rows;
  cta_tile_range(ntiles, ring.tile_begin, ring.tile_end);
  ring.start(ss);  // contains __syncthreads (xs visible after it)

  const int tpr = p.tpr;
  const int sub = threadIdx.x % tpr;
  const int rows_per_pass = blockDim.x / tpr;

  for (int64_t k = 0; k < ring.tile_end - ring.tile_begin; ++k) {
    const int stage = ring.acquire(ss, k);
    const int64_t tile = ring.tile_begin + k;
    const int rows = ring.rows_of(tile);
    const int64_t r0 = tile * tile_rows;
    const double* A = reinterpret_cast<const double*>(ring.stage_ptr(stage, ss, 0));

    for (int rb = 0; rb < rows; rb += rows_per_pass) {
      const int r = rb + static_cast<int>(threadIdx.x) / tpr;
      const bool live = r < rows;
      double acc[DX];
#pragma unroll
      for (int j = 0; j < DX; ++j) acc[j] = 0.0;
      if (live) {
        const double* arow = A + static_cast<size_t>(r) * d;
        for (int c = sub; c < d; c += tpr) {
          const double s = arow[c];
          const double* xr = xs + c * DX;
#pragma unroll
          for (int j = 0; j < DX; ++j) acc[j] = fma(s, xr[j], acc[j]);
        }
      }
      if (tpr > 1) {
        for (int o = tpr >> 1; o > 0; o >>= 1) {
#pragma unroll
          for (int j = 0; j < DX; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o, tpr);
        }
      }
      if (live && sub == 0) {
        for (int q = 0; q < p.nfk; ++q) {
          const int32_t* fkt = reinterpret_cast<const int32_t*>(ring.stage_ptr(stage, ss, 1 + q));
          const double* zr = p.z[q] + static_cast<int64_t>(fkt[r]) * DX;
#pragma unroll
          for (int j = 0; j < DX; ++j) acc[j] += __ldg(zr + j);
        }
        double* o = p.out + (r0 + r) * p.ldo;
#pragma unroll
        for (int j = 0; j < DX; ++j) o[j] = acc[j];
      }
    }
    ring.release(ss, k);
  }
}

// ------------------------------------------------------------------ host launcher
static int pick_tpr(int d) {
  if (d <= 32) return 1;
  if (d <= 64) return 2;
  if (d <= 128) return 4;
  return 8;
}

template <int DX>
static cudaError_t launch_lmm_dx(const LmmArgs& a, cudaStream_t st, int num_sms) {
  LmmArgs p = a;
  p.tpr = pick_tpr(p.d);
  const int threads = 256;
  const int tile_rows = threads / p.tpr;  // multiple of 4
  StreamSet ss{};
  ss.count = 1 + p.nfk;
  ss.base[0] = reinterpret_cast<const char*>(p.a);
  ss.row_bytes[0] = static_cast<uint32_t>(p.d) * 8u;
  for (int q = 0; q < p.nfk; ++q) {
    ss.base[1 + q] = reinterpret_cast<const char*>(p.fk[q]);
    ss.row_bytes[1 + q] = 4u;
  }
  stream_layout(ss, tile_rows);
  const size_t xs_bytes = (static_cast<size_t>(p.d) * DX * 8 + 127) & ~size_t(127);
  const size_t budget = 200 * 1024;
  int stages = static_cast<int>((budget - xs_bytes - 128) / ss.stage_bytes);
  if (stages > 4) stages = 4;
  if (stages < 2) stages = 2;
  const size_t smem = xs_bytes + 128 + static_cast<size_t>(stages) * ss.stage_bytes;
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  auto kern = lmm_rows_kernel<DX>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int per_sm = static_cast<int>((227 * 1024) / (smem + 1024));
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 4) per_sm = 4;
  const int64_t ntiles = (p.n + tile_rows - 1) / tile_rows;
  const int grid = grid_for(ntiles, 1, per_sm, num_sms);
  kern<<<grid, threads, smem, st>>>(p, ss, stages, tile_rows);
  FB_LAUNCHED();
  return cudaGetLastError();
}

cudaError_t launch_lmm_rows(const double* a, int64_t n, int d, const double* x, int dx, int64_t ldx,
                            int nfk,
                            const int32_t* const* fk, const double* const* z, double* out,
                            int64_t ldo, cudaStream_t st, int num_sms) {
  if (n <= 0) return cudaSuccess;
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
  switch (dx) {
#define FB_DX_CASE(N) \
  case N:             \
    return launch_lmm_dx<N>(p, st, num_sms);
    FB_DX_CASE(1)
    FB_DX_CASE(2)
    FB_DX_CASE(3)
    FB_DX_CASE(4)
    FB_DX_CASE(5)
    FB_DX_CASE(6)
    FB_DX_CASE(7)
    FB_DX_CASE(8)
    FB_DX_CASE(10)
    FB_DX_CASE(12)
    FB_DX_CASE(16)
#undef FB_DX_CASE
    default:
      return cudaErrorNotSupported;  // caller splits X into supported column chunks
  }
}

}  // namespace fb
