// fb_build.cu — normalized-matrix construction on the device.
//
// Replaces build_pkfk / build_star's key handling (normmat.py:182-214, 217-237):
//   * _check_keys: 1-based keys must lie in [1, n_R]; the first offending entity row
//     is reported (normmat.py:191-197)            -> key_check_hist (atomicMin on row)
//   * _remap_part: np.unique of the used keys, dropping unreferenced R rows and
//     compacting to 0-based targets (normmat.py:168-179)
//                                                  -> histogram, flag scan, remap
//   * IndicatorMatrix.counts = bincount (indicator.py:61-66) -> integer histogram
//   * R[used] row gather                           -> gather_rows
// All integer work is exact, so targets, source rows and counts are bit-identical to
// the reference's.
#include "fb_kernels.cuh"

namespace fb {

__global__ void key_check_hist_kernel(const int64_t* __restrict__ key, int64_t n, int64_t n_r,
                                      int32_t* __restrict__ counts,
                                      unsigned long long* __restrict__ first_bad) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const int64_t k = key[i];
    if (k < 1 || k > n_r) {
      atomicMin(first_bad, static_cast<unsigned long long>(i));
    } else {
      red_add(counts + (k - 1), 1);
    }
  }
}

__global__ void fk_hist_kernel(const int32_t* __restrict__ fk, int64_t n, int32_t* __restrict__ counts) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    red_add(counts + fk[i], 1);
}

// ---- exclusive scan of used flags (counts > 0) in three phases
constexpr int kScanBlock = 1024;

__global__ void scan_block_sums_kernel(const int32_t* __restrict__ counts, int64_t n_r,
                                       int32_t* __restrict__ block_sums) {
  __shared__ int32_t warp_tot[32];
  const int64_t i = blockIdx.x * static_cast<int64_t>(kScanBlock) + threadIdx.x;
  int32_t f = (i < n_r && counts[i] > 0) ? 1 : 0;
  f = __reduce_add_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0) warp_tot[threadIdx.x >> 5] = f;
  __syncthreads();
  if (threadIdx.x < 32) {
    int32_t v = warp_tot[threadIdx.x];
    v = __reduce_add_sync(0xffffffffu, v);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = v;
  }
}

// single CTA: exclusive scan of block sums in place; total -> *n_used
__global__ void scan_block_prefix_kernel(int32_t* block_sums, int64_t nblocks, int32_t* n_used) {
  __shared__ int32_t carry;
  __shared__ int32_t warp_tot[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nblocks; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    int32_t v = i < nblocks ? block_sums[i] : 0;
    // inclusive warp scan
    int32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      int32_t t = __shfl_up_sync(0xffffffffu, x, o);
      if ((threadIdx.x & 31) >= o) x += t;
    }
    if ((threadIdx.x & 31) == 31) warp_tot[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      int32_t w = warp_tot[threadIdx.x];
      int32_t y = w;
      for (int o = 1; o < 32; o <<= 1) {
        int32_t t = __shfl_up_sync(0xffffffffu, y, o);
        if (threadIdx.x >= o) y += t;
      }
      warp_tot[threadIdx.x] = y - w;  // exclusive warp offsets
    }
    __syncthreads();
    const int32_t excl = carry + warp_tot[threadIdx.x >> 5] + x - v;
    if (i < nblocks) block_sums[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_used = carry;
}

__global__ void scan_write_kernel(const int32_t* __restrict__ counts, int64_t n_r,
                                  const int32_t* __restrict__ block_off, int32_t* __restrict__ lookup) {
  __shared__ int32_t warp_tot[32];
  const int64_t i = blockIdx.x * static_cast<int64_t>(kScanBlock) + threadIdx.x;
  const int32_t f = (i < n_r && counts[i] > 0) ? 1 : 0;
  const unsigned bal = __ballot_sync(0xffffffffu, f);
  const int lane = threadIdx.x & 31;
  const int32_t in_warp = __popc(bal & ((1u << lane) - 1u));
  if (lane == 0) warp_tot[threadIdx.x >> 5] = __popc(bal);
  __syncthreads();
  if (threadIdx.x < 32) {
    int32_t w = warp_tot[threadIdx.x];
    int32_t y = w;
    for (int o = 1; o < 32; o <<= 1) {
      int32_t t = __shfl_up_sync(0xffffffffu, y, o);
      if (threadIdx.x >= o) y += t;
    }
    warp_tot[threadIdx.x] = y - w;
  }
  __syncthreads();
  if (i < n_r) lookup[i] = f ? block_off[blockIdx.x] + warp_tot[threadIdx.x >> 5] + in_warp : -1;
}

__global__ void remap_kernel(const int64_t* __restrict__ key, int64_t n,
                             const int32_t* __restrict__ lookup, int32_t* __restrict__ target) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    target[i] = lookup[key[i] - 1];
}

__global__ void used_kernel(const int32_t* __restrict__ lookup, const int32_t* __restrict__ counts,
                            int64_t n_r, int64_t* __restrict__ used_idx,
                            int32_t* __restrict__ counts_kept) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < n_r; j += stride) {
    const int32_t l = lookup[j];
    if (l >= 0) {
      used_idx[l] = j;
      counts_kept[l] = counts[j];
    }
  }
}

// out[r, :] = in[idx[r], :]; one warp per row, 16-byte vectors when aligned.
__global__ void gather_rows_kernel(const double* __restrict__ in, int64_t ld_in,
                                   const int64_t* __restrict__ idx64,
                                   const int32_t* __restrict__ idx32, int64_t nrows, int d,
                                   double* __restrict__ out, int64_t ld_out) {
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; r < nrows;
       r += warps) {
    const int64_t src = idx64 ? idx64[r] : static_cast<int64_t>(idx32[r]);
    const double* a = in + src * ld_in;
    double* o = out + r * ld_out;
    for (int c = lane; c < d; c += 32) o[c] = a[c];
  }
}

__global__ void i32_to_f64_kernel(const int32_t* __restrict__ in, double* __restrict__ out, int64_t n) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    out[i] = static_cast<double>(in[i]);
}

// ------------------------------------------------------------------ launchers
static int eltwise_grid(int64_t n, int num_sms) { return grid_for(n, 256 * 4, 8, num_sms); }

cudaError_t launch_key_check_hist(const int64_t* key, int64_t n, int64_t n_r, int32_t* counts,
                                  unsigned long long* first_bad, cudaStream_t st, int num_sms) {
  cudaError_t e = cudaMemsetAsync(counts, 0, static_cast<size_t>(n_r) * sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(first_bad, 0xff, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  if (n > 0) {
    key_check_hist_kernel<<<eltwise_grid(n, num_sms), 256, 0, st>>>(key, n, n_r, counts, first_bad);
    FB_LAUNCHED();
  }
  return cudaGetLastError();
}

size_t used_scan_ws_ints(int64_t n_r) { return static_cast<size_t>((n_r + kScanBlock - 1) / kScanBlock) + 1; }

cudaError_t launch_used_scan(const int32_t* counts, int64_t n_r, int32_t* lookup, int32_t* n_used,
                             int32_t* block_ws, cudaStream_t st, int num_sms) {
  (void)num_sms;
  const int64_t nb = (n_r + kScanBlock - 1) / kScanBlock;
  if (nb == 0) return cudaMemsetAsync(n_used, 0, sizeof(int32_t), st);
  scan_block_sums_kernel<<<static_cast<unsigned>(nb), kScanBlock, 0, st>>>(counts, n_r, block_ws);
  FB_LAUNCHED();
  scan_block_prefix_kernel<<<1, 1024, 0, st>>>(block_ws, nb, n_used);
  FB_LAUNCHED();
  scan_write_kernel<<<static_cast<unsigned>(nb), kScanBlock, 0, st>>>(counts, n_r, block_ws, lookup);
  FB_LAUNCHED();
  return cudaGetLastError();
}

cudaError_t launch_remap(const int64_t* key, int64_t n, const int32_t* lookup, const int32_t* counts,
                         int64_t n_r, int32_t* target, int64_t* used_idx, int32_t* counts_kept,
                         cudaStream_t st, int num_sms) {
  if (n > 0) {
    remap_kernel<<<eltwise_grid(n, num_sms), 256, 0, st>>>(key, n, lookup, target);
    FB_LAUNCHED();
  }
  if (n_r > 0) {
    used_kernel<<<eltwise_grid(n_r, num_sms), 256, 0, st>>>(lookup, counts, n_r, used_idx, counts_kept);
    FB_LAUNCHED();
  }
  return cudaGetLastError();
}

cudaError_t launch_fk_hist(const int32_t* fk, int64_t n, int32_t* counts, int64_t nbins,
                           cudaStream_t st, int num_sms) {
  cudaError_t e = cudaMemsetAsync(counts, 0, static_cast<size_t>(nbins) * sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  if (n > 0) {
    fk_hist_kernel<<<eltwise_grid(n, num_sms), 256, 0, st>>>(fk, n, counts);
    FB_LAUNCHED();
  }
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const double* in, int64_t ld_in, const int64_t* idx64,
                               const int32_t* idx32, int64_t nrows, int d, double* out,
                               int64_t ld_out, cudaStream_t st, int num_sms) {
  if (nrows <= 0 || d <= 0) return cudaSuccess;
  const int grid = grid_for(nrows, 8, 8, num_sms);
  gather_rows_kernel<<<grid, 256, 0, st>>>(in, ld_in, idx64, idx32, nrows, d, out, ld_out);
  FB_LAUNCHED();
  return cudaGetLastError();
}

cudaError_t launch_i32_to_f64(const int32_t* in, double* out, int64_t n, cudaStream_t st, int num_sms) {
  if (n > 0) {
    i32_to_f64_kernel<<<eltwise_grid(n, num_sms), 256, 0, st>>>(in, out, n);
    FB_LAUNCHED();
  }
  return cudaGetLastError();
}

// CSR -> dense rows (a sparse factor matrix of the reference, kernel.py:110-121, expanded into
// the row-major HBM layout every operator reads). Canonical CSR: no duplicate (row, col) entries,
// so each output cell has at most one writer. A warp per row; the zero fill is a memset.
__global__ void csr_expand_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                                  const double* __restrict__ data, int64_t nrows, double* __restrict__ out,
                                  int64_t ld_out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < nrows; r += warps) {
    const int64_t b = indptr[r], e = indptr[r + 1];
    double* row = out + r * ld_out;
    for (int64_t k = b + lane; k < e; k += 32) row[indices[k]] = data[k];
  }
}

cudaError_t launch_csr_expand(const int64_t* indptr, const int32_t* indices, const double* data,
                              int64_t nrows, int32_t ncols, double* out, int64_t ld_out,
                              cudaStream_t st, int num_sms) {
  if (nrows <= 0 || ncols <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(out, 0, static_cast<size_t>(nrows) * ld_out * sizeof(double), st);
  if (e != cudaSuccess) return e;
  csr_expand_kernel<<<grid_for(nrows, 8, 8, num_sms), 256, 0, st>>>(indptr, indices, data, nrows, out, ld_out);
  FB_LAUNCHED();
  return cudaGetLastError();
}

}  // namespace fb

