// fb_dense.cu — the small dense and sparse pieces of the rest of the operator surface.
//
// The reference's row Gram, double multiplication and pair product (rewrite.py:301-446,
// indicator.py:144-162) reduce to a handful of primitives that sit beside
// the factorized hot path (their inputs are the factor tables, their outputs n × n or n × m
// dense or an n_a × n_b sparse count matrix):
//   * dense_mm_kernel: C (+)= op(A)·op(B) on the FP64 tensor cores (mma.sync m8n8k4, SASS
//     DMMA), each warp a 32 × 32 block of C, fragments read straight from global/L2 (the
//     operands are factor tables of at most a few hundred columns);
//   * gather2_add_kernel: C[i, j] += M[ta[i], tb[j]] — the two-sided indicator expansion
//     E_a M E_bᵀ of a block product (rewrite.py:308-313, 436-444);
//   * scatter_rows_kernel: out[t[i], :] += a[i, :] — Eᵀa (indicator.py:107-118) with REDG;
//   * pair_counts: E_aᵀE_b as sorted (row·n_b + col) keys with counts — a CUB radix sort of the
//     combined keys plus a run-length encode (indicator.py:144-162's coo → csr);
//   * csr_spmm_kernel: Y = P·X for a CSR P (warp per row, lanes over X's columns) — the
//     sparse-dense products of pair_product counts and of CSR factor matrices.
#include <cub/cub.cuh>

#include "fb_kernels.cuh"

namespace fb {

// ------------------------------------------------------------------ dense GEMM (DMMA)
// C[m × n] = op(A)·op(B) (+ C when accumulate), row-major with leading dimensions;
// op(A)[i][k] = ta ? A[k·lda + i] : A[i·lda + k], op(B)[k][j] = tb ? B[j·ldb + k] : B[k·ldb + j].
__global__ void dense_mm_kernel(int64_t m, int64_t n, int64_t k, const double* __restrict__ a, int64_t lda, int ta,
                                const double* __restrict__ b, int64_t ldb, int tbf, double* __restrict__ c,
                                int64_t ldc, int accumulate) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t tiles_n = (n + 31) / 32;
  const int64_t i0 = (wid / tiles_n) * 32, j0 = (wid % tiles_n) * 32;
  if (i0 >= m) return;
  double acc[4][4][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  for (int64_t k0 = 0; k0 < k; k0 += 4) {
    const int64_t kk = k0 + t;
    double af[4], bf[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int64_t i = i0 + 8 * x + g;
      af[x] = (i < m && kk < k) ? (ta ? __ldg(a + kk * lda + i) : __ldg(a + i * lda + kk)) : 0.0;
      const int64_t j = j0 + 8 * x + g;
      bf[x] = (j < n && kk < k) ? (tbf ? __ldg(b + j * ldb + kk) : __ldg(b + kk * ldb + j)) : 0.0;
    }
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) dmma_8x8x4(acc[x][y][0], acc[x][y][1], af[x], bf[y]);
  }
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int64_t i = i0 + 8 * x + g;
    if (i >= m) continue;
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t j = j0 + 8 * y + 2 * t + e;
        if (j >= n) continue;
        double* o = c + i * ldc + j;
        *o = accumulate ? *o + acc[x][y][e] : acc[x][y][e];
      }
  }
}

cudaError_t launch_dense_mm(int64_t m, int64_t n, int64_t k, const double* a, int64_t lda, int ta, const double* b,
                            int64_t ldb, int tb, double* c, int64_t ldc, int accumulate, cudaStream_t st) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  if (k <= 0) {
    if (accumulate) return cudaSuccess;
    return cudaMemset2DAsync(c, static_cast<size_t>(ldc) * 8, 0, static_cast<size_t>(n) * 8, static_cast<size_t>(m), st);
  }
  const int64_t warps = ((m + 31) / 32) * ((n + 31) / 32);
  const int64_t blocks = (warps + 7) / 8;
  dense_mm_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(m, n, k, a, lda, ta, b, ldb, tb, c, ldc, accumulate);
  FB_LAUNCHED();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ two-sided gather
// c[i·ldc + j] += mat[ra[i]·ldm + cb[j]] (ra / cb int32 row / column maps; cb == nullptr: identity)
__global__ void gather2_add_kernel(int64_t m, int64_t n, const double* __restrict__ mat, int64_t ldm,
                                   const int32_t* __restrict__ ra, const int32_t* __restrict__ cb, double* c,
                                   int64_t ldc) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    const int64_t src_c = cb ? cb[j] : j;
    c[i * ldc + j] += __ldg(mat + static_cast<int64_t>(ra[i]) * ldm + src_c);
  }
}

cudaError_t launch_gather2_add(int64_t m, int64_t n, const double* mat, int64_t ldm, const int32_t* ra,
                               const int32_t* cb, double* c, int64_t ldc, cudaStream_t st, int num_sms) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  const int grid = grid_for(m * n, 256, 8, num_sms);
  gather2_add_kernel<<<grid, 256, 0, st>>>(m, n, mat, ldm, ra, cb, c, ldc);
  FB_LAUNCHED();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ Eᵀa scatter
// out[t[i]·d + j] += a[i·lda + j] (out zeroed by the caller); REDG f64, order-free sums
__global__ void scatter_rows_kernel(int64_t n, int d, const int32_t* __restrict__ tgt, const double* __restrict__ a,
                                    int64_t lda, double* out) {
  const int64_t total = n * d;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / d;
    const int j = static_cast<int>(e % d);
    red_add(out + static_cast<int64_t>(tgt[i]) * d + j, __ldg(a + i * lda + j));
  }
}

cudaError_t launch_scatter_rows(int64_t n, int d, const int32_t* tgt, const double* a, int64_t lda, double* out,
                                int64_t out_rows, cudaStream_t st, int num_sms) {
  cudaError_t e = cudaMemsetAsync(out, 0, static_cast<size_t>(out_rows) * d * 8, st);
  if (e != cudaSuccess || n <= 0 || d <= 0) return e;
  const int grid = grid_for(n * d, 256, 8, num_sms);
  scatter_rows_kernel<<<grid, 256, 0, st>>>(n, d, tgt, a, lda, out);
  FB_LAUNCHED();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ pair counts
__global__ void pair_keys_kernel(int64_t n, const int32_t* __restrict__ ta, const int32_t* __restrict__ tb,
                                 int64_t cols_b, int64_t* __restrict__ key) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    key[i] = static_cast<int64_t>(ta[i]) * cols_b + tb[i];
}

// indptr[r] = number of unique keys with key / cols_b < r (a binary search per row boundary)
__global__ void pair_indptr_kernel(const int64_t* __restrict__ ukeys, const int64_t* __restrict__ nnz_p,
                                   int64_t rows_a, int64_t cols_b, int64_t* __restrict__ indptr) {
  const int64_t nnz = *nnz_p;
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r <= rows_a;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t bound = r * cols_b;
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ukeys[mid] < bound)
        lo = mid + 1;
      else
        hi = mid;
    }
    indptr[r] = lo;
  }
}

__global__ void pair_split_kernel(const int64_t* __restrict__ ukeys, const int32_t* __restrict__ cnt,
                                  const int64_t* __restrict__ nnz_p, int64_t cols_b, int64_t* __restrict__ col,
                                  double* __restrict__ val) {
  const int64_t nnz = *nnz_p;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    col[i] = ukeys[i] % cols_b;
    val[i] = static_cast<double>(cnt[i]);
  }
}

size_t pair_counts_workspace_bytes(int64_t n) {
  size_t sort_b = 0, rle_b = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, sort_b, static_cast<int64_t*>(nullptr), static_cast<int64_t*>(nullptr),
                                 static_cast<int>(n > 0 ? n : 1));
  cub::DeviceRunLengthEncode::Encode(nullptr, rle_b, static_cast<int64_t*>(nullptr), static_cast<int64_t*>(nullptr),
                                     static_cast<int32_t*>(nullptr), static_cast<int64_t*>(nullptr),
                                     static_cast<int>(n > 0 ? n : 1));
  const size_t nn = static_cast<size_t>(n > 0 ? n : 1);
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  return al(nn * 8) * 3 + al(nn * 4) + al(8) + al(sort_b > rle_b ? sort_b : rle_b) + 256;
}

// E_aᵀE_b in CSR: indptr (rows_a + 1), col / val (capacity n); *nnz (device) = stored entries
cudaError_t launch_pair_counts(int64_t n, const int32_t* ta, const int32_t* tb, int64_t rows_a, int64_t cols_b,
                               int64_t* indptr, int64_t* col, double* val, int64_t* nnz, void* ws, size_t ws_bytes,
                               cudaStream_t st, int num_sms) {
  if (ws_bytes < pair_counts_workspace_bytes(n)) return cudaErrorInvalidValue;
  if (n > INT32_MAX) return cudaErrorNotSupported;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t nn = static_cast<size_t>(n > 0 ? n : 1);
  char* p = static_cast<char*>(ws);
  int64_t* keys = reinterpret_cast<int64_t*>(p);
  p += al(nn * 8);
  int64_t* sorted = reinterpret_cast<int64_t*>(p);
  p += al(nn * 8);
  int64_t* ukeys = reinterpret_cast<int64_t*>(p);
  p += al(nn * 8);
  int32_t* cnt = reinterpret_cast<int32_t*>(p);
  p += al(nn * 4);
  p += al(8);
  void* tmp = p;
  size_t tmp_b = ws_bytes - static_cast<size_t>(p - static_cast<char*>(ws));
  cudaError_t e = cudaMemsetAsync(nnz, 0, 8, st);
  if (e != cudaSuccess) return e;
  if (n > 0) {
    const int grid = grid_for(n, 256, 8, num_sms);
    pair_keys_kernel<<<grid, 256, 0, st>>>(n, ta, tb, cols_b, keys);
    FB_LAUNCHED();
    int bits = 1;
    while (bits < 63 && (int64_t(1) << bits) < rows_a * cols_b) ++bits;
    e = cub::DeviceRadixSort::SortKeys(tmp, tmp_b, keys, sorted, static_cast<int>(n), 0, bits, st);
    if (e != cudaSuccess) return e;
    e = cub::DeviceRunLengthEncode::Encode(tmp, tmp_b, sorted, ukeys, cnt, nnz, static_cast<int>(n), st);
    if (e != cudaSuccess) return e;
  }
  pair_indptr_kernel<<<grid_for(rows_a + 1, 256, 4, num_sms), 256, 0, st>>>(ukeys, nnz, rows_a, cols_b, indptr);
  FB_LAUNCHED();
  pair_split_kernel<<<grid_for(n, 256, 8, num_sms), 256, 0, st>>>(ukeys, cnt, nnz, cols_b, col, val);
  FB_LAUNCHED();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ CSR · dense
// y[i, 0:k] (+)= Σ_p val[p]·x[col[p], 0:k] for rows i of a CSR matrix. A group of 2^lg lanes
// (the smallest power of two >= min(k, 32)) takes a row, so narrow products keep every lane busy
// (k = 16: two rows per warp, k = 1: 32); lanes over k in chunks of the group size. The entries of
// a row are taken eight at a time — eight (value, column) pairs, then eight independent x
// loads, then the eight FMAs in stored order (the reference's scipy csr @ dense order, so the
// sums are unchanged): the one-entry-at-a-time loop was a chain of dependent L2 round trips
// (c4's 100k × 10M-entry pair-count product: 0.54 ms per 16 columns).
template <typename IT>
__global__ void csr_spmm_kernel(int64_t rows, const int64_t* __restrict__ indptr, const IT* __restrict__ col,
                                const double* __restrict__ val, const double* __restrict__ x, int64_t ldx, int k,
                                double* y, int64_t ldy, int accumulate, int lg) {
  const int lane = threadIdx.x & 31;
  const int gl = lane & ((1 << lg) - 1);  // lane within the row group
  const int rpw = 32 >> lg;               // rows per warp
  const int gsz = 1 << lg;
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  for (int64_t i = w0 * rpw + (lane >> lg); i < rows; i += warps * rpw) {
    const int64_t p0 = indptr[i], p1 = indptr[i + 1];
    for (int c0 = 0; c0 < k; c0 += gsz) {
      const int c = c0 + gl;
      const bool on = c < k;
      const double* xc = x + (on ? c : 0);
      double s = 0.0;
      int64_t p = p0;
      for (; p + 8 <= p1; p += 8) {
        double v[8], xv[8];
        int64_t cc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          v[e] = __ldg(val + p + e);
          cc[e] = static_cast<int64_t>(__ldg(col + p + e));
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) xv[e] = __ldg(xc + cc[e] * ldx);
#pragma unroll
        for (int e = 0; e < 8; ++e) s = fma(v[e], xv[e], s);
      }
      for (; p < p1; ++p) s = fma(__ldg(val + p), __ldg(xc + static_cast<int64_t>(__ldg(col + p)) * ldx), s);
      if (on) y[i * ldy + c] = accumulate ? y[i * ldy + c] + s : s;
    }
  }
}

cudaError_t launch_csr_spmm(int64_t rows, const int64_t* indptr, const void* col, int col_is64, const double* val,
                            const double* x, int64_t ldx, int k, double* y, int64_t ldy, int accumulate,
                            cudaStream_t st, int num_sms) {
  if (rows <= 0 || k <= 0) return cudaSuccess;
  int lg = 0;
  while (lg < 5 && (1 << lg) < k) ++lg;
  const int rpw = 32 >> lg;
  const int grid = grid_for((rows + rpw - 1) / rpw * 32, 256, 8, num_sms);
  if (col_is64)
    csr_spmm_kernel<int64_t><<<grid, 256, 0, st>>>(rows, indptr, static_cast<const int64_t*>(col), val, x, ldx, k, y,
                                                   ldy, accumulate, lg);
  else
    csr_spmm_kernel<int32_t><<<grid, 256, 0, st>>>(rows, indptr, static_cast<const int32_t*>(col), val, x, ldx, k, y,
                                                   ldy, accumulate, lg);
  FB_LAUNCHED();
  return cudaGetLastError();
}

// Y = Pᵀ·X for a CSR P (rows × cols): y[col[p], :] += val[p]·x[i, :] (REDG, y zeroed by the
// launcher) — the transposed products (RMM / Tᵀ·X) of a CSR factor.
template <typename IT>
__global__ void csr_spmm_t_kernel(int64_t rows, const int64_t* __restrict__ indptr, const IT* __restrict__ col,
                                  const double* __restrict__ val, const double* __restrict__ x, int64_t ldx, int k,
                                  double* y, int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < rows; i += warps) {
    const int64_t p0 = indptr[i], p1 = indptr[i + 1];
    for (int c0 = 0; c0 < k; c0 += 32) {
      const int c = c0 + lane;
      if (c >= k) continue;
      const double xv = __ldg(x + i * ldx + c);
      for (int64_t p = p0; p < p1; ++p) red_add(y + static_cast<int64_t>(__ldg(col + p)) * ldy + c, __ldg(val + p) * xv);
    }
  }
}

cudaError_t launch_csr_spmm_t(int64_t rows, int64_t cols, const int64_t* indptr, const void* col, int col_is64,
                              const double* val, const double* x, int64_t ldx, int k, double* y, int64_t ldy,
                              cudaStream_t st, int num_sms) {
  cudaError_t e = cudaMemset2DAsync(y, static_cast<size_t>(ldy) * 8, 0, static_cast<size_t>(k) * 8,
                                    static_cast<size_t>(cols > 0 ? cols : 0), st);
  if (e != cudaSuccess || rows <= 0 || k <= 0 || cols <= 0) return e;
  const int grid = grid_for(rows * 32, 256, 8, num_sms);
  if (col_is64)
    csr_spmm_t_kernel<int64_t><<<grid, 256, 0, st>>>(rows, indptr, static_cast<const int64_t*>(col), val, x, ldx, k, y,
                                                     ldy);
  else
    csr_spmm_t_kernel<int32_t><<<grid, 256, 0, st>>>(rows, indptr, static_cast<const int32_t*>(col), val, x, ldx, k, y,
                                                     ldy);
  FB_LAUNCHED();
  return cudaGetLastError();
}

}  // namespace fb
