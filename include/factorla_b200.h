/* factorla_b200.h — C ABI of the B200 factorized linear-algebra library.
 *
 * The reference (factorla, /root/reference/pkg/src/factorla) is pure Python over
 * NumPy/SciPy/OpenBLAS and has no FFI layer of its own. The hot path
 * sits behind its operator functions in rewrite.py and the ML drivers in ml.py; each
 * entry point below replaces the native calls one of those functions makes, and the
 * Python package paper_1612_07448_b200 binds them through ctypes exactly where the
 * reference calls NumPy/SciPy/BLAS (see INTEGRATION.md for the binding).
 *
 * Conventions
 *  - All pointers are DEVICE pointers unless stated; matrices are row-major float64,
 *    FK columns int32 (0-based targets after remapping), sizes int64.
 *  - Every compute entry point is stream-ordered on `stream`, performs no host
 *    synchronisation and is CUDA-graph capturable. Scratch memory comes from the
 *    caller's workspace (`ws`, `ws_bytes`); query the size with the *_workspace_bytes
 *    function. The library never frees caller memory.
 *  - Return value: FB_OK or an FB_ERR_* code; fb_last_error() gives the message
 *    (thread-local). The Python layer maps codes to the reference's exception classes
 *    (exceptions.py: ShapeError, DataError, NumericError).
 */
#ifndef FACTORLA_B200_H
#define FACTORLA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* fb_stream_t; /* == cudaStream_t */

#define FB_ABI_VERSION 4
#define FB_MAX_PARTS 4

enum {
  FB_OK = 0,
  FB_ERR_ARG = 1,     /* bad argument (null pointer, unsupported size) -> ValueError */
  FB_ERR_SHAPE = 2,   /* non-conforming operands -> ShapeError */
  FB_ERR_CUDA = 3,    /* CUDA runtime / launch failure -> RuntimeError */
  FB_ERR_DATA = 4,    /* bad keys -> DataError */
  FB_ERR_NUMERIC = 5, /* numeric failure -> NumericError */
  FB_ERR_NCCL = 6
};

/* One attribute block (K_i, R_i) of a normalized matrix (normmat.py:47-130). */
typedef struct fb_part {
  const int32_t* fk;    /* n_s targets into rows of r (IndicatorMatrix.target, indicator.py:35) */
  const double* r;      /* n_r x d_r row-major attribute table (unreferenced rows dropped) */
  int64_t n_r;
  int32_t d_r;
  int32_t skewed;       /* hint: some target holds a large share of rows (scatter kernels then
                           combine equal keys within a warp before the atomic); 0 = uniform */
  const double* counts; /* optional cached colSums(K) as f64 (indicator.py:61-66); may be NULL */
  /* optional hot-target tables for skewed FKs (scatter kernels privatise these bins per CTA):
     hot_slot[n_r] = slot in [0, nhot) for the nhot most frequent targets, -1 otherwise;
     hot_key[nhot] = the targets. nhot = 0 disables. */
  const int16_t* hot_slot;
  const int32_t* hot_key;
  int32_t nhot;
  /* optional FK-sorted order (fb_fk_sort): when set, X·K scatters run as segmented sums
     over sorted positions instead of one atomic per row */
  const int32_t* perm;
  const int32_t* fk_sorted;
} fb_part;

/* Untransposed PK-FK / star normalized matrix T = [S, K_1 R_1, ..., K_q R_q]. */
typedef struct fb_normalized {
  const double* s; /* n_s x d_s row-major entity table (d_s may be 0) */
  int64_t n_s;
  int32_t d_s;
  int32_t q;       /* number of attribute blocks, 0..FB_MAX_PARTS */
  fb_part part[FB_MAX_PARTS];
} fb_normalized;

/* ---- library ---------------------------------------------------------------- */
int fb_abi_version(void);
const char* fb_last_error(void);
/* Cache the SM count of `device` (the caller's current device is not changed). */
int fb_init(int device);
/* Number of kernels this library has launched in this process (instrumentation). */
uint64_t fb_launch_count(void);

/* ---- construction (normmat.py:182-237, indicator.py:61-66) --------------------- */
/* counts_full[j] = #{i : key[i] == j+1}; *first_bad = smallest i with key outside
 * [1, n_r] or UINT64_MAX (device scalar). Replaces _check_keys' validation. */
int fb_key_check(const int64_t* key, int64_t n, int64_t n_r, int32_t* counts_full,
                 unsigned long long* first_bad, fb_stream_t stream);
size_t fb_key_remap_workspace_bytes(int64_t n_r);
/* _remap_part (normmat.py:168-179): lookup[j] = rank of j among used keys or -1,
 * *n_used (device), target[i] = lookup[key[i]-1], used_idx[l] = j, counts_kept[l]. */
int fb_key_remap(const int64_t* key, int64_t n, int64_t n_r, const int32_t* counts_full,
                 int32_t* lookup, int32_t* n_used, int32_t* target, int64_t* used_idx,
                 int32_t* counts_kept, void* ws, size_t ws_bytes, fb_stream_t stream);
/* bincount of 0-based targets (IndicatorMatrix.counts). */
int fb_fk_counts(const int32_t* fk, int64_t n, int32_t* counts, int64_t n_r, fb_stream_t stream);
/* out[r,:] = in[idx[r],:]  (ndarray.take(axis=0)); idx int64. */
int fb_gather_rows(const double* in, int64_t ld_in, const int64_t* idx, int64_t nrows, int32_t d,
                   double* out, int64_t ld_out, fb_stream_t stream);
int fb_gather_rows_i32(const double* in, int64_t ld_in, const int32_t* idx, int64_t nrows,
                       int32_t d, double* out, int64_t ld_out, fb_stream_t stream);
int fb_i32_to_f64(const int32_t* in, double* out, int64_t n, fb_stream_t stream);
/* Sparse factor matrix ingestion (kernel.py:110-121 stores factors as scipy CSR; dataio.py:208-214
 * picks CSR at density <= 5%): canonical CSR (sorted, duplicate-free; indptr int64[nrows+1],
 * indices int32[nnz], data f64[nnz]) expanded into the dense row-major layout (ld_out >= ncols). */
int fb_csr_expand(const int64_t* indptr, const int32_t* indices, const double* data, int64_t nrows,
                  int32_t ncols, double* out, int64_t ld_out, fb_stream_t stream);

/* ---- operators (rewrite.py) ------------------------------------------------------ */
/* LMM T·X (rewrite.py:172-191). x: d x d_x row-major, d = d_s + sum d_r; out: n_s x d_x. */
size_t fb_lmm_workspace_bytes(const fb_normalized* nm, int32_t d_x);
int fb_lmm(const fb_normalized* nm, const double* x, int32_t d_x, double* out, void* ws,
           size_t ws_bytes, fb_stream_t stream);

/* FK-band layout of a PK-FK / star matrix: a cached copy of S and of the FK columns with the rows
 * grouped into n_bands contiguous key ranges of part 0 (band of row i = fk_0[i]·n_bands / n_r;
 * storage order kept inside a band — a stable sort), plus the permutation back to storage
 * order. The device analogue of the reference's cached derived layouts of K (indicator.py:71-86):
 * built once per matrix, it lets a pass over S gather z_0 = R_0·X from one L2-resident slice at a
 * time when the whole table is larger than L2. Used by the K-Means step (every result there is
 * a sum over rows) and, opt-in, by the wide-X LMM. */
typedef struct fb_band_layout {
  int32_t n_bands;
  const int32_t* perm;             /* n_s: storage row of band position i */
  const int32_t* fk[FB_MAX_PARTS]; /* n_s each: part[q].fk in band order */
  const double* s;                 /* n_s x d_s: S rows in band order */
} fb_band_layout;
size_t fb_band_build_workspace_bytes(int64_t n);
/* Elements between the parts of fk_band (n rounded up so every part starts 256-byte aligned). */
int64_t fb_band_fk_stride(int64_t n);
/* fk_band: q x fb_band_fk_stride(n_s) int32 (part-major); s_band: n_s x d_s. */
int fb_band_build(const fb_normalized* nm, int32_t n_bands, int32_t* perm, int32_t* fk_band,
                  double* s_band, void* ws, size_t ws_bytes, fb_stream_t stream);
/* out[perm[i]] = in[i] (band order back to storage order). */
int fb_scatter_i32(const int32_t* in, const int32_t* perm, int64_t n, int32_t* out, fb_stream_t stream);
/* fb_lmm with the S pass reading the band layout (q = 1, d_s <= 32, column chunks of 8 or 16;
 * other shapes run fb_lmm's storage-order pass). Results are bitwise equal to fb_lmm's. */
int fb_lmm_banded(const fb_normalized* nm, const fb_band_layout* band, const double* x, int32_t d_x,
                  double* out, void* ws, size_t ws_bytes, fb_stream_t stream);

/* rowSums(T) (rewrite.py:118-128): out n_s x 1. */
size_t fb_row_sums_workspace_bytes(const fb_normalized* nm);
int fb_row_sums(const fb_normalized* nm, double* out, void* ws, size_t ws_bytes,
                fb_stream_t stream);

/* Weighted transposed product out(j, c) = sum_i w(i, j) T(i, c), j < n_w, c < d, with
 * w(i, j) = w[i*w_rs + j*w_cs] and out(j, c) = out[j*o_js + c*o_cs]. Covers
 *   rmm X·T (rewrite.py:194-212):          w = X^T  (w_rs = 1,   w_cs = n_s)
 *   lmm on T.T, i.e. T^T·X (rewrite.py:182-183): w = X (w_rs = n_w, w_cs = 1)
 * The X·K halves are FK scatter-adds (indicator.py:130-141) fused into the S pass. */
size_t fb_wt_workspace_bytes(const fb_normalized* nm, int32_t n_w);
int fb_wt(const fb_normalized* nm, const double* w, int32_t n_w, int64_t w_rs, int64_t w_cs,
          double* out, int64_t o_js, int64_t o_cs, void* ws, size_t ws_bytes, fb_stream_t stream);

/* colSums(T) (rewrite.py:131-149): out 1 x d. Uses part.counts when given. */
size_t fb_col_sums_workspace_bytes(const fb_normalized* nm);
int fb_col_sums(const fb_normalized* nm, double* out, void* ws, size_t ws_bytes,
                fb_stream_t stream);
/* sum(T) (rewrite.py:152-165): out[0] (device scalar). */
int fb_sum_all(const fb_normalized* nm, double* out, void* ws, size_t ws_bytes,
               fb_stream_t stream);

/* FK-sorted row order (the GPU analogue of IndicatorMatrix._csr_t's stable argsort,
 * indicator.py:78-86): perm[j] = j-th row in ascending (fk, row) order, fk_sorted[j] =
 * fk[perm[j]]. Built once per indicator and cached by the caller. */
size_t fb_fk_sort_workspace_bytes(int64_t n);
int fb_fk_sort(const int32_t* fk, int64_t n, int64_t n_r, int32_t* perm, int32_t* fk_sorted, void* ws,
               size_t ws_bytes, fb_stream_t stream);

/* crossprod(T) = TᵀT (rewrite.py:245-298, efficient method), exactly symmetric; out is
 * d × d row-major. q = 0 (plain SᵀS) or q = 1 with perm/fk_sorted from fb_fk_sort and
 * part[0].counts set. For an even d_s <= 128 the S side is one pass over S in FK-sorted order
 * (SᵀS on the FP64 tensor cores and KᵀS as a segmented sum from the same tiles); the R side
 * is a second pass over R with B = KᵀS. A star schema (q >= 2) is composed from one call per
 * part on [S, K_i R_i] plus pair-count cross blocks (fb_pair_counts, fb_csr_spmm, fb_rows_wt);
 * odd / wider S and M:N matrices go through fb_wt per block column (crossprod_impl.py). */
size_t fb_crossprod_workspace_bytes(const fb_normalized* nm);
int fb_crossprod(const fb_normalized* nm, const int32_t* perm, const int32_t* fk_sorted, double* out, void* ws,
                 size_t ws_bytes, fb_stream_t stream);

/* ---- split passes: the R-row-sliced multi-GPU composition (dist.py) ----
 * Each operator's S pass runs on a rank's own S rows; its R-side work runs on the rank's slice
 * of R rows, joined by all-gather (z) / reduce-scatter (bins, KᵀS) / all-reduce (small results)
 * in the caller. Single-GPU callers use the whole-operator entries above. */
/* Doubles per z row for d_x <= 16 columns (even: gathered rows are 16-byte copies); 0 otherwise. */
int fb_z_stride(int32_t d_x);
/* z rows [row_lo, row_hi) of part `part`: z[r*zst + c] = (R_part · X[off_part : off_part + d_r, :])[r, c]
 * (rewrite.py:187, "R·X before K"); z is the base of the whole n_r × zst table. d_x <= 16. */
int fb_lmm_zpass(const fb_normalized* nm, const double* x, int32_t d_x, int32_t part, int64_t row_lo, int64_t row_hi,
                 double* z, fb_stream_t stream);
/* out = S·X[0:d_s] + Σ_i z_i[fk_i] with caller z tables (n_r,i × fb_z_stride(d_x)); d_x <= 16
 * (rewrite.py:186-190). */
int fb_lmm_spass(const fb_normalized* nm, const double* x, int32_t d_x, const double* const* z, double* out,
                 fb_stream_t stream);
/* The S pass of fb_wt: out(j, c) = Σ_i w(i, j) S(i, c) for c < d_s (w = NULL: all-ones weights,
 * i.e. colSums(S)), and bins[i] (n_r,i × n_w row-major, zeroed here) = X·K_i (indicator.py:130-141)
 * for every part whose bins[i] is not NULL (bins = NULL: none). n_w <= 16. */
size_t fb_wt_spass_workspace_bytes(const fb_normalized* nm, int32_t n_w);
int fb_wt_spass(const fb_normalized* nm, const double* w, int32_t n_w, int64_t w_rs, int64_t w_cs, double* out,
                int64_t o_js, int64_t o_cs, double* const* bins, void* ws, size_t ws_bytes, fb_stream_t stream);
/* Weighted column sums of dense rows: out(j, c) = Σ_i w(i, j) a(i, c) (the binsᵀ·R / counts·R
 * pass of rmm / colSums on one R-row slice, rewrite.py:131-149, 194-212). */
size_t fb_rows_wt_workspace_bytes(int32_t d, int32_t n_w);
int fb_rows_wt(const double* a, int64_t n, int32_t d, const double* w, int32_t n_w, int64_t w_rs, int64_t w_cs,
               double* out, int64_t o_js, int64_t o_cs, void* ws, size_t ws_bytes, fb_stream_t stream);
/* The two halves of fb_crossprod (workspace: fb_crossprod_workspace_bytes). spass: out = the
 * SᵀS block (rest zero) and kts (n_r × d_s) = KᵀS of this rank's rows. rpass: nm->part[0] is one
 * R-row slice (r, n_r, counts of that slice) and kts its KᵀS rows: out = the blocks involving R
 * ((KᵀS)ᵀR and Rᵀdiag(c)R, both triangles; rest zero). Summing the halves over ranks and slices
 * gives TᵀT (rewrite.py:245-298). */
int fb_crossprod_spass(const fb_normalized* nm, const int32_t* perm, const int32_t* fk_sorted, double* out,
                       double* kts, void* ws, size_t ws_bytes, fb_stream_t stream);
int fb_crossprod_rpass(const fb_normalized* nm, const double* kts, double* out, void* ws, size_t ws_bytes,
                       fb_stream_t stream);

/* ---- ML driver steps (ml.py) ------------------------------------------------------ */
/* One fused GLM evaluation over T (d = d_s + Σ d_r, w a device d-vector, y n_s targets):
 *   mode 0 (logistic_gd, ml.py:207-213): p = y/(1+exp(T w)), loss = Σ log1p(exp(-|y·Tw|)) + max(-y·Tw, 0)
 *   mode 1 (linreg_gd,   ml.py:247-252): p = T w - y,        loss = Σ p²
 * writes g = Tᵀp (d) and *loss (device). S is read once (Tw, p and Sᵀp in one pass). */
size_t fb_glm_workspace_bytes(const fb_normalized* nm);
int fb_glm_eval(const fb_normalized* nm, const double* y, const double* w, int32_t mode, double* g, double* loss,
                void* ws, size_t ws_bytes, fb_stream_t stream);
/* fb_glm_eval followed by w += alpha·g, trace[it] = loss, and *diverged = it at the first
 * iteration whose weights are not finite (ml.py:190-192; *diverged starts at -1). */
int fb_glm_step(const fb_normalized* nm, const double* y, double* w, int32_t mode, double alpha, int32_t it,
                double* trace, int32_t* diverged, void* ws, size_t ws_bytes, fb_stream_t stream);
/* A whole GD run (iters steps of fb_glm_step: ml.py:199-215 / 239-254). When the factors are
   L2-resident it runs as ONE cooperative launch (three grid barriers per iteration), else as
   iters fused steps. w, trace[iters] and *diverged (= -1) are initialised by the caller;
   results match fb_glm_step's up to the order of the Kᵀp atomics.
   Replaces the reference's driver loop ml.py:205-214 / 245-253. */
size_t fb_glm_run_workspace_bytes(const fb_normalized* nm);
/* 1 when fb_glm_run takes the single cooperative launch for this matrix (not graph-captured). */
int fb_glm_run_fused(const fb_normalized* nm);
int fb_glm_run(const fb_normalized* nm, const double* y, double* w, int32_t mode, double alpha, int32_t iters,
               double* trace, int32_t* diverged, void* ws, size_t ws_bytes, fb_stream_t stream);

/* One K-Means iteration (ml.py:275-283) on an untransposed T with k <= 4096 clusters (k <= 16: one
 * fused pass over S; above: chunked T·(2C), assign, one-hot and R passes):
 * c is the d × k centroid matrix (updated in place; empty clusters keep theirs), cc[j] =
 * Σ c[:, j]² (in/out), d_t = rowSums(T²) (n_s), assign (n_s int32) the argmin cluster
 * (ties to the lowest index), trace[it] = Σ_i min_j dist, *nan_row = (it << 40) | row for the
 * first row whose distances hold a NaN in the first iteration that had one (device; start at
 * UINT64_MAX; atomicMin keeps the earliest). */
size_t fb_kmeans_workspace_bytes(const fb_normalized* nm, int32_t k);
int fb_kmeans_step(const fb_normalized* nm, const double* d_t, double* c, double* cc, int32_t k, int32_t it,
                   double* trace, int32_t* assign, unsigned long long* nan_row, void* ws, size_t ws_bytes,
                   fb_stream_t stream);

/* fb_kmeans_step reading the rows through an FK-band layout: d_t and assign are in band order
 * (d_t_band[i] = d_t[perm[i]]; fb_scatter_i32 brings the final assign back), *nan_row holds a band
 * position. Needs the fused pass (k <= 16, d_s <= 32); every other output is a sum over rows. */
int fb_kmeans_step_banded(const fb_normalized* nm, const fb_band_layout* band, const double* d_t_band, double* c,
                          double* cc, int32_t k, int32_t it, double* trace, int32_t* assign_band,
                          unsigned long long* nan_row, void* ws, size_t ws_bytes, fb_stream_t stream);
/* 1 when fb_kmeans_step_banded can run this shape. */
int fb_kmeans_banded_supported(const fb_normalized* nm, int32_t k);

/* The two halves of fb_kmeans_step, for row-sharded data: the partial writes this shard's
 * TᵀA (d × k row-major) and integer cluster sizes (k) and its objective into trace[it];
 * after summing those over the shards, fb_kmeans_update moves the centroids (empty
 * clusters keep theirs) and refreshes cc. */
int fb_kmeans_partial(const fb_normalized* nm, const double* d_t, const double* c, const double* cc, int32_t k,
                      int32_t it, double* trace, int32_t* assign, unsigned long long* nan_row, double* tta,
                      int32_t* sizes, void* ws, size_t ws_bytes, fb_stream_t stream);
int fb_kmeans_update(double* c, const double* tta, const int32_t* sizes, int64_t d, int32_t k, double* cc,
                     fb_stream_t stream);

/* One GNMF multiplicative-update iteration (ml.py:306-315), r <= 256 (r <= 16: one fused pass over S per
 * W step; wider r: operator by operator): w (n_s × r), h (d × r),
 * ttw = Tᵀw (d × r, in: for the current w, out: for the updated w), cpw = wᵀw (r × r,
 * in/out), sum_t2 = Σ T² (device scalar), trace[it] = Frobenius objective. */
size_t fb_gnmf_workspace_bytes(const fb_normalized* nm, int32_t r);
int fb_gnmf_step(const fb_normalized* nm, double* w, double* h, double* ttw, double* cpw, const double* sum_t2,
                 int32_t r, int32_t it, double* trace, void* ws, size_t ws_bytes, fb_stream_t stream);

/* GLM update on its own (after an all-reduce of g and loss over the shards). */
int fb_glm_update(double* w, const double* g, int64_t d, double alpha, const double* loss, double* trace, int32_t it,
                  int32_t* diverged, fb_stream_t stream);
/* GNMF building blocks (ml.py:306-315): f = f ∘ num / (f·g + 1e-12) for a rows × r factor
 * and r × r g; g = fᵀf with an exact mirror; the Frobenius objective into trace[it]. */
int fb_nmf_update(double* f, const double* num, const double* g, int64_t rows, int32_t r, fb_stream_t stream);
int fb_small_gram(const double* f, int64_t rows, int32_t r, double* g, fb_stream_t stream);
int fb_nmf_objective(const double* sum_t2, const double* ttw, const double* h, int64_t dr, const double* cpw,
                     const double* cph, int32_t rr, double* trace, int32_t it, fb_stream_t stream);

/* a[r, c] = a[c, r] for r > c: exact symmetry from the upper triangle of a d × d matrix
 * (kernel._mirror_upper, kernel.py:132-135). */
int fb_mirror_upper(double* a, int64_t d, fb_stream_t stream);

/* Element-wise scalar op / function on one factor matrix (kernel.py:219-300).
 * op: 0 add 1 radd 2 sub 3 rsub 4 mul 5 rmul 6 div 7 rdiv 8 pow 9 rpow
 * fn: 0 exp 1 log 2 square 3 sqrt 4 abs 5 negative 6 log1p 7 expm1 8 sin 9 cos 10 tanh
 *     11 sigmoid 12 reciprocal 13 identity */
int fb_scalar_map(const double* in, double* out, int64_t n, int32_t op, double x,
                  fb_stream_t stream);
int fb_unary_map(const double* in, double* out, int64_t n, int32_t fn, fb_stream_t stream);

/* ---- dense / sparse pieces of the rest of the operator surface ---- */
/* C[m x n] (+)= op(A)·op(B) on the FP64 tensor cores, row-major; op(A)[i][k] = ta ? A[k*lda+i]
 * : A[i*lda+k], op(B)[k][j] = tb ? B[j*ldb+k] : B[k*ldb+j]. The block products of
 * gram_transposed / dmm / dmm_gram (rewrite.py:301-446; kernel.py:110-121 dense @). */
int fb_dense_mm(int64_t m, int64_t n, int64_t k, const double* a, int64_t lda, int32_t ta, const double* b,
                int64_t ldb, int32_t tb, double* c, int64_t ldc, int32_t accumulate, fb_stream_t stream);
/* c[i, j] += mat[ra[i], cb ? cb[j] : j]: the two-sided indicator expansion E_a M E_b^T of a block
 * product (rewrite.py:308-313, 436-444). */
int fb_gather2_add(int64_t m, int64_t n, const double* mat, int64_t ldm, const int32_t* ra, const int32_t* cb,
                   double* c, int64_t ldc, fb_stream_t stream);
/* out[tgt[i], :] += a[i, :] (out: out_rows x d, zeroed here): E^T a (indicator.py:107-118). */
int fb_scatter_rows(int64_t n, int32_t d, const int32_t* tgt, const double* a, int64_t lda, double* out,
                    int64_t out_rows, fb_stream_t stream);
/* E_a^T E_b as CSR counts (indicator.py:144-162): indptr[rows_a + 1], col / val with capacity n,
 * *nnz (device int64) = stored entries, columns ascending within a row. */
size_t fb_pair_counts_workspace_bytes(int64_t n);
int fb_pair_counts(int64_t n, const int32_t* ta, const int32_t* tb, int64_t rows_a, int64_t cols_b, int64_t* indptr,
                   int64_t* col, double* val, int64_t* nnz, void* ws, size_t ws_bytes, fb_stream_t stream);
/* y (+)= P·x for a CSR P (rows x ?, int64 indptr, int32 or int64 column indices, f64 values):
 * scipy's csr @ dense (kernel.py:110-121, the sparse factor products). */
int fb_csr_spmm(int64_t rows, const int64_t* indptr, const void* col, int32_t col_is64, const double* val,
                const double* x, int64_t ldx, int32_t k, double* y, int64_t ldy, int32_t accumulate,
                fb_stream_t stream);
/* y = P^T·x for a CSR P (rows x cols): y is cols x k, zeroed here (kernel.py:141-148 csr.T @). */
int fb_csr_spmm_t(int64_t rows, int64_t cols, const int64_t* indptr, const void* col, int32_t col_is64,
                  const double* val, const double* x, int64_t ldx, int32_t k, double* y, int64_t ldy,
                  fb_stream_t stream);

/* Point-wise halves of the GD loops on a transposed matrix (ml.py:207-213, 247-252 with T = M^T,
 * where T·w and T^T·p come from fb_wt / fb_lmm): p and the summed loss from tw = T·w and y
 * (mode 0 logistic: p = y / (1 + exp(tw)), the stable log-loss; mode 1: p = tw - y, Σp²) into
 * trace[it]; and w += alpha·g with *diverged (start at -1) latching the first iteration that
 * left a non-finite weight. */
size_t fb_glm_pointwise_workspace_bytes(void);
int fb_glm_pointwise(const double* tw, const double* y, int64_t n, int32_t mode, double* p, double* trace,
                     int32_t it, void* ws, size_t ws_bytes, fb_stream_t stream);
int fb_axpy_check(double alpha, const double* x, double* y, int64_t n, int32_t it, int32_t* diverged,
                  fb_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* FACTORLA_B200_H */
