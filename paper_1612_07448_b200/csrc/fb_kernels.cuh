// fb_kernels.cuh — internal launcher declarations shared by the .cu files and the C-ABI.
#pragma once
#include "fb_stream.cuh"

namespace fb {

constexpr int kMaxParts = 4;  // attribute tables per star schema handled in one pass

// fb_lmm.cu ------------------------------------------------------------------------
// out[i, 0:dx] (ld ldo) = a[i, :] · x (d × dx, ld ldx) + Σ_q z_q[fk_q[i], 0:dx]
// z_q rows have zstride doubles (even, >= dx): see z_stride().
inline int z_stride(int dx) { return dx < 2 ? 2 : (dx + 1) & ~1; }
cudaError_t launch_lmm_rows(const double* a, int64_t n, int d, const double* x, int dx, int64_t ldx,
                            int nfk, const int32_t* const* fk, const double* const* z, int zstride, double* out,
                            int64_t ldo, cudaStream_t st, int num_sms, const int64_t* z_rows = nullptr);

// S pass over an FK-band layout (fb_band_layout): rows of a_band / fk_band / perm in band order.
bool lmm_band_supported(int d, int dx, int64_t ldo, const double* out);
cudaError_t launch_lmm_band(const double* a_band, const int32_t* fk_band, const int32_t* perm, int64_t n, int d,
                            const double* x, int dx, int64_t ldx, const double* z, int zstride, int64_t z_rows,
                            double* out, int64_t ldo, cudaStream_t st, int num_sms);

// fb_reduce.cu ---------------------------------------------------------------------
struct ColReduce {
  const double* a;  // rows streamed: n × d row-major
  int64_t n;
  int d;
  int nx;           // weight columns (1 with w == nullptr means all-ones weights)
  const double* w;  // w(i, j) = w[i*w_rs + j*w_cs]
  int64_t w_rs, w_cs;
  int nfk;                         // fused Kᵀ scatter of the same weights
  const int32_t* fk[kMaxParts];    // (original row order; warp-aggregated atomics)
  double* bins[kMaxParts];         // n_R,q × nx row-major, zeroed by the launcher
  int64_t nbins[kMaxParts];
  int aggregate[kMaxParts];        // warp-aggregate equal keys (skewed FK)
  const int16_t* hot_slot[kMaxParts];  // per target: slot of the hottest targets, -1 otherwise
  const int32_t* hot_key[kMaxParts];   // slot -> target
  int nhot[kMaxParts];                 // hot slots (0: none)
  double* out;                     // out(j, c) = out[j*o_js + c*o_cs]
  int64_t o_js, o_cs;
  double* partials;                // workspace: grid × nx × d
  unsigned int* counter;           // workspace: one zeroed word
};
size_t colreduce_workspace_doubles(int64_t n, int d, int nx, int num_sms);
// bins(key, j) = Σ_{p: keys[p] = key} w(perm[p], j) over FK-sorted positions (zeroes bins first)
cudaError_t launch_segsum(const int32_t* perm, const int32_t* keys, int64_t n, const double* w, int64_t w_rs,
                          int64_t w_cs, int nx, double* bins, int64_t n_bins, cudaStream_t st, int num_sms);
cudaError_t launch_colreduce(const ColReduce& c, cudaStream_t st, int num_sms);

// fb_elementwise.cu ------------------------------------------------------------------
enum ScalarOp : int {
  kAdd = 0, kRadd, kSub, kRsub, kMul, kRmul, kDiv, kRdiv, kPow, kRpow
};
enum UnaryFn : int {
  kExp = 0, kLog, kSquare, kSqrt, kAbs, kNeg, kLog1p, kExpm1, kSin, kCos, kTanh, kSigmoid,
  kReciprocal, kIdentity
};
cudaError_t launch_scalar_map(const double* in, double* out, int64_t n, int op, double x,
                              cudaStream_t st, int num_sms);
size_t glm_pointwise_workspace_bytes(int num_sms);
cudaError_t launch_glm_pointwise(const double* tw, const double* y, int64_t n, int mode, double* p, double* trace,
                                 int it, void* ws, cudaStream_t st, int num_sms);
cudaError_t launch_axpy_check(double alpha, const double* x, double* y, int64_t n, int it, int* diverged,
                              cudaStream_t st, int num_sms);
cudaError_t launch_unary_map(const double* in, double* out, int64_t n, int fn, cudaStream_t st,
                             int num_sms);

// fb_build.cu ------------------------------------------------------------------------
cudaError_t launch_key_check_hist(const int64_t* key, int64_t n, int64_t n_r, int32_t* counts,
                                  unsigned long long* first_bad, cudaStream_t st, int num_sms);
cudaError_t launch_used_scan(const int32_t* counts, int64_t n_r, int32_t* lookup,
                             int32_t* n_used, int32_t* block_ws, cudaStream_t st, int num_sms);
size_t used_scan_ws_ints(int64_t n_r);
cudaError_t launch_remap(const int64_t* key, int64_t n, const int32_t* lookup,
                         const int32_t* counts, int64_t n_r, int32_t* target, int64_t* used_idx,
                         int32_t* counts_kept, cudaStream_t st, int num_sms);
cudaError_t launch_fk_hist(const int32_t* fk, int64_t n, int32_t* counts, int64_t nbins,
                           cudaStream_t st, int num_sms);
cudaError_t launch_gather_rows(const double* in, int64_t ld_in, const int64_t* idx64,
                               const int32_t* idx32, int64_t nrows, int d, double* out,
                               int64_t ld_out, cudaStream_t st, int num_sms);
cudaError_t launch_i32_to_f64(const int32_t* in, double* out, int64_t n, cudaStream_t st,
                              int num_sms);
cudaError_t launch_csr_expand(const int64_t* indptr, const int32_t* indices, const double* data,
                              int64_t nrows, int32_t ncols, double* out, int64_t ld_out,
                              cudaStream_t st, int num_sms);

// fb_crossprod.cu --------------------------------------------------------------------
// Crossprod of a PK-FK (q = 1) or dense (q = 0) normalized matrix.
struct CrossArgs {
  const double* s;
  int64_t n_s;
  int d_s;
  const int32_t* perm;       // FK-sorted order of S rows (q = 1)
  const int32_t* fk_sorted;  // fk[perm]
  const double* r;           // nullptr when q = 0
  int64_t n_r;
  int d_r;
  const double* counts;      // f64 colSums(K)
  double* out;               // d × d, d = d_s + d_r
  // split passes for R-row-sliced multi-GPU crossprod (dist.py): 0 = whole, 1 = S pass only
  // (SᵀS block of out, KᵀS into kts), 2 = R pass only (r / n_r / counts / kts = one R slice;
  // out gets only the blocks that involve R)
  int mode;
  double* kts;               // caller KᵀS (n_r × d_s): written in mode 1, read in mode 2
};
size_t fk_sort_workspace_bytes(int64_t n);
cudaError_t launch_fk_sort(const int32_t* fk, int64_t n, int64_t n_r, int32_t* perm, int32_t* fk_sorted, void* ws,
                           size_t ws_bytes, cudaStream_t st, int num_sms);
// Library-owned side stream (fb_capi.cu): fork from / join back into `main` (graph-capturable).
cudaError_t side_fork(cudaStream_t main, cudaStream_t* side);
cudaError_t side_join(cudaStream_t main);

// out(c, j) = Σ_r R(r, c)·X(r, j) on the FP64 tensor cores (fb_crossprod.cu); nx even.
bool rtx_supported(int d_r, int nx);
size_t rtx_workspace_bytes(int d_r, int nx, int num_sms);
cudaError_t launch_rtx(const double* r, int64_t n_r, int d_r, const double* x, int nx, double* out, int64_t o_rs,
                       int64_t o_cs, void* ws, size_t ws_bytes, cudaStream_t st, int num_sms);

size_t crossprod_workspace_bytes(int64_t n_s, int d_s, int64_t n_r, int d_r, int q, int num_sms);
cudaError_t launch_crossprod(const CrossArgs& c, void* ws, size_t ws_bytes, cudaStream_t st, int num_sms);

// fb_ml.cu --------------------------------------------------------------------------
struct GlmArgs {
  const double* s;  // n × d entity rows
  int64_t n;
  int d;
  const double* y;  // n labels / targets
  const double* w;  // d entity weights
  int mode;         // 0: logistic (ml.py:207-213), 1: least squares (ml.py:247-252)
  int nfk;
  const int32_t* fk[kMaxParts];
  const double* z[kMaxParts];  // R_q·w_q
  double* bins[kMaxParts];     // Kᵀp accumulators (zeroed by the caller)
  double* g_out;               // d: Sᵀp
  double* loss_out;            // 1
  double* partials;            // glm_partials_doubles
  unsigned* counter;           // one zeroed word
};
size_t glm_partials_doubles(int d, int num_sms);

// Whole GD run in one cooperative launch (fb_glm_run.cu), for L2-resident problems.
struct GlmRunIn {
  const double* s;
  int64_t n;
  int ds;
  const double* y;
  int mode;
  double alpha;  // the step size (sign applied per mode)
  int q;
  const int32_t* fk[kMaxParts];
  const double* r[kMaxParts];
  int64_t nr[kMaxParts];
  int dr[kMaxParts];
  double* w;
  int iters;
  double* trace;
  int* diverged;
};
bool glm_run_eligible(int64_t n, int ds, int q, const int* dr, int num_sms);
size_t glm_run_workspace_bytes(int d, const int64_t* nr, int q, int num_sms);
cudaError_t launch_glm_run(const GlmRunIn& in, void* ws, size_t ws_bytes, cudaStream_t st, int num_sms);
cudaError_t launch_glm_spass(const GlmArgs& g, cudaStream_t st, int num_sms);
cudaError_t launch_glm_update(double* w, const double* g, int d, double alpha, const double* loss, double* trace,
                              int it, int* diverged, cudaStream_t st);

// Widest K-Means / GNMF problems of the operator-by-operator steps (k, r <= 16 take the fused passes):
// the assign pass keeps cc[k] and k size counters in shared memory, the NMF update an r-wide row
// per warp; the gram of W is a q = 0 crossprod (d <= 256).
constexpr int kKmeansMaxK = 4096;
constexpr int kNmfStepMaxR = 256;

struct KmFk {
  int nfk;
  const int32_t* fk[kMaxParts];
  int32_t* bins[kMaxParts];  // n_R,q × k integer histograms (zeroed by the caller)
};
cudaError_t launch_kmeans_assign(const double* tc, const double* d_t, const double* cc, int64_t n, int k,
                                 const KmFk& fks, int32_t* assign, int32_t* sizes, double* partials, unsigned* counter,
                                 double* trace, int it, unsigned long long* nan_row, cudaStream_t st, int num_sms);
// One fused pass over S per K-Means iteration (fb_kmeans.cu): T·(2C), argmin, objective,
// sizes, K_qᵀA histograms and SᵀA.
struct KmPass {
  const double* s;  // n × d entity rows (d <= 32; d may be 0)
  int64_t n;
  int d;
  const double* d_t;  // rowSums(T²)
  const double* c2s;  // (2C)[0:d, :] row-major d × k
  const double* cc;   // Σ_r c[r, j]²
  int k;              // <= 16
  int nfk;
  const int32_t* fk[kMaxParts];
  const double* z[kMaxParts];  // R_q·(2C)_q, n_R,q × zst
  size_t ztable_bytes[kMaxParts];
  int zst;
  int32_t* bins[kMaxParts];  // n_R,q × k, zeroed by the caller
  int32_t* assign;
  int32_t* sizes;            // k, zeroed by the caller
  double* partials;          // kmeans_pass_partials_doubles
  unsigned* counter;         // one word (zeroed by the launcher)
  double* trace;
  int it;
  unsigned long long* nan_row;
  double* sta;               // SᵀA into tta[c*k + j], c < d
  bool rr;                   // rows in FK-band order: round-robin tiles (fb_band_layout)
};
bool kmeans_pass_supported(int d_s, int k, int nfk);
size_t kmeans_pass_partials_doubles(int num_sms);
cudaError_t launch_kmeans_pass(const KmPass& p, cudaStream_t st, int num_sms);
// One fused pass over S per GNMF W step (fb_gnmf.cu): th = T·H, the W update in place,
// SᵀW, WᵀW and the K_qᵀW bins of the updated W.
struct NmfPass {
  const double* s;  // n × d (d <= 32)
  int64_t n;
  int d;
  double* w;          // n × r, updated in place
  int r;              // <= 16
  const double* h;    // H[0:d, :] (d × r)
  const double* cph;  // HᵀH, r × r
  double eps;
  int nfk;            // >= 1
  const int32_t* fk[kMaxParts];
  const double* z[kMaxParts];  // R_q·H_q, n_R,q × zst
  size_t ztable_bytes[kMaxParts];
  int zst;
  double* bins[kMaxParts];     // n_R,q × r, zeroed by the caller
  const int16_t* hot_slot[kMaxParts];
  const int32_t* hot_key[kMaxParts];
  int nhot[kMaxParts];         // <= 64
  double* partials;            // nmf_pass_partials_doubles
  double* ttw_s;               // SᵀW (d × r)
  double* cpw;                 // WᵀW (r × r)
};
bool nmf_pass_supported(int d_s, int r, int nfk);
size_t nmf_pass_partials_doubles(int num_sms);
cudaError_t launch_nmf_wpass(const NmfPass& p, cudaStream_t st, int num_sms);
// out(c, j) = Σ_r R[r, c]·H[r, j], H int32 n × nx (d_r <= 64, nx <= 16), FP64 tensor cores
bool rth_supported(int d_r, int nx);
size_t rth_partials_doubles(int num_sms);
cudaError_t launch_rth(const double* r, int64_t n, int d_r, const int32_t* h, int nx, double* out, int64_t o_rs,
                       int64_t o_cs, double* partials, unsigned* counter, cudaStream_t st, int num_sms);
// same, f64 weights
cudaError_t launch_rth(const double* r, int64_t n, int d_r, const double* h, int nx, double* out, int64_t o_rs,
                       int64_t o_cs, double* partials, unsigned* counter, cudaStream_t st, int num_sms);
size_t onehot_partials_doubles(int d, int k, int num_sms);
cudaError_t launch_onehot_colsum(const double* s, int64_t n, int d, const int32_t* assign, int k, double* partials,
                                 unsigned* counter, double* out, cudaStream_t st, int num_sms);
cudaError_t launch_kmeans_update(double* c, const double* tta, const int32_t* sizes, int d, int k, double* cc,
                                 cudaStream_t st);
cudaError_t launch_nmf_update(double* f, const double* num, const double* g, int64_t rows, int r, double eps,
                              cudaStream_t st, int num_sms);
cudaError_t launch_small_gram(const double* f, int64_t rows, int r, double* g, cudaStream_t st);
cudaError_t launch_nmf_objective(const double* sum_t2, const double* ttw, const double* h, int64_t dr,
                                 const double* cpw, const double* cph, int rr, double* trace, int it,
                                 cudaStream_t st);

// fb_dense.cu -----------------------------------------------------------------------
cudaError_t launch_dense_mm(int64_t m, int64_t n, int64_t k, const double* a, int64_t lda, int ta, const double* b,
                            int64_t ldb, int tb, double* c, int64_t ldc, int accumulate, cudaStream_t st);
cudaError_t launch_gather2_add(int64_t m, int64_t n, const double* mat, int64_t ldm, const int32_t* ra,
                               const int32_t* cb, double* c, int64_t ldc, cudaStream_t st, int num_sms);
cudaError_t launch_scatter_rows(int64_t n, int d, const int32_t* tgt, const double* a, int64_t lda, double* out,
                                int64_t out_rows, cudaStream_t st, int num_sms);
size_t pair_counts_workspace_bytes(int64_t n);
cudaError_t launch_pair_counts(int64_t n, const int32_t* ta, const int32_t* tb, int64_t rows_a, int64_t cols_b,
                               int64_t* indptr, int64_t* col, double* val, int64_t* nnz, void* ws, size_t ws_bytes,
                               cudaStream_t st, int num_sms);
cudaError_t launch_csr_spmm(int64_t rows, const int64_t* indptr, const void* col, int col_is64, const double* val,
                            const double* x, int64_t ldx, int k, double* y, int64_t ldy, int accumulate,
                            cudaStream_t st, int num_sms);
cudaError_t launch_csr_spmm_t(int64_t rows, int64_t cols, const int64_t* indptr, const void* col, int col_is64,
                              const double* val, const double* x, int64_t ldx, int k, double* y, int64_t ldy,
                              cudaStream_t st, int num_sms);

}  // namespace fb
