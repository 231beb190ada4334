// fb_capi.cu — extern "C" entry points declared in include/factorla_b200.h.
//
// Validation (shapes, nulls, supported sizes) happens here, before any launch, and
// failures come back as FB_ERR_* codes with a thread-local message; the Python layer
// maps them onto the reference's exception classes (exceptions.py).
#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "factorla_b200.h"
#include "fb_kernels.cuh"

namespace fb {
static std::atomic<unsigned long long> g_launches{0};
static int g_debug_sync = -1;
void count_launch(const char* file, int line) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (g_debug_sync < 0) {
    const char* e = getenv("FB_DEBUG_SYNC");
    g_debug_sync = (e && e[0] == '1') ? 1 : 0;
  }
  if (g_debug_sync) {
    cudaError_t err = cudaDeviceSynchronize();
    if (err == cudaSuccess) err = cudaGetLastError();
    if (err != cudaSuccess) fprintf(stderr, "[fb] kernel launched at %s:%d failed: %s\n", file, line, cudaGetErrorString(err));
  }
}
namespace {
// Fork/join onto a library-owned side stream so independent passes of one operator overlap
// (stream-ordered and CUDA-graph capturable: record → wait → launch → record → wait).
struct SideStream {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  int device = -1;
};
constexpr int kMaxDevices = 64;
// one side stream (+ its fork/join events) per (thread, device): switching devices neither
// recreates nor leaks them
thread_local SideStream g_side[kMaxDevices];

SideStream* side_for_current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return (dev >= 0 && dev < kMaxDevices) ? &g_side[dev] : nullptr;
}
}  // namespace


cudaError_t side_fork(cudaStream_t main, cudaStream_t* side) {
  SideStream* ss = side_for_current_device();
  if (!ss) return cudaErrorInvalidDevice;
  if (ss->side == nullptr) {
    cudaError_t e = cudaStreamCreateWithFlags(&ss->side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ss->fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ss->join, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = cudaEventRecord(ss->fork, main);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(ss->side, ss->fork, 0);
  *side = ss->side;
  return e;
}

cudaError_t side_join(cudaStream_t main) {
  SideStream* ss = side_for_current_device();
  if (!ss || !ss->side) return cudaErrorInvalidResourceHandle;
  cudaError_t e = cudaEventRecord(ss->join, ss->side);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(main, ss->join, 0);
  return e;
}

}  // namespace fb

namespace {

thread_local char g_err[512] = "";
// SM count per device (fb_init fills it; 148 = B200 until then), read for the current device
std::atomic<int> g_sms[64];

int current_num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  const int v = (dev >= 0 && dev < 64) ? g_sms[dev].load(std::memory_order_relaxed) : 0;
  return v > 0 ? v : 148;
}
#define g_num_sms current_num_sms()

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return FB_OK;
  if (e == cudaErrorNotSupported) return fail(FB_ERR_ARG, "%s: unsupported size", what);
  return fail(FB_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

inline cudaStream_t cs(fb_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// Carves a caller workspace; returns nullptr when it runs out.
struct Carver {
  char* p;
  size_t left;
  template <class T>
  T* take(size_t count) {
    size_t b = align256(count * sizeof(T));
    if (b > left) return nullptr;
    T* r = reinterpret_cast<T*>(p);
    p += b;
    left -= b;
    return r;
  }
};

int check_nm(const fb_normalized* nm) {
  if (!nm) return fail(FB_ERR_ARG, "normalized matrix is NULL");
  if (nm->q < 0 || nm->q > FB_MAX_PARTS)
    return fail(FB_ERR_ARG, "q=%d attribute blocks outside [0, %d]", nm->q, FB_MAX_PARTS);
  if (nm->n_s < 0 || nm->d_s < 0) return fail(FB_ERR_SHAPE, "negative entity shape");
  if (nm->d_s > 0 && !nm->s && nm->n_s > 0) return fail(FB_ERR_ARG, "S is NULL");
  for (int i = 0; i < nm->q; ++i) {
    const fb_part& p = nm->part[i];
    if (p.n_r < 1 || p.d_r < 0) return fail(FB_ERR_SHAPE, "part %d: bad shape %lldx%d", i, (long long)p.n_r, p.d_r);
    if ((!p.fk && nm->n_s > 0) || (!p.r && p.d_r > 0)) return fail(FB_ERR_ARG, "part %d: NULL pointer", i);
  }
  return FB_OK;
}

int64_t total_cols(const fb_normalized* nm) {
  int64_t d = nm->d_s;
  for (int i = 0; i < nm->q; ++i) d += nm->part[i].d_r;
  return d;
}

int64_t max_width(const fb_normalized* nm) {
  int64_t d = nm->d_s;
  for (int i = 0; i < nm->q; ++i) d = nm->part[i].d_r > d ? nm->part[i].d_r : d;
  return d;
}

// Column chunk widths the templated kernels are instantiated for.
int chunk_width(int rem) {
  if (rem >= 16) return 16;
  static const int ok[] = {12, 10, 8, 7, 6, 5, 4, 3, 2, 1};
  if (rem == 16 || rem == 12 || rem == 10 || rem <= 8) return rem;
  for (int w : ok)
    if (w <= rem) return w;
  return 1;
}

__global__ void fill_kernel(double* p, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void band_id_kernel(const int32_t* fk, int64_t n, int64_t n_r, int64_t n_bands, int32_t* band) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    band[i] = static_cast<int32_t>(static_cast<int64_t>(fk[i]) * n_bands / n_r);
}

__global__ void gather_i32_kernel(const int32_t* in, const int32_t* idx, int64_t n, int32_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[idx[i]];
}

__global__ void scatter_i32_kernel(const int32_t* in, const int32_t* idx, int64_t n, int32_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[idx[i]] = in[i];
}

__global__ void mirror_upper_kernel(double* a, int64_t d) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e >= d * d) return;
  const int64_t r = e / d, c = e % d;
  if (r > c) a[e] = a[c * d + r];
}

__global__ void sum_vector_kernel(const double* v, int64_t n, double* out) {
  // single warp, fixed order per lane then a fixed shuffle tree: deterministic
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 32) s += v[i];
  s = fb::warp_sum(s);
  if (threadIdx.x == 0) *out = s;
}

}  // namespace

extern "C" {

int fb_abi_version(void) { return FB_ABI_VERSION; }
const char* fb_last_error(void) { return g_err; }
uint64_t fb_launch_count(void) { return fb::g_launches.load(); }

int fb_init(int device) {
  // caches the device's SM count; the caller's current device is left as it was
  if (device < 0 || device >= 64) return fail(FB_ERR_ARG, "fb_init: device %d out of range", device);
  int sms = 0;
  cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return cuda_status(e, "cudaDeviceGetAttribute");
  g_sms[device].store(sms, std::memory_order_relaxed);
  return FB_OK;
}

// ------------------------------------------------------------------ construction
int fb_key_check(const int64_t* key, int64_t n, int64_t n_r, int32_t* counts_full,
                 unsigned long long* first_bad, fb_stream_t stream) {
  if (n < 0 || n_r < 1) return fail(FB_ERR_SHAPE, "key_check: n=%lld n_r=%lld", (long long)n, (long long)n_r);
  if ((n > 0 && !key) || !counts_full || !first_bad) return fail(FB_ERR_ARG, "key_check: NULL pointer");
  return cuda_status(fb::launch_key_check_hist(key, n, n_r, counts_full, first_bad, cs(stream), g_num_sms),
                     "key_check");
}

size_t fb_key_remap_workspace_bytes(int64_t n_r) {
  return align256(fb::used_scan_ws_ints(n_r) * sizeof(int32_t)) + 256;
}

int fb_key_remap(const int64_t* key, int64_t n, int64_t n_r, const int32_t* counts_full,
                 int32_t* lookup, int32_t* n_used, int32_t* target, int64_t* used_idx,
                 int32_t* counts_kept, void* ws, size_t ws_bytes, fb_stream_t stream) {
  if (ws_bytes < fb_key_remap_workspace_bytes(n_r) || !ws) return fail(FB_ERR_ARG, "key_remap: workspace too small");
  cudaError_t e = fb::launch_used_scan(counts_full, n_r, lookup, n_used, static_cast<int32_t*>(ws), cs(stream), g_num_sms);
  if (e != cudaSuccess) return cuda_status(e, "used_scan");
  return cuda_status(fb::launch_remap(key, n, lookup, counts_full, n_r, target, used_idx, counts_kept, cs(stream), g_num_sms),
                     "remap");
}

int fb_fk_counts(const int32_t* fk, int64_t n, int32_t* counts, int64_t n_r, fb_stream_t stream) {
  if ((n > 0 && !fk) || !counts) return fail(FB_ERR_ARG, "fk_counts: NULL pointer");
  return cuda_status(fb::launch_fk_hist(fk, n, counts, n_r, cs(stream), g_num_sms), "fk_counts");
}

int fb_gather_rows(const double* in, int64_t ld_in, const int64_t* idx, int64_t nrows, int32_t d,
                   double* out, int64_t ld_out, fb_stream_t stream) {
  return cuda_status(fb::launch_gather_rows(in, ld_in, idx, nullptr, nrows, d, out, ld_out, cs(stream), g_num_sms),
                     "gather_rows");
}

int fb_gather_rows_i32(const double* in, int64_t ld_in, const int32_t* idx, int64_t nrows, int32_t d,
                       double* out, int64_t ld_out, fb_stream_t stream) {
  return cuda_status(fb::launch_gather_rows(in, ld_in, nullptr, idx, nrows, d, out, ld_out, cs(stream), g_num_sms),
                     "gather_rows_i32");
}

int fb_i32_to_f64(const int32_t* in, double* out, int64_t n, fb_stream_t stream) {
  return cuda_status(fb::launch_i32_to_f64(in, out, n, cs(stream), g_num_sms), "i32_to_f64");
}

int fb_csr_expand(const int64_t* indptr, const int32_t* indices, const double* data, int64_t nrows,
                  int32_t ncols, double* out, int64_t ld_out, fb_stream_t stream) {
  if (nrows < 0 || ncols < 0 || ld_out < ncols) return fail(FB_ERR_SHAPE, "csr_expand: bad shape");
  return cuda_status(fb::launch_csr_expand(indptr, indices, data, nrows, ncols, out, ld_out, cs(stream), g_num_sms),
                     "csr_expand");
}

// ------------------------------------------------------------------ LMM / rowSums
size_t fb_lmm_workspace_bytes(const fb_normalized* nm, int32_t d_x) {
  if (!nm) return 0;
  int w = d_x < 16 ? d_x : 16;
  size_t b = 0;
  for (int i = 0; i < nm->q; ++i)
    b += align256(static_cast<size_t>(nm->part[i].n_r) * fb::z_stride(w) * sizeof(double));
  return b + 256;
}

int fb_lmm(const fb_normalized* nm, const double* x, int32_t d_x, double* out, void* ws,
           size_t ws_bytes, fb_stream_t stream) {
  int st = check_nm(nm);
  if (st) return st;
  if (d_x < 1) return fail(FB_ERR_SHAPE, "lmm: d_x=%d", d_x);
  if (!x || (!out && nm->n_s > 0)) return fail(FB_ERR_ARG, "lmm: NULL pointer");
  if (ws_bytes < fb_lmm_workspace_bytes(nm, d_x)) return fail(FB_ERR_ARG, "lmm: workspace too small");
  if (max_width(nm) > 256) return fail(FB_ERR_ARG, "lmm: factor widths above 256 are not supported");
  for (int c0 = 0; c0 < d_x;) {
    const int w = chunk_width(d_x - c0);
    Carver cv{static_cast<char*>(ws), ws_bytes};
    const int32_t* fks[FB_MAX_PARTS];
    const double* zs[FB_MAX_PARTS];
    int64_t zrows[FB_MAX_PARTS];
    int64_t off = nm->d_s;
    for (int i = 0; i < nm->q; ++i) {
      const fb_part& p = nm->part[i];
      const int zst = fb::z_stride(w);
      double* z = cv.take<double>(static_cast<size_t>(p.n_r) * zst);
      // z_i = R_i · X[off:off+d_r, c0:c0+w]   (rewrite.py:187)
      cudaError_t e = fb::launch_lmm_rows(p.r, p.n_r, p.d_r, x + off * d_x + c0, w, d_x, 0, nullptr,
                                          nullptr, 0, z, zst, cs(stream), g_num_sms);
      if (e != cudaSuccess) return cuda_status(e, "lmm(z)");
      fks[i] = p.fk;
      zs[i] = z;
      zrows[i] = p.n_r;
      off += p.d_r;
    }
    // out = S · X[0:d_s, c0:c0+w] + Σ z_i[fk_i]   (rewrite.py:186-190)
    cudaError_t e = fb::launch_lmm_rows(nm->s, nm->n_s, nm->d_s, x + c0, w, d_x, nm->q, fks, zs,
                                        fb::z_stride(w), out + c0, d_x, cs(stream), g_num_sms, zrows);
    if (e != cudaSuccess) return cuda_status(e, "lmm(S)");
    c0 += w;
  }
  return FB_OK;
}

// ------------------------------------------------------------------ FK-band layout
size_t fb_band_build_workspace_bytes(int64_t n) {
  return fb::fk_sort_workspace_bytes(n) + 2 * align256(static_cast<size_t>(n > 0 ? n : 1) * 4) + 256;
}

int64_t fb_band_fk_stride(int64_t n) { return (n + 63) & ~int64_t(63); }

int fb_band_build(const fb_normalized* nm, int32_t n_bands, int32_t* perm, int32_t* fk_band, double* s_band,
                  void* ws, size_t ws_bytes, fb_stream_t stream) {
  int st = check_nm(nm);
  if (st) return st;
  if (nm->q < 1) return fail(FB_ERR_ARG, "band_build: needs an attribute table (q=%d)", nm->q);
  if (n_bands < 1 || n_bands > 4096) return fail(FB_ERR_ARG, "band_build: n_bands=%d outside [1, 4096]", n_bands);
  const int64_t n = nm->n_s;
  if (n == 0) return FB_OK;
  if (!perm || !fk_band || (!s_band && nm->d_s > 0) || !ws) return fail(FB_ERR_ARG, "band_build: NULL pointer");
  if (ws_bytes < fb_band_build_workspace_bytes(n)) return fail(FB_ERR_ARG, "band_build: workspace too small");
  const fb_part& p = nm->part[0];
  const size_t ib = align256(static_cast<size_t>(n) * 4);
  int32_t* band = static_cast<int32_t*>(ws);
  int32_t* band_sorted = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + ib);
  void* sort_ws = static_cast<char*>(ws) + 2 * ib;
  band_id_kernel<<<g_num_sms * 8, 256, 0, cs(stream)>>>(p.fk, n, p.n_r, n_bands, band);
  FB_LAUNCHED();
  // stable sort by band: storage order survives inside a band
  cudaError_t e = fb::launch_fk_sort(band, n, n_bands, perm, band_sorted, sort_ws, ws_bytes - 2 * ib, cs(stream),
                                     g_num_sms);
  if (e != cudaSuccess) return cuda_status(e, "band_build(sort)");
  for (int q = 0; q < nm->q; ++q) {
    gather_i32_kernel<<<g_num_sms * 8, 256, 0, cs(stream)>>>(nm->part[q].fk, perm, n, fk_band + q * fb_band_fk_stride(n));
    FB_LAUNCHED();
  }
  if (nm->d_s > 0) {
    e = fb::launch_gather_rows(nm->s, nm->d_s, nullptr, perm, n, nm->d_s, s_band, nm->d_s, cs(stream), g_num_sms);
    if (e != cudaSuccess) return cuda_status(e, "band_build(gather)");
  }
  return cuda_status(cudaGetLastError(), "band_build");
}

int fb_scatter_i32(const int32_t* in, const int32_t* perm, int64_t n, int32_t* out, fb_stream_t stream) {
  if (n < 0 || (n > 0 && (!in || !perm || !out))) return fail(FB_ERR_ARG, "scatter_i32: bad argument");
  if (n == 0) return FB_OK;
  scatter_i32_kernel<<<g_num_sms * 8, 256, 0, cs(stream)>>>(in, perm, n, out);
  FB_LAUNCHED();
  return cuda_status(cudaGetLastError(), "scatter_i32");
}

int fb_lmm_banded(const fb_normalized* nm, const fb_band_layout* band, const double* x, int32_t d_x, double* out,
                  void* ws, size_t ws_bytes, fb_stream_t stream) {
  int st = check_nm(nm);
  if (st) return st;
  if (!band || nm->q != 1 || nm->d_s < 1 || nm->d_s > 32 || nm->n_s == 0 || !band->perm || !band->fk[0] || !band->s)
    return fb_lmm(nm, x, d_x, out, ws, ws_bytes, stream);
  if (d_x < 1) return fail(FB_ERR_SHAPE, "lmm: d_x=%d", d_x);
  if (!x || !out) return fail(FB_ERR_ARG, "lmm: NULL pointer");
  if (ws_bytes < fb_lmm_workspace_bytes(nm, d_x)) return fail(FB_ERR_ARG, "lmm: workspace too small");
  if (max_width(nm) > 256) return fail(FB_ERR_ARG, "lmm: factor widths above 256 are not supported");
  const fb_part& p = nm->part[0];
  for (int c0 = 0; c0 < d_x;) {
    const int w = chunk_width(d_x - c0);
    const int zst = fb::z_stride(w);
    Carver cv{static_cast<char*>(ws), ws_bytes};
    double* z = cv.take<double>(static_cast<size_t>(p.n_r) * zst);
    // z = R · X[d_s:, c0:c0+w]   (rewrite.py:187)
    cudaError_t e = fb::launch_lmm_rows(p.r, p.n_r, p.d_r, x + static_cast<int64_t>(nm->d_s) * d_x + c0, w, d_x, 0,
                                        nullptr, nullptr, 0, z, zst, cs(stream), g_num_sms);
    if (e != cudaSuccess) return cuda_status(e, "lmm(z)");
    // out = S · X[0:d_s, c0:c0+w] + z[fk]   (rewrite.py:186-190), rows visited band by band
    if (fb::lmm_band_supported(nm->d_s, w, d_x, out + c0)) {
      e = fb::launch_lmm_band(band->s, band->fk[0], band->perm, nm->n_s, nm->d_s, x + c0, w, d_x, z, zst, p.n_r,
                              out + c0, d_x, cs(stream), g_num_sms);
    } else {
      const int32_t* fks[1] = {p.fk};
      const double* zs[1] = {z};
      const int64_t zrows[1] = {p.n_r};
      e = fb::launch_lmm_rows(nm->s, nm->n_s, nm->d_s, x + c0, w, d_x, 1, fks, zs, zst, out + c0, d_x, cs(stream),
                              g_num_sms, zrows);
    }
    if (e != cudaSuccess) return cuda_status(e, "lmm(S, banded)");
    c0 += w;
  }
  return FB_OK;
}

size_t fb_row_sums_workspace_bytes(const fb_normalized* nm) {
  if (!nm) return 0;
  return fb_lmm_workspace_bytes(nm, 1) + align256(static_cast<size_t>(total_cols(nm) + 1) * sizeof(double));
}

int fb_row_sums(const fb_normalized* nm, double* out, void* ws, size_t ws_bytes, fb_stream_t stream) {
  int st = check_nm(nm);
  if (st) return st;
  if (ws_bytes < fb_row_sums_workspace_bytes(nm)) return fail(FB_ERR_ARG, "row_sums: workspace too small");
  const int64_t d = total_cols(nm);
  double* ones = static_cast<double*>(ws);
  const size_t ob = align256(static_cast<size_t>(d + 1) * sizeof(double));
  fill_kernel<<<1, 256, 0, cs(stream)>>>(ones, d + 1, 1.0);
  FB_LAUNCHED();
  // rowSums(T) = S·1 + Σ K_i·(R_i·1): the LMM pass with X = ones (kernel.py:174-182)
  return fb_lmm(nm, ones, 1, out, static_cast<char*>(ws) + ob, ws_bytes - ob, stream);
}

// ------------------------------------------------------------------ Wᵀ·T family
size_t fb_wt_workspace_bytes(const fb_normalized* nm, int32_t n_w) {
  if (!nm) return 0;
  const int w = n_w < 16 ? n_w : 16;
  size_t b = 0;
  for (int i = 0; i < nm->q; ++i) b += align256(static_cast<size_t>(nm->part[i].n_r) * w * sizeof(double));
  b += align256(fb::colreduce_workspace_doubles(0, static_cast<int>(max_width(nm)), w, g_num_sms) * sizeof(double));
  b += 256;  // counter
  return b;
}

// X·K for a uniform FK: one RED per row fused into the S pass (the bins — n_R·n_x doubles, 8 MB at
// c2 — stay L2-resident, and the weights are read in storage order with the S tiles). Skewed FKs
// (a hot target holding > 1/256 of the rows) take the segmented sums over the cached FK-sorted
// order instead. FB_WT_SCATTER=seg|atomic overrides the choice (measurement only).
static bool use_segsum(const fb_part& pt) {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("FB_WT_SCATTER");
    mode = (e && e[0] == 's') ? 1 : (e && e[0] == 'a') ? 2 : 0;
  }
  if (mode == 1) return true;
  if (mode == 2) return false;
  return pt.skewed != 0;
}

static int wt_impl(const fb_normalized* nm, const double* w, int32_t n_w, int64_t w_rs, int64_t w_cs,
                   const double* const* part_weights, double* out, int64_t o_js, int64_t o_cs, void* ws,
                   size_t ws_bytes, fb_stream_t stream, double* const* bins_out = nullptr, bool r_pass = true) {
  // part_weights != nullptr: colSums mode — S pass with implicit ones, R_i pass with counts_i.
  // bins_out (n_w <= 16): the X·K bins go to the caller's buffers; r_pass = false stops after
  // the S pass (the R-row-sliced multi-GPU composition runs the R passes itself).
  for (int j0 = 0; j0 < n_w;) {
    const int nx = chunk_width(n_w - j0);
    Carver cv{static_cast<char*>(ws), ws_bytes};
    double* bins[FB_MAX_PARTS] = {};
    if (!part_weights)
      for (int i = 0; i < nm->q; ++i)
        bins[i] = bins_out ? bins_out[i] : cv.take<double>(static_cast<size_t>(nm->part[i].n_r) * nx);
    double* partials = cv.take<double>(fb::colreduce_workspace_doubles(0, static_cast<int>(max_width(nm)), nx, g_num_sms));
    unsigned int* counter = cv.take<unsigned int>(1);
    if (!partials || !counter) return fail(FB_ERR_ARG, "wt: workspace too small");

    bool forked = false;
    cudaStream_t side = nullptr;
    fb::ColReduce c{};
    c.a = nm->s;
    c.n = nm->n_s;
    c.d = nm->d_s;
    c.nx = nx;
    c.w = w ? w + j0 * w_cs : nullptr;
    c.w_rs = w_rs;
    c.w_cs = w_cs;
    c.nfk = 0;
    for (int i = 0; !part_weights && i < nm->q; ++i) {
      const fb_part& pt = nm->part[i];
      if (!bins[i]) continue;  // no scatter wanted for this part
      if (pt.perm && pt.fk_sorted && nm->n_s > 0 && use_segsum(pt)) {
        // X·K_i as segmented sums over the FK-sorted order (few atomics, no hot-line
        // contention), on the side stream so they overlap the S pass
        if (!forked) {
          cudaError_t e = fb::side_fork(cs(stream), &side);
          if (e != cudaSuccess) return cuda_status(e, "wt(fork)");
          forked = true;
        }
        cudaError_t e = fb::launch_segsum(pt.perm, pt.fk_sorted, nm->n_s, w + j0 * w_cs, w_rs, w_cs, nx, bins[i],
                                          pt.n_r, side, g_num_sms);
        if (e != cudaSuccess) return cuda_status(e, "wt(segsum)");
        continue;
      }
      const int f = c.nfk++;  // fused into the S pass: one atomic per row
      c.fk[f] = pt.fk;
      c.bins[f] = bins[i];
      c.nbins[f] = pt.n_r;
      c.aggregate[f] = pt.skewed;
      if (pt.nhot > 0 && pt.hot_slot && pt.hot_key) {
        c.nhot[f] = pt.nhot < 64 ? pt.nhot : 64;
        c.hot_slot[f] = pt.hot_slot;
        c.hot_key[f] = pt.hot_key;
      }
    }
    c.out = out + j0 * o_js;
    c.o_js = o_js;
    c.o_cs = o_cs;
    c.partials = partials;
    c.counter = counter;
    cudaError_t e = fb::launch_colreduce(c, cs(stream), g_num_sms);
    if (e != cudaSuccess) return cuda_status(e, "wt(S)");
    if (forked) {
      e = fb::side_join(cs(stream));  // the R passes below read the segmented bins
      if (e != cudaSuccess) return cuda_status(e, "wt(join)");
    }
    int64_t off = nm->d_s;
    for (int i = 0; r_pass && i < nm->q; ++i) {
      const fb_part& p = nm->part[i];
      fb::ColReduce r{};
      r.a = p.r;
      r.n = p.n_r;
      r.d = p.d_r;
      r.nx = nx;
      r.w = part_weights ? part_weights[i] : bins[i];
      r.w_rs = nx;
      r.w_cs = 1;
      r.nfk = 0;
      r.out = out + j0 * o_js + off * o_cs;
      r.o_js = o_js;
      r.o_cs = o_cs;
      r.partials = partials;
      r.counter = counter;
      e = fb::launch_colreduce(r, cs(stream), g_num_sms);
      if (e != cudaSuccess) return cuda_status(e, "wt(R)");
      off += p.d_r;
    }
    j0 += nx;
  }
  return FB_OK;
}

int fb_wt(const fb_normalized* nm, const double* w, int32_t n_w, int64_t w_rs, int64_t w_cs, double* out,
          int64_t o_js, int64_t o_cs, void* ws, size_t ws_bytes, fb_stream_t stream) {
  int st = check_nm(nm);
  if (st) return st;
  if (n_w < 1) return fail(FB_ERR_SHAPE, "wt: n_w=%d", n_w);
  if ((!w && nm->n_s > 0) || !out) return fail(FB_ERR_ARG, "wt: NULL pointer");
  if (max_width(nm) > 256) return fail(FB_ERR_ARG, "wt: factor widths above 256 are not supported");
  if (ws_bytes < fb_wt_workspace_bytes(nm, n_w)) return fail(FB_ERR_ARG, "wt: workspace too small");
  return wt_impl(nm, w, n_w, w_rs, w_cs, nullptr, out, o_js, o_cs, ws, ws_bytes, stream);
}

size_t fb_col_sums_workspace_bytes(const fb_normalized* nm) {
  if (!nm) return 0;
  size_t b = fb_wt_workspace_bytes(nm, 1);
  for (int i = 0; i < nm->q; ++i) b += align256(static_cast<size_t>(nm->part[i].n_r) * sizeof(double));
  return b + align256(static_cast<size_t>(total_cols(nm)) * sizeof(double));
}

int fb_col_sums(const fb_normalized* nm, double* out, void* ws, size_t ws_bytes, fb_stream_t stream) {
  int st = check_nm(nm);
  if (st) return st;
  if (max_width(nm) > 256) return fail(FB_ERR_ARG, "col_sums: factor widths above 256 are not supported");
  if (ws_bytes < fb_col_sums_workspace_bytes(nm)) return fail(FB_ERR_ARG, "col_sums: workspace too small");
  // colSums(T) = [1ᵀS, colSums(K_i)·R_i]  (rewrite.py:131-149); counts are cached per
  // indicator (indicator.py:61-66) — derive them here only when the caller has none.
  Carver cv{static_cast<char*>(ws), ws_bytes};
  const double* cnt[FB_MAX_PARTS] = {};
  for (int i = 0; i < nm->q; ++i) {
    const fb_part& p = nm->part[i];
    if (p.counts) {
      cnt[i] = p.counts;
    } else {
      double* c = cv.take<double>(static_cast<size_t>(p.n_r));
      int32_t* ci = reinterpret_cast<int32_t*>(cv.take<double>(static_cast<size_t>(p.n_r)));
      cudaError_t e = fb::launch_fk_hist(p.fk, nm->n_s, ci, p.n_r, cs(stream), g_num_sms);
      if (e == cudaSuccess) e = fb::launch_i32_to_f64(ci, c, p.n_r, cs(stream), g_num_sms);
      if (e != cudaSuccess) return cuda_status(e, "col_sums(counts)");
      cnt[i] = c;
    }
  }
  return wt_impl(nm, nullptr, 1, 1, 1, cnt, out, 0, 1, cv.p, cv.left, stream);
}

int fb_sum_all(const fb_normalized* nm, double* out, void* ws, size_t ws_bytes, fb_stream_t stream) {
  int st = check_nm(nm);
  if (st) return st;
  const int64_t d = total_cols(nm);
  const size_t vb = align256(static_cast<size_t>(d > 0 ? d : 1) * sizeof(double));
  if (ws_bytes < vb + fb_col_sums_workspace_bytes(nm)) return fail(FB_ERR_ARG, "sum_all: workspace too small");
  double* v = static_cast<double*>(ws);
  // sum(T) = sum(S) + colSums(K)·rowSums(R) (rewrite.py:152-165) = Σ_c colSums(T)_c
  st = fb_col_sums(nm, v, static_cast<char*>(ws) + vb, ws_bytes - vb, stream);
  if (st) return st;
  sum_vector_kernel<<<1, 32, 0, cs(stream)>>>(v, d, out);
  FB_LAUNCHED();
  return cuda_status(cudaGetLastError(), "sum_all");
}

// ------------------------------------------------------------------ split passes (multi-GPU)
int fb_z_stride(int32_t d_x) { return d_x >= 1 && d_x <= 16 ? fb::z_stride(d_x) : 0; }

int fb_lmm_zpass(const fb_normalized* nm, const double* x, int32_t d_x, int32_t part, int64_t row_lo, int64_t row_hi,
                 double* z, fb_stream_t stream) {
  int st = check_nm(nm);
  if (st) return st;
  if (d_x < 1 || d_x > 16) return fail(FB_ERR_ARG, "lmm_zpass: d_x=%d outside [1, 16]", d_x);
  if (part < 0 || part >= nm->q) return fail(FB_ERR_ARG, "lmm_zpass: part %d of %d", part, nm->q);
  const fb_part& p = nm->part[part];
  if (row_lo < 0 || row_hi > p.n_r || row_lo > row_hi) return fail(FB_ERR_SHAPE, "lmm_zpass: rows [%lld, %lld) of %lld",
                                                                  (long long)row_lo, (long long)row_hi, (long long)p.n_r);
  if (!x || !z) return fail(FB_ERR_ARG, "lmm_zpass: NULL pointer");
  if (max_width(nm) > 256) return fail(FB_ERR_ARG, "lmm_zpass: factor widths above 256 are not supported");
  int64_t off = nm->d_s;
  for (int i = 0; i < part; ++i) off += nm->part[i].d_r;
  const int zst = fb::z_stride(d_x);
  return cuda_status(fb::launch_lmm_rows(p.r + row_lo * p.d_r, row_hi - row_lo, p.d_r, x + off * d_x, d_x, d_x, 0,
                                         nullptr, nullptr, 0, z + row_lo * zst, zst, cs(stream), g_num_sms),
                     "lmm_zpass");
}

int fb_lmm_spass(const fb_normalized* nm, const double* x, int32_t d_x, const double* const* z, double* out,
                 fb_stream_t stream) {
  int st = check_nm(nm);
  if (st) return st;
  if (d_x < 1 || d_x > 16) return fail(FB_ERR_ARG, "lmm_spass: d_x=%d outside [1, 16]", d_x);
  if (!x || (!out && nm->n_s > 0) || (nm->q > 0 && !z)) return fail(FB_ERR_ARG, "lmm_spass: NULL pointer");
  if (max_width(nm) > 256) return fail(FB_ERR_ARG, "lmm_spass: factor widths above 256 are not supported");
  const int32_t* fks[FB_MAX_PARTS];
  const double* zs[FB_MAX_PARTS];
  int64_t zrows[FB_MAX_PARTS];
  for (int i = 0; i < nm->q; ++i) {
    if (!z[i]) return fail(FB_ERR_ARG, "lmm_spass: z[%d] is NULL", i);
    fks[i] = nm->part[i].fk;
    zs[i] = z[i];
    zrows[i] = nm->part[i].n_r;
  }
  return cuda_status(fb::launch_lmm_rows(nm->s, nm->n_s, nm->d_s, x, d_x, d_x, nm->q, fks, zs, fb::z_stride(d_x), out,
                                         d_x, cs(stream), g_num_sms, zrows),
                     "lmm_spass");
}

size_t fb_wt_spass_workspace_bytes(const fb_normalized* nm, int32_t n_w) {
  if (!nm) return 0;
  const int w = n_w < 16 ? n_w : 16;
  return align256(fb::colreduce_workspace_doubles(0, static_cast<int>(max_width(nm)), w, g_num_sms) * sizeof(double)) +
         256;
}

int fb_wt_spass(const fb_normalized* nm, const double* w, int32_t n_w, int64_t w_rs, int64_t w_cs, double* out,
                int64_t o_js, int64_t o_cs, double* const* bins, void* ws, size_t ws_bytes, fb_stream_t stream) {
  int st = check_nm(nm);
  if (st) return st;
  if (n_w < 1 || n_w > 16) return fail(FB_ERR_ARG, "wt_spass: n_w=%d outside [1, 16]", n_w);
  if (!out) return fail(FB_ERR_ARG, "wt_spass: NULL output");
  if (!w && bins) return fail(FB_ERR_ARG, "wt_spass: the X·K scatter needs explicit weights");
  if (max_width(nm) > 256) return fail(FB_ERR_ARG, "wt_spass: factor widths above 256 are not supported");
  if (ws_bytes < fb_wt_spass_workspace_bytes(nm, n_w)) return fail(FB_ERR_ARG, "wt_spass: workspace too small");
  double* none[FB_MAX_PARTS] = {};
  if (!w) {  // all-ones weights: colSums of S
    fb_normalized s_only = *nm;
    s_only.q = 0;
    return wt_impl(&s_only, nullptr, 1, 1, 1, nullptr, out, o_js, o_cs, ws, ws_bytes, stream, none, false);
  }
  return wt_impl(nm, w, n_w, w_rs, w_cs, nullptr, out, o_js, o_cs, ws, ws_bytes, stream, bins ? bins : none, false);
}

size_t fb_rows_wt_workspace_bytes(int32_t d, int32_t n_w) {
  const int w = n_w < 16 ? n_w : 16;
  return align256(fb::colreduce_workspace_doubles(0, d > 0 ? d : 1, w > 0 ? w : 1, g_num_sms) * sizeof(double)) + 256;
}

int fb_rows_wt(const double* a, int64_t n, int32_t d, const double* w, int32_t n_w, int64_t w_rs, int64_t w_cs,
               double* out, int64_t o_js, int64_t o_cs, void* ws, size_t ws_bytes, fb_stream_t stream) {
  if (n < 0 || d < 0 || n_w < 1) return fail(FB_ERR_SHAPE, "rows_wt: n=%lld d=%d n_w=%d", (long long)n, d, n_w);
  if (d > 256) return fail(FB_ERR_ARG, "rows_wt: widths above 256 are not supported");
  if ((n > 0 && (!a || !w)) || !out) return fail(FB_ERR_ARG, "rows_wt: NULL pointer");
  if (ws_bytes < fb_rows_wt_workspace_bytes(d, n_w)) return fail(FB_ERR_ARG, "rows_wt: workspace too small");
  for (int j0 = 0; j0 < n_w;) {
    const int nx = chunk_width(n_w - j0);
    Carver cv{static_cast<char*>(ws), ws_bytes};
    double* partials = cv.take<double>(fb::colreduce_workspace_doubles(0, d > 0 ? d : 1, nx, g_num_sms));
    unsigned int* counter = cv.take<unsigned int>(1);
    fb::ColReduce r{};
    r.a = a;
    r.n = n;
    r.d = d;
    r.nx = nx;
    r.w = w + j0 * w_cs;
    r.w_rs = w_rs;
    r.w_cs = w_cs;
    r.out = out + j0 * o_js;
    r.o_js = o_js;
    r.o_cs = o_cs;
    r.partials = partials;
    r.counter = counter;
    if (n == 0) {
      for (int j = 0; j < nx; ++j) {  // empty slice: zero output (colreduce needs rows)
        cudaError_t e = cudaMemset2DAsync(out + (j0 + j) * o_js, o_cs * sizeof(double), 0, sizeof(double), d, cs(stream));
        if (e != cudaSuccess) return cuda_status(e, "rows_wt(empty)");
      }
    } else {
      cudaError_t e = fb::launch_colreduce(r, cs(stream), g_num_sms);
      if (e != cudaSuccess) return cuda_status(e, "rows_wt");
    }
    j0 += nx;
  }
  return FB_OK;
}

// ------------------------------------------------------------------ crossprod
size_t fb_fk_sort_workspace_bytes(int64_t n) { return fb::fk_sort_workspace_bytes(n); }

int fb_fk_sort(const int32_t* fk, int64_t n, int64_t n_r, int32_t* perm, int32_t* fk_sorted, void* ws,
               size_t ws_bytes, fb_stream_t stream) {
  if (n < 0 || n_r < 1) return fail(FB_ERR_SHAPE, "fk_sort: n=%lld n_r=%lld", (long long)n, (long long)n_r);
  if (n > 0 && (!fk || !perm || !fk_sorted || !ws)) return fail(FB_ERR_ARG, "fk_sort: NULL pointer");
  if (ws_bytes < fb::fk_sort_workspace_bytes(n)) return fail(FB_ERR_ARG, "fk_sort: workspace too small");
  return cuda_status(fb::launch_fk_sort(fk, n, n_r, perm, fk_sorted, ws, ws_bytes, cs(stream), g_num_sms), "fk_sort");
}

size_t fb_crossprod_workspace_bytes(const fb_normalized* nm) {
  if (!nm) return 0;
  const bool q = nm->q > 0;
  return fb::crossprod_workspace_bytes(nm->n_s, nm->d_s, q ? nm->part[0].n_r : 0, q ? nm->part[0].d_r : 0,
                                       q ? 1 : 0, g_num_sms);
}

static int crossprod_impl(const fb_normalized* nm, const int32_t* perm, const int32_t* fk_sorted, double* out, void* ws,
                          size_t ws_bytes, fb_stream_t stream, int mode, double* kts) {
  int st = check_nm(nm);
  if (st) return st;
  if (nm->q > 1) return fail(FB_ERR_ARG, "crossprod: star schemas (q=%d) are not supported by the device path", nm->q);
  if (nm->d_s > 256 || max_width(nm) > 256 || (nm->q == 1 && nm->d_s > 128))
    return fail(FB_ERR_ARG, "crossprod: factor widths above 256 (d_S above 128 with an FK) are not supported");
  if (!out) return fail(FB_ERR_ARG, "crossprod: NULL output");
  if (ws_bytes < fb_crossprod_workspace_bytes(nm)) return fail(FB_ERR_ARG, "crossprod: workspace too small");
  fb::CrossArgs c{};
  c.s = nm->s;
  c.n_s = nm->n_s;
  c.d_s = nm->d_s;
  if (nm->q == 1) {
    const fb_part& p = nm->part[0];
    if (mode != 2 && nm->n_s > 0 && (!perm || !fk_sorted)) return fail(FB_ERR_ARG, "crossprod: FK-sorted order missing");
    if (!p.counts) return fail(FB_ERR_ARG, "crossprod: counts missing");
    c.perm = perm;
    c.fk_sorted = fk_sorted;
    c.r = p.r;
    c.n_r = p.n_r;
    c.d_r = p.d_r;
    c.counts = p.counts;
  }
  c.out = out;
  c.mode = mode;
  c.kts = kts;
  if (mode != 0 && nm->q == 1 && !kts) return fail(FB_ERR_ARG, "crossprod: split passes need the KᵀS buffer");
  return cuda_status(fb::launch_crossprod(c, ws, ws_bytes, cs(stream), g_num_sms), "crossprod");
}

int fb_crossprod(const fb_normalized* nm, const int32_t* perm, const int32_t* fk_sorted, double* out, void* ws,
                 size_t ws_bytes, fb_stream_t stream) {
  return crossprod_impl(nm, perm, fk_sorted, out, ws, ws_bytes, stream, 0, nullptr);
}

int fb_crossprod_spass(const fb_normalized* nm, const int32_t* perm, const int32_t* fk_sorted, double* out,
                       double* kts, void* ws, size_t ws_bytes, fb_stream_t stream) {
  return crossprod_impl(nm, perm, fk_sorted, out, ws, ws_bytes, stream, 1, kts);
}

int fb_crossprod_rpass(const fb_normalized* nm, const double* kts, double* out, void* ws, size_t ws_bytes,
                       fb_stream_t stream) {
  if (nm && nm->q != 1) return fail(FB_ERR_ARG, "crossprod_rpass: needs exactly one attribute block (q=%d)", nm->q);
  return crossprod_impl(nm, nullptr, nullptr, out, ws, ws_bytes, stream, 2, const_cast<double*>(kts));
}

// ------------------------------------------------------------------ GLM steps
size_t fb_glm_workspace_bytes(const fb_normalized* nm) {
  if (!nm) return 0;
  size_t b = 0;
  for (int i = 0; i < nm->q; ++i) b += 3 * align256(static_cast<size_t>(nm->part[i].n_r) * sizeof(double));
  const int64_t d = total_cols(nm);
  b += align256(static_cast<size_t>(d + 1) * sizeof(double));                                 // g
  b += align256(sizeof(double));                                                               // loss
  b += align256(fb::glm_partials_doubles(nm->d_s, g_num_sms) * sizeof(double));                // S partials
  b += align256(fb::colreduce_workspace_doubles(0, static_cast<int>(max_width(nm)), 1, g_num_sms) * sizeof(double));
  b += 2 * 256;                                                                                // counters
  return b + 256;
}

static int glm_eval_impl(const fb_normalized* nm, const double* y, const double* w, int32_t mode, double* g,
                         double* loss, Carver& cv, fb_stream_t stream) {
  cudaStream_t st = cs(stream);
  fb::GlmArgs a{};
  a.s = nm->s;
  a.n = nm->n_s;
  a.d = nm->d_s;
  a.y = y;
  a.w = w;
  a.mode = mode;
  a.nfk = nm->q;
  int64_t off = nm->d_s;
  double* bins[FB_MAX_PARTS] = {};
  for (int i = 0; i < nm->q; ++i) {
    const fb_part& p = nm->part[i];
    double* z = cv.take<double>(static_cast<size_t>(p.n_r) * fb::z_stride(1));
    bins[i] = cv.take<double>(static_cast<size_t>(p.n_r));
    if (!z || !bins[i]) return fail(FB_ERR_ARG, "glm: workspace too small");
    // z_q = R_q · w_q  (rewrite.py:187, R·X before K)
    cudaError_t e = fb::launch_lmm_rows(p.r, p.n_r, p.d_r, w + off, 1, 1, 0, nullptr, nullptr, 0, z, fb::z_stride(1),
                                        st, g_num_sms);
    if (e == cudaSuccess) e = cudaMemsetAsync(bins[i], 0, static_cast<size_t>(p.n_r) * sizeof(double), st);
    if (e != cudaSuccess) return cuda_status(e, "glm(z)");
    a.fk[i] = p.fk;
    a.z[i] = z;
    a.bins[i] = bins[i];
    off += p.d_r;
  }
  a.g_out = g;
  a.loss_out = loss;
  a.partials = cv.take<double>(fb::glm_partials_doubles(nm->d_s, g_num_sms));
  a.counter = cv.take<unsigned>(1);
  double* cpart = cv.take<double>(fb::colreduce_workspace_doubles(0, static_cast<int>(max_width(nm)), 1, g_num_sms));
  unsigned* ccnt = cv.take<unsigned>(1);
  if (!a.partials || !a.counter || !cpart || !ccnt) return fail(FB_ERR_ARG, "glm: workspace too small");
  if (nm->n_s > 0) {
    cudaError_t e = fb::launch_glm_spass(a, st, g_num_sms);
    if (e != cudaSuccess) return cuda_status(e, "glm(S pass)");
  }
  // g_q = bins_qᵀ R_q  (rmm's (X·K)·R half, rewrite.py:207-209)
  off = nm->d_s;
  for (int i = 0; i < nm->q; ++i) {
    const fb_part& p = nm->part[i];
    fb::ColReduce r{};
    r.a = p.r;
    r.n = p.n_r;
    r.d = p.d_r;
    r.nx = 1;
    r.w = bins[i];
    r.w_rs = 1;
    r.w_cs = 1;
    r.out = g + off;
    r.o_js = 0;
    r.o_cs = 1;
    r.partials = cpart;
    r.counter = ccnt;
    cudaError_t e = fb::launch_colreduce(r, st, g_num_sms);
    if (e != cudaSuccess) return cuda_status(e, "glm(R pass)");
    off += p.d_r;
  }
  return FB_OK;
}

int fb_glm_eval(const fb_normalized* nm, const double* y, const double* w, int32_t mode, double* g, double* loss,
                void* ws, size_t ws_bytes, fb_stream_t stream) {
  int st = check_nm(nm);
  if (st) return st;
  if (mode != 0 && mode != 1) return fail(FB_ERR_ARG, "glm: unknown mode %d", mode);
  if ((!y && nm->n_s > 0) || !w || !g || !loss) return fail(FB_ERR_ARG, "glm: NULL pointer");
  if (nm->d_s > 256 || max_width(nm) > 256) return fail(FB_ERR_ARG, "glm: factor widths above 256 are not supported");
  if (ws_bytes < fb_glm_workspace_bytes(nm)) return fail(FB_ERR_ARG, "glm: workspace too small");
  Carver cv{static_cast<char*>(ws), ws_bytes};
  return glm_eval_impl(nm, y, w, mode, g, loss, cv, stream);
}

int fb_glm_step(const fb_normalized* nm, const double* y, double* w, int32_t mode, double alpha, int32_t it,
                double* trace, int32_t* diverged, void* ws, size_t ws_bytes, fb_stream_t stream) {
  int st = check_nm(nm);
  if (st) return st;
  if (mode != 0 && mode != 1) return fail(FB_ERR_ARG, "glm: unknown mode %d", mode);
  if ((!y && nm->n_s > 0) || !w || !trace || !diverged) return fail(FB_ERR_ARG, "glm: NULL pointer");
  if (nm->d_s > 256 || max_width(nm) > 256) return fail(FB_ERR_ARG, "glm: factor widths above 256 are not supported");
  if (ws_bytes < fb_glm_workspace_bytes(nm)) return fail(FB_ERR_ARG, "glm: workspace too small");
  Carver cv{static_cast<char*>(ws), ws_bytes};
  const int64_t d = total_cols(nm);
  double* g = cv.take<double>(static_cast<size_t>(d + 1));
  double* loss = cv.take<double>(1);
  st = glm_eval_impl(nm, y, w, mode, g, loss, cv, stream);
  if (st) return st;
  // logistic: w += α Tᵀp (ml.py:212); least squares: w -= α Tᵀ(Tw - y) (ml.py:251)
  return cuda_status(fb::launch_glm_update(w, g, static_cast<int>(d), mode == 0 ? alpha : -alpha, loss, trace, it,
                                           diverged, cs(stream)),
                     "glm(update)");
}

// Whole GD run: one cooperative launch when the factors are L2-resident (fb_glm_run.cu),
// else `iters` fused steps. The caller initialises w, trace and *diverged (= -1).
size_t fb_glm_run_workspace_bytes(const fb_normalized* nm) {
  if (!nm) return 0;
  int64_t nr[FB_MAX_PARTS] = {};
  for (int i = 0; i < nm->q; ++i) nr[i] = nm->part[i].n_r;
  return std::max(fb_glm_workspace_bytes(nm),
                  fb::glm_run_workspace_bytes(static_cast<int>(total_cols(nm)), nr, nm->q, g_num_sms));
}

int fb_glm_run_fused(const fb_normalized* nm) {
  if (!nm || check_nm(nm)) return 0;
  if (getenv("FB_GLM_STEPWISE")) return 0;  // force the per-iteration path (tests, comparisons)
  int dr[FB_MAX_PARTS] = {};
  for (int i = 0; i < nm->q; ++i) dr[i] = nm->part[i].d_r;
  return fb::glm_run_eligible(nm->n_s, nm->d_s, nm->q, dr, g_num_sms) ? 1 : 0;
}

int fb_glm_run(const fb_normalized* nm, const double* y, double* w, int32_t mode, double alpha, int32_t iters,
               double* trace, int32_t* diverged, void* ws, size_t ws_bytes, fb_stream_t stream) {
  int st = check_nm(nm);
  if (st) return st;
  if (mode != 0 && mode != 1) return fail(FB_ERR_ARG, "glm: unknown mode %d", mode);
  if ((!y && nm->n_s > 0) || !w || !trace || !diverged || iters < 0) return fail(FB_ERR_ARG, "glm: bad argument");
  if (nm->d_s > 256 || max_width(nm) > 256) return fail(FB_ERR_ARG, "glm: factor widths above 256 are not supported");
  if (ws_bytes < fb_glm_run_workspace_bytes(nm)) return fail(FB_ERR_ARG, "glm: workspace too small");
  int dr[FB_MAX_PARTS] = {};
  for (int i = 0; i < nm->q; ++i) dr[i] = nm->part[i].d_r;
  if (iters > 0 && fb_glm_run_fused(nm)) {
    fb::GlmRunIn in{};
    in.s = nm->s;
    in.n = nm->n_s;
    in.ds = nm->d_s;
    in.y = y;
    in.mode = mode;
    in.alpha = alpha;
    in.q = nm->q;
    for (int i = 0; i < nm->q; ++i) {
      in.fk[i] = nm->part[i].fk;
      in.r[i] = nm->part[i].r;
      in.nr[i] = nm->part[i].n_r;
      in.dr[i] = nm->part[i].d_r;
    }
    in.w = w;
    in.iters = iters;
    in.trace = trace;
    in.diverged = diverged;
    return cuda_status(fb::launch_glm_run(in, ws, ws_bytes, cs(stream), g_num_sms), "glm_run");
  }
  for (int it = 0; it < iters; ++it) {
    st = fb_glm_step(nm, y, w, mode, alpha, it, trace, diverged, ws, ws_bytes, stream);
    if (st) return st;
  }
  return FB_OK;
}

// ------------------------------------------------------------------ K-Means / GNMF steps
size_t fb_kmeans_workspace_bytes(const fb_normalized* nm, int32_t k) {
  if (!nm || k < 1) return 0;
  const int64_t d = total_cols(nm);
  size_t b = 0;
  b += align256(static_cast<size_t>(d) * k * 8);            // 2c
  b += align256(static_cast<size_t>(nm->n_s) * k * 8);      // tc
  b += align256(static_cast<size_t>(d) * k * 8);            // TᵀA
  b += align256(static_cast<size_t>(k) * 4);                // sizes
  b += align256(static_cast<size_t>(g_num_sms) * 8 * 8);    // assign partials
  b += align256(fb::onehot_partials_doubles(nm->d_s > 0 ? nm->d_s : 1, k, g_num_sms) * 8);
  b += align256(fb::colreduce_workspace_doubles(0, static_cast<int>(max_width(nm)), k, g_num_sms) * 8);
  b += 3 * 256;                                             // counters
  b += align256(std::max(fb::kmeans_pass_partials_doubles(g_num_sms), fb::rth_partials_doubles(g_num_sms)) * 8);
  size_t rtx = 0;
  for (int i = 0; i < nm->q; ++i) {
    b += align256(static_cast<size_t>(nm->part[i].n_r) * k * 4) + align256(static_cast<size_t>(nm->part[i].n_r) * k * 8);
    if (fb::rtx_supported(nm->part[i].d_r, k)) rtx = std::max(rtx, fb::rtx_workspace_bytes(nm->part[i].d_r, k, g_num_sms));
  }
  return b + align256(rtx) + fb_lmm_workspace_bytes(nm, k) + 256;
}

static int kmeans_partial_impl(const fb_normalized* nm, const double* d_t, const double* c, const double* cc,
                               int32_t k, int32_t it, double* trace, int32_t* assign, unsigned long long* nan_row,
                               double* tta_out, int32_t* sizes_out, void* ws, size_t ws_bytes, fb_stream_t stream,
                               const fb_band_layout* band = nullptr);

static int kmeans_finish(const fb_normalized* nm, double* c, double* cc, int32_t k, void* ws, size_t ws_bytes,
                         fb_stream_t stream) {
  // the partial left TᵀA and the sizes at the head of the workspace
  const int64_t d = total_cols(nm);
  Carver cv{static_cast<char*>(ws), ws_bytes};
  cv.take<double>(static_cast<size_t>(d) * k);
  cv.take<double>(static_cast<size_t>(nm->n_s) * k);
  double* tta = cv.take<double>(static_cast<size_t>(d) * k);
  int32_t* sizes = cv.take<int32_t>(k);
  return cuda_status(fb::launch_kmeans_update(c, tta, sizes, static_cast<int>(d), k, cc, cs(stream)), "kmeans(update)");
}

int fb_kmeans_banded_supported(const fb_normalized* nm, int32_t k) {
  return nm && nm->q >= 1 && nm->n_s > 0 && fb::kmeans_pass_supported(nm->d_s, k, nm->q) ? 1 : 0;
}

int fb_kmeans_step_banded(const fb_normalized* nm, const fb_band_layout* band, const double* d_t_band, double* c,
                          double* cc, int32_t k, int32_t it, double* trace, int32_t* assign_band,
                          unsigned long long* nan_row, void* ws, size_t ws_bytes, fb_stream_t stream) {
  if (!band || !band->perm || !band->s) return fail(FB_ERR_ARG, "kmeans_banded: NULL band layout");
  if (!fb_kmeans_banded_supported(nm, k)) return fail(FB_ERR_ARG, "kmeans_banded: shape needs the storage-order step");
  for (int q = 0; q < nm->q; ++q)
    if (!band->fk[q]) return fail(FB_ERR_ARG, "kmeans_banded: band layout lacks part %d", q);
  int st = kmeans_partial_impl(nm, d_t_band, c, cc, k, it, trace, assign_band, nan_row, nullptr, nullptr, ws, ws_bytes,
                               stream, band);
  if (st) return st;
  return kmeans_finish(nm, c, cc, k, ws, ws_bytes, stream);
}

int fb_kmeans_step(const fb_normalized* nm, const double* d_t, double* c, double* cc, int32_t k, int32_t it,
                   double* trace, int32_t* assign, unsigned long long* nan_row, void* ws, size_t ws_bytes,
                   fb_stream_t stream) {
  int st = kmeans_partial_impl(nm, d_t, c, cc, k, it, trace, assign, nan_row, nullptr, nullptr, ws, ws_bytes, stream);
  if (st) return st;
  return kmeans_finish(nm, c, cc, k, ws, ws_bytes, stream);
}

int fb_kmeans_partial(const fb_normalized* nm, const double* d_t, const double* c, const double* cc, int32_t k,
                      int32_t it, double* trace, int32_t* assign, unsigned long long* nan_row, double* tta,
                      int32_t* sizes, void* ws, size_t ws_bytes, fb_stream_t stream) {
  if (!tta || !sizes) return fail(FB_ERR_ARG, "kmeans_partial: NULL output");
  return kmeans_partial_impl(nm, d_t, c, cc, k, it, trace, assign, nan_row, tta, sizes, ws, ws_bytes, stream);
}

int fb_kmeans_update(double* c, const double* tta, const int32_t* sizes, int64_t d, int32_t k, double* cc,
                     fb_stream_t stream) {
  if (!c || !tta || !sizes || !cc || d < 1 || k < 1) return fail(FB_ERR_ARG, "kmeans_update: bad argument");
  return cuda_status(fb::launch_kmeans_update(c, tta, sizes, static_cast<int>(d), k, cc, cs(stream)), "kmeans(update)");
}

static int kmeans_partial_impl(const fb_normalized* nm, const double* d_t, const double* c, const double* cc,
                               int32_t k, int32_t it, double* trace, int32_t* assign, unsigned long long* nan_row,
                               double* tta_out, int32_t* sizes_out, void* ws, size_t ws_bytes, fb_stream_t stream,
                               const fb_band_layout* band) {
  int st = check_nm(nm);
  if (st) return st;
  // k <= 16: one fused pass over S (fb_kmeans.cu); wider: T·(2C) in 16-column chunks, then the
  // assign pass, one-hot passes over windows of 64 clusters and column-chunked R passes
  if (k < 1 || k > fb::kKmeansMaxK) return fail(FB_ERR_ARG, "kmeans: k=%d outside [1, %d]", k, fb::kKmeansMaxK);
  if (!d_t || !c || !cc || !trace || !assign || !nan_row) return fail(FB_ERR_ARG, "kmeans: NULL pointer");
  if (max_width(nm) > 256) return fail(FB_ERR_ARG, "kmeans: factor widths above 256 are not supported");
  if (ws_bytes < fb_kmeans_workspace_bytes(nm, k)) return fail(FB_ERR_ARG, "kmeans: workspace too small");
  cudaStream_t s = cs(stream);
  const int64_t d = total_cols(nm);
  Carver cv{static_cast<char*>(ws), ws_bytes};
  double* c2 = cv.take<double>(static_cast<size_t>(d) * k);
  double* tc = cv.take<double>(static_cast<size_t>(nm->n_s) * k);
  double* tta = cv.take<double>(static_cast<size_t>(d) * k);
  int32_t* sizes = cv.take<int32_t>(k);
  if (tta_out) tta = tta_out;
  if (sizes_out) sizes = sizes_out;
  double* apart = cv.take<double>(static_cast<size_t>(g_num_sms) * 8);
  double* opart = cv.take<double>(fb::onehot_partials_doubles(nm->d_s > 0 ? nm->d_s : 1, k, g_num_sms));
  double* cpart = cv.take<double>(fb::colreduce_workspace_doubles(0, static_cast<int>(max_width(nm)), k, g_num_sms));
  unsigned* cnt0 = cv.take<unsigned>(1);
  unsigned* cnt1 = cv.take<unsigned>(1);
  unsigned* cnt2 = cv.take<unsigned>(1);
  fb::KmFk fks{};
  fks.nfk = nm->q;
  double* fbins[FB_MAX_PARTS] = {};
  size_t rtx_bytes = 0;
  for (int i = 0; i < nm->q; ++i) {
    fks.fk[i] = nm->part[i].fk;
    fks.bins[i] = cv.take<int32_t>(static_cast<size_t>(nm->part[i].n_r) * k);
    fbins[i] = cv.take<double>(static_cast<size_t>(nm->part[i].n_r) * k);
    if (fb::rtx_supported(nm->part[i].d_r, k))
      rtx_bytes = std::max(rtx_bytes, fb::rtx_workspace_bytes(nm->part[i].d_r, k, g_num_sms));
  }
  char* rtx_ws = rtx_bytes ? cv.take<char>(rtx_bytes) : nullptr;
  double* kpart = cv.take<double>(std::max(fb::kmeans_pass_partials_doubles(g_num_sms), fb::rth_partials_doubles(g_num_sms)));
  // tc = (2T)·C computed as T·(2C): scaling by two is exact, so the products match bit for bit
  cudaError_t e = fb::launch_scalar_map(c, c2, d * k, fb::kMul, 2.0, s, g_num_sms);
  if (e != cudaSuccess) return cuda_status(e, "kmeans(2c)");
  for (int i = 0; i < nm->q; ++i) {
    e = cudaMemsetAsync(fks.bins[i], 0, static_cast<size_t>(nm->part[i].n_r) * k * 4, s);
    if (e != cudaSuccess) return cuda_status(e, "kmeans(memset)");
  }
  static const bool fused_on = [] { const char* v = getenv("FB_KMEANS_FUSED"); return !(v && atoi(v) == 0); }();
  if ((fused_on || band) && nm->n_s > 0 && fb::kmeans_pass_supported(nm->d_s, k, nm->q)) {
    // one pass over S (fb_kmeans.cu) after the z-passes z_q = R_q · (2C)_q
    fb::KmPass kp{};
    kp.s = band ? band->s : nm->s;
    kp.rr = band != nullptr;
    kp.n = nm->n_s;
    kp.d = nm->d_s;
    kp.d_t = d_t;
    kp.c2s = c2;
    kp.cc = cc;
    kp.k = k;
    kp.nfk = nm->q;
    kp.zst = fb::z_stride(k);
    int64_t zoff = nm->d_s;
    for (int i = 0; i < nm->q; ++i) {
      const fb_part& p = nm->part[i];
      double* z = cv.take<double>(static_cast<size_t>(p.n_r) * kp.zst);
      if (!z) return fail(FB_ERR_ARG, "kmeans: workspace too small");
      e = fb::launch_lmm_rows(p.r, p.n_r, p.d_r, c2 + zoff * k, k, k, 0, nullptr, nullptr, 0, z, kp.zst, s, g_num_sms);
      if (e != cudaSuccess) return cuda_status(e, "kmeans(z)");
      kp.fk[i] = band ? band->fk[i] : p.fk;
      kp.z[i] = z;
      kp.ztable_bytes[i] = static_cast<size_t>(p.n_r) * kp.zst * sizeof(double);
      kp.bins[i] = fks.bins[i];
      zoff += p.d_r;
    }
    kp.assign = assign;
    kp.sizes = sizes;
    kp.partials = kpart;
    kp.counter = cnt0;
    kp.trace = trace;
    kp.it = it;
    kp.nan_row = nan_row;
    kp.sta = tta;
    e = cudaMemsetAsync(sizes, 0, sizeof(int32_t) * k, s);
    if (e != cudaSuccess) return cuda_status(e, "kmeans(sizes)");
    e = fb::launch_kmeans_pass(kp, s, g_num_sms);
    if (e != cudaSuccess) return cuda_status(e, "kmeans(pass)");
  } else {
    st = fb_lmm(nm, c2, k, tc, cv.p, cv.left, stream);
    if (st) return st;
    e = fb::launch_kmeans_assign(tc, d_t, cc, nm->n_s, k, fks, assign, sizes, apart, cnt0, trace, it, nan_row, s,
                                 g_num_sms);
    if (e != cudaSuccess) return cuda_status(e, "kmeans(assign)");
    // TᵀA: S part by one-hot column sums, R parts as R_qᵀ (A_qᵀ K_q) from the integer histograms
    if (nm->d_s > 0) {
      e = fb::launch_onehot_colsum(nm->s, nm->n_s, nm->d_s, assign, k, opart, cnt1, tta, s, g_num_sms);
      if (e != cudaSuccess) return cuda_status(e, "kmeans(onehot)");
    }
  }
  int64_t off = nm->d_s;
  for (int i = 0; i < nm->q; ++i) {
    const fb_part& p = nm->part[i];
    if (fb::rth_supported(p.d_r, k)) {  // R_qᵀ H_q straight from the integer histograms
      e = fb::launch_rth(p.r, p.n_r, p.d_r, fks.bins[i], k, tta + off * k, k, 1, kpart, cnt2, s, g_num_sms);
      if (e != cudaSuccess) return cuda_status(e, "kmeans(R pass)");
      off += p.d_r;
      continue;
    }
    e = fb::launch_i32_to_f64(fks.bins[i], fbins[i], p.n_r * k, s, g_num_sms);
    if (e != cudaSuccess) return cuda_status(e, "kmeans(bins)");
    if (rtx_ws && fb::rtx_supported(p.d_r, k)) {  // R_qᵀ H_q on the tensor cores
      e = fb::launch_rtx(p.r, p.n_r, p.d_r, fbins[i], k, tta + off * k, k, 1, rtx_ws, rtx_bytes, s, g_num_sms);
      if (e != cudaSuccess) return cuda_status(e, "kmeans(R pass)");
      off += p.d_r;
      continue;
    }
    for (int c0 = 0; c0 < k;) {  // column chunks of the widths the reduction is instantiated for
      const int w = chunk_width(k - c0);
      fb::ColReduce r{};
      r.a = p.r;
      r.n = p.n_r;
      r.d = p.d_r;
      r.nx = w;
      r.w = fbins[i] + c0;
      r.w_rs = k;
      r.w_cs = 1;
      r.out = tta + off * k + c0;
      r.o_js = 1;
      r.o_cs = k;
      r.partials = cpart;
      r.counter = cnt2;
      e = fb::launch_colreduce(r, s, g_num_sms);
      if (e != cudaSuccess) return cuda_status(e, "kmeans(R pass)");
      c0 += w;
    }
    off += p.d_r;
  }
  return FB_OK;
}

size_t fb_gnmf_workspace_bytes(const fb_normalized* nm, int32_t r) {
  if (!nm || r < 1) return 0;
  fb_normalized wm{};
  wm.n_s = nm->n_s;
  wm.d_s = r;
  size_t inner = fb_lmm_workspace_bytes(nm, r);
  inner = std::max(inner, fb_wt_workspace_bytes(nm, r));
  inner = std::max(inner, fb_crossprod_workspace_bytes(&wm));
  size_t fused = align256(std::max(fb::nmf_pass_partials_doubles(g_num_sms), fb::rth_partials_doubles(g_num_sms)) * 8) + 256;
  for (int i = 0; i < nm->q; ++i) fused += align256(static_cast<size_t>(nm->part[i].n_r) * r * 8);
  return align256(static_cast<size_t>(nm->n_s) * r * 8) + align256(static_cast<size_t>(r) * r * 8) + fused + inner + 256;
}

int fb_gnmf_step(const fb_normalized* nm, double* w, double* h, double* ttw, double* cpw, const double* sum_t2,
                 int32_t r, int32_t it, double* trace, void* ws, size_t ws_bytes, fb_stream_t stream) {
  int st = check_nm(nm);
  if (st) return st;
  // r <= 16: one fused pass over S per W step (fb_gnmf.cu); wider: the operator-by-operator step
  if (r < 1 || r > fb::kNmfStepMaxR) return fail(FB_ERR_ARG, "gnmf: r=%d outside [1, %d]", r, fb::kNmfStepMaxR);
  if (!w || !h || !ttw || !cpw || !sum_t2 || !trace) return fail(FB_ERR_ARG, "gnmf: NULL pointer");
  if (ws_bytes < fb_gnmf_workspace_bytes(nm, r)) return fail(FB_ERR_ARG, "gnmf: workspace too small");
  cudaStream_t s = cs(stream);
  const int64_t d = total_cols(nm);
  const double eps = 1e-12;
  Carver cv{static_cast<char*>(ws), ws_bytes};
  double* th = cv.take<double>(static_cast<size_t>(nm->n_s) * r);
  double* cph = cv.take<double>(static_cast<size_t>(r) * r);
  // h = h ∘ ttw / (h·cpw + eps); cph = hᵀh
  cudaError_t e = fb::launch_nmf_update(h, ttw, cpw, d, r, eps, s, g_num_sms);
  if (e == cudaSuccess) e = fb::launch_small_gram(h, d, r, cph, s);
  if (e != cudaSuccess) return cuda_status(e, "gnmf(h)");
  double* npart = cv.take<double>(std::max(fb::nmf_pass_partials_doubles(g_num_sms), fb::rth_partials_doubles(g_num_sms)));
  unsigned* ncnt = cv.take<unsigned>(1);
  double* nbins[FB_MAX_PARTS] = {};
  for (int i = 0; i < nm->q; ++i) nbins[i] = cv.take<double>(static_cast<size_t>(nm->part[i].n_r) * r);
  static const bool fused_on = [] { const char* v = getenv("FB_GNMF_FUSED"); return !(v && atoi(v) == 0); }();
  if (fused_on && nm->n_s > 0 && fb::nmf_pass_supported(nm->d_s, r, nm->q)) {
    // one pass over S (fb_gnmf.cu): th, the W update, SᵀW, WᵀW and the K_qᵀW bins; then R_qᵀ bins_q
    fb::NmfPass np{};
    np.s = nm->s;
    np.n = nm->n_s;
    np.d = nm->d_s;
    np.w = w;
    np.r = r;
    np.h = h;
    np.cph = cph;
    np.eps = eps;
    np.nfk = nm->q;
    np.zst = fb::z_stride(r);
    int64_t off = nm->d_s;
    for (int i = 0; i < nm->q; ++i) {
      const fb_part& p = nm->part[i];
      double* z = cv.take<double>(static_cast<size_t>(p.n_r) * np.zst);
      if (!z) return fail(FB_ERR_ARG, "gnmf: workspace too small");
      // z_q = R_q · H[off:off+d_r]   (rewrite.py:187)
      e = fb::launch_lmm_rows(p.r, p.n_r, p.d_r, h + off * r, r, r, 0, nullptr, nullptr, 0, z, np.zst, s, g_num_sms);
      if (e == cudaSuccess) e = cudaMemsetAsync(nbins[i], 0, static_cast<size_t>(p.n_r) * r * 8, s);
      if (e != cudaSuccess) return cuda_status(e, "gnmf(z)");
      np.fk[i] = p.fk;
      np.z[i] = z;
      np.ztable_bytes[i] = static_cast<size_t>(p.n_r) * np.zst * sizeof(double);
      np.bins[i] = nbins[i];
      if (p.nhot > 0 && p.hot_slot && p.hot_key) {
        np.hot_slot[i] = p.hot_slot;
        np.hot_key[i] = p.hot_key;
        np.nhot[i] = p.nhot < 64 ? p.nhot : 64;
      }
      off += p.d_r;
    }
    np.partials = npart;
    np.ttw_s = ttw;
    np.cpw = cpw;
    e = fb::launch_nmf_wpass(np, s, g_num_sms);
    if (e != cudaSuccess) return cuda_status(e, "gnmf(W pass)");
    off = nm->d_s;
    for (int i = 0; i < nm->q; ++i) {  // ttw[off:off+d_r] = R_qᵀ (K_qᵀ W)
      const fb_part& p = nm->part[i];
      if (fb::rth_supported(p.d_r, r)) {
        e = fb::launch_rth(p.r, p.n_r, p.d_r, static_cast<const double*>(nbins[i]), r, ttw + off * r, r, 1, npart,
                           ncnt, s, g_num_sms);
      } else {
        fb::ColReduce c{};
        c.a = p.r;
        c.n = p.n_r;
        c.d = p.d_r;
        c.nx = r;
        c.w = nbins[i];
        c.w_rs = r;
        c.w_cs = 1;
        c.out = ttw + off * r;
        c.o_js = 1;
        c.o_cs = r;
        c.partials = npart;
        c.counter = ncnt;
        e = cudaMemsetAsync(ncnt, 0, sizeof(unsigned), s);
        if (e == cudaSuccess) e = fb::launch_colreduce(c, s, g_num_sms);
      }
      if (e != cudaSuccess) return cuda_status(e, "gnmf(R pass)");
      off += p.d_r;
    }
    return cuda_status(fb::launch_nmf_objective(sum_t2, ttw, h, d * r, cpw, cph, r * r, trace, it, s),
                       "gnmf(objective)");
  }
  // th = T·h; w = w ∘ th / (w·cph + eps)
  st = fb_lmm(nm, h, r, th, cv.p, cv.left, stream);
  if (st) return st;
  e = fb::launch_nmf_update(w, th, cph, nm->n_s, r, eps, s, g_num_sms);
  if (e != cudaSuccess) return cuda_status(e, "gnmf(w)");
  // ttw = Tᵀw (also the next iteration's ttw, ml.py:307/312); cpw = wᵀw
  st = fb_wt(nm, w, r, r, 1, ttw, 1, r, cv.p, cv.left, stream);
  if (st) return st;
  fb_normalized wm{};
  wm.s = w;
  wm.n_s = nm->n_s;
  wm.d_s = r;
  st = fb_crossprod(&wm, nullptr, nullptr, cpw, cv.p, cv.left, stream);
  if (st) return st;
  return cuda_status(fb::launch_nmf_objective(sum_t2, ttw, h, d * r, cpw, cph, r * r, trace, it, s), "gnmf(objective)");
}

int fb_glm_update(double* w, const double* g, int64_t d, double alpha, const double* loss, double* trace, int32_t it,
                  int32_t* diverged, fb_stream_t stream) {
  if (!w || !g || !loss || !trace || !diverged || d < 1) return fail(FB_ERR_ARG, "glm_update: bad argument");
  return cuda_status(fb::launch_glm_update(w, g, static_cast<int>(d), alpha, loss, trace, it, diverged, cs(stream)),
                     "glm(update)");
}

int fb_nmf_update(double* f, const double* num, const double* g, int64_t rows, int32_t r, fb_stream_t stream) {
  if (!f || !num || !g || r < 1 || r > fb::kNmfStepMaxR || rows < 0) return fail(FB_ERR_ARG, "nmf_update: bad argument");
  return cuda_status(fb::launch_nmf_update(f, num, g, rows, r, 1e-12, cs(stream), g_num_sms), "nmf_update");
}

int fb_small_gram(const double* f, int64_t rows, int32_t r, double* g, fb_stream_t stream) {
  if (!f || !g || r < 1 || rows < 0) return fail(FB_ERR_ARG, "small_gram: bad argument");
  return cuda_status(fb::launch_small_gram(f, rows, r, g, cs(stream)), "small_gram");
}

int fb_nmf_objective(const double* sum_t2, const double* ttw, const double* h, int64_t dr, const double* cpw,
                     const double* cph, int32_t rr, double* trace, int32_t it, fb_stream_t stream) {
  if (!sum_t2 || !ttw || !h || !cpw || !cph || !trace) return fail(FB_ERR_ARG, "nmf_objective: NULL pointer");
  return cuda_status(fb::launch_nmf_objective(sum_t2, ttw, h, dr, cpw, cph, rr, trace, it, cs(stream)),
                     "nmf_objective");
}

int fb_mirror_upper(double* a, int64_t d, fb_stream_t stream) {
  if (d < 0 || (d > 0 && !a)) return fail(FB_ERR_ARG, "mirror_upper: bad argument");
  if (d == 0) return FB_OK;
  const int64_t n = d * d;
  mirror_upper_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, cs(stream)>>>(a, d);
  FB_LAUNCHED();
  return cuda_status(cudaGetLastError(), "mirror_upper");
}

// ------------------------------------------------------------------ element-wise
int fb_scalar_map(const double* in, double* out, int64_t n, int32_t op, double x, fb_stream_t stream) {
  if (op < 0 || op > 9) return fail(FB_ERR_ARG, "scalar_map: unknown op %d", op);
  if (op == fb::kDiv && x == 0.0) return fail(FB_ERR_NUMERIC, "division by zero scalar");
  if (n > 0 && (!in || !out)) return fail(FB_ERR_ARG, "scalar_map: NULL pointer");
  return cuda_status(fb::launch_scalar_map(in, out, n, op, x, cs(stream), g_num_sms), "scalar_map");
}

int fb_unary_map(const double* in, double* out, int64_t n, int32_t fn, fb_stream_t stream) {
  if (fn < 0 || fn > 13) return fail(FB_ERR_ARG, "unary_map: unknown function %d", fn);
  if (n > 0 && (!in || !out)) return fail(FB_ERR_ARG, "unary_map: NULL pointer");
  return cuda_status(fb::launch_unary_map(in, out, n, fn, cs(stream), g_num_sms), "unary_map");
}

size_t fb_glm_pointwise_workspace_bytes(void) { return fb::glm_pointwise_workspace_bytes(g_num_sms); }

int fb_glm_pointwise(const double* tw, const double* y, int64_t n, int32_t mode, double* p, double* trace, int32_t it,
                     void* ws, size_t ws_bytes, fb_stream_t stream) {
  if (n < 0 || (mode != 0 && mode != 1) || it < 0) return fail(FB_ERR_ARG, "glm_pointwise: bad argument");
  if ((n > 0 && (!tw || !y || !p)) || !trace || !ws) return fail(FB_ERR_ARG, "glm_pointwise: NULL pointer");
  if (ws_bytes < fb_glm_pointwise_workspace_bytes()) return fail(FB_ERR_ARG, "glm_pointwise: workspace too small");
  return cuda_status(fb::launch_glm_pointwise(tw, y, n, mode, p, trace, it, ws, cs(stream), g_num_sms), "glm_pointwise");
}

int fb_axpy_check(double alpha, const double* x, double* y, int64_t n, int32_t it, int32_t* diverged,
                  fb_stream_t stream) {
  if (n < 0 || (n > 0 && (!x || !y)) || !diverged) return fail(FB_ERR_ARG, "axpy_check: bad argument");
  return cuda_status(fb::launch_axpy_check(alpha, x, y, n, it, diverged, cs(stream), g_num_sms), "axpy_check");
}

// ------------------------------------------------------------------ dense / sparse pieces (fb_dense.cu)
int fb_dense_mm(int64_t m, int64_t n, int64_t k, const double* a, int64_t lda, int32_t ta, const double* b,
                int64_t ldb, int32_t tb, double* c, int64_t ldc, int32_t accumulate, fb_stream_t stream) {
  if (m < 0 || n < 0 || k < 0 || ldc < n) return fail(FB_ERR_SHAPE, "dense_mm: bad shape");
  if ((m > 0 && n > 0) && (!c || (k > 0 && (!a || !b)))) return fail(FB_ERR_ARG, "dense_mm: NULL pointer");
  return cuda_status(fb::launch_dense_mm(m, n, k, a, lda, ta, b, ldb, tb, c, ldc, accumulate, cs(stream)), "dense_mm");
}

int fb_gather2_add(int64_t m, int64_t n, const double* mat, int64_t ldm, const int32_t* ra, const int32_t* cb,
                   double* c, int64_t ldc, fb_stream_t stream) {
  if (m < 0 || n < 0 || ldc < n) return fail(FB_ERR_SHAPE, "gather2_add: bad shape");
  if (m > 0 && n > 0 && (!mat || !ra || !c)) return fail(FB_ERR_ARG, "gather2_add: NULL pointer");
  return cuda_status(fb::launch_gather2_add(m, n, mat, ldm, ra, cb, c, ldc, cs(stream), g_num_sms), "gather2_add");
}

int fb_scatter_rows(int64_t n, int32_t d, const int32_t* tgt, const double* a, int64_t lda, double* out,
                    int64_t out_rows, fb_stream_t stream) {
  if (n < 0 || d < 0 || out_rows < 0) return fail(FB_ERR_SHAPE, "scatter_rows: bad shape");
  if ((n > 0 && d > 0 && (!tgt || !a)) || (out_rows > 0 && d > 0 && !out)) return fail(FB_ERR_ARG, "scatter_rows: NULL pointer");
  return cuda_status(fb::launch_scatter_rows(n, d, tgt, a, lda, out, out_rows, cs(stream), g_num_sms), "scatter_rows");
}

size_t fb_pair_counts_workspace_bytes(int64_t n) { return fb::pair_counts_workspace_bytes(n); }

int fb_pair_counts(int64_t n, const int32_t* ta, const int32_t* tb, int64_t rows_a, int64_t cols_b, int64_t* indptr,
                   int64_t* col, double* val, int64_t* nnz, void* ws, size_t ws_bytes, fb_stream_t stream) {
  if (n < 0 || rows_a < 0 || cols_b < 0) return fail(FB_ERR_SHAPE, "pair_counts: bad shape");
  if (!indptr || !nnz || (n > 0 && (!ta || !tb || !col || !val))) return fail(FB_ERR_ARG, "pair_counts: NULL pointer");
  if (ws_bytes < fb::pair_counts_workspace_bytes(n)) return fail(FB_ERR_ARG, "pair_counts: workspace too small");
  return cuda_status(fb::launch_pair_counts(n, ta, tb, rows_a, cols_b, indptr, col, val, nnz, ws, ws_bytes, cs(stream),
                                            g_num_sms),
                     "pair_counts");
}

int fb_csr_spmm(int64_t rows, const int64_t* indptr, const void* col, int32_t col_is64, const double* val,
                const double* x, int64_t ldx, int32_t k, double* y, int64_t ldy, int32_t accumulate,
                fb_stream_t stream) {
  if (rows < 0 || k < 0 || ldy < k) return fail(FB_ERR_SHAPE, "csr_spmm: bad shape");
  if (rows > 0 && k > 0 && (!indptr || !y)) return fail(FB_ERR_ARG, "csr_spmm: NULL pointer");
  return cuda_status(fb::launch_csr_spmm(rows, indptr, col, col_is64, val, x, ldx, k, y, ldy, accumulate, cs(stream),
                                         g_num_sms),
                     "csr_spmm");
}

int fb_csr_spmm_t(int64_t rows, int64_t cols, const int64_t* indptr, const void* col, int32_t col_is64,
                  const double* val, const double* x, int64_t ldx, int32_t k, double* y, int64_t ldy,
                  fb_stream_t stream) {
  if (rows < 0 || cols < 0 || k < 0 || ldy < k) return fail(FB_ERR_SHAPE, "csr_spmm_t: bad shape");
  if (cols > 0 && k > 0 && !y) return fail(FB_ERR_ARG, "csr_spmm_t: NULL pointer");
  return cuda_status(fb::launch_csr_spmm_t(rows, cols, indptr, col, col_is64, val, x, ldx, k, y, ldy, cs(stream),
                                           g_num_sms),
                     "csr_spmm_t");
}

}  // extern "C"
