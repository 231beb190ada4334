// fb_elementwise.cu — element-wise scalar operators on factor matrices.
//
// Replaces kernel.scalar_map / kernel.unary_map (kernel.py:219-300) as driven by
// rewrite.scalar_op / scalar_fn (rewrite.py:61-99): the operator is applied to each
// factor matrix (S and every R_i) and the indicators are carried over unchanged.
// Pure HBM streaming: 16-byte vector loads/stores, grid sized to whole waves.
#include <cmath>

#include "fb_kernels.cuh"

namespace fb {

FB_DEV double apply_scalar(int op, double v, double x) {
  switch (op) {
    case kAdd:
    case kRadd:
      return v + x;
    case kSub:
      return v - x;
    case kRsub:
      return x - v;
    case kMul:
    case kRmul:
      return v * x;
    case kDiv:
      return v / x;
    case kRdiv:
      return x / v;
    case kPow:
      return pow(v, x);
    default:  // kRpow
      return pow(x, v);
  }
}

FB_DEV double apply_unary(int fn, double v) {
  switch (fn) {
    case kExp:
      return exp(v);
    case kLog:
      return log(v);
    case kSquare:
      return v * v;
    case kSqrt:
      return sqrt(v);
    case kAbs:
      return fabs(v);
    case kNeg:
      return -v;
    case kLog1p:
      return log1p(v);
    case kExpm1:
      return expm1(v);
    case kSin:
      return sin(v);
    case kCos:
      return cos(v);
    case kTanh:
      return tanh(v);
    case kSigmoid:
      return 1.0 / (1.0 + exp(-v));
    case kReciprocal:
      return 1.0 / v;
    default:
      return v;
  }
}

template <bool kUnary>
__global__ void __launch_bounds__(256) map_kernel(const double* __restrict__ in,
                                                  double* __restrict__ out, int64_t n, int op,
                                                  double x) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u) == 0;
  if (vec) {
    const int64_t n2 = n / 2;
    const double2* in2 = reinterpret_cast<const double2*>(in);
    double2* out2 = reinterpret_cast<double2*>(out);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n2;
         i += stride) {
      double2 v = ld_stream_d2(in2 + i);
      if (kUnary) {
        v.x = apply_unary(op, v.x);
        v.y = apply_unary(op, v.y);
      } else {
        v.x = apply_scalar(op, v.x, x);
        v.y = apply_scalar(op, v.y, x);
      }
      out2[i] = v;
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
      const double v = in[n - 1];
      out[n - 1] = kUnary ? apply_unary(op, v) : apply_scalar(op, v, x);
    }
  } else {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += stride) {
      const double v = in[i];
      out[i] = kUnary ? apply_unary(op, v) : apply_scalar(op, v, x);
    }
  }
}

static int map_grid(int64_t n, int num_sms) {
  return grid_for((n + 1) / 2, 256 * 4, 8, num_sms);
}

cudaError_t launch_scalar_map(const double* in, double* out, int64_t n, int op, double x,
                              cudaStream_t st, int num_sms) {
  if (n <= 0) return cudaSuccess;
  map_kernel<false><<<map_grid(n, num_sms), 256, 0, st>>>(in, out, n, op, x);
  FB_LAUNCHED();
  return cudaGetLastError();
}

cudaError_t launch_unary_map(const double* in, double* out, int64_t n, int fn, cudaStream_t st,
                             int num_sms) {
  if (n <= 0) return cudaSuccess;
  map_kernel<true><<<map_grid(n, num_sms), 256, 0, st>>>(in, out, n, fn, 0.0);
  FB_LAUNCHED();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ GLM point-wise pieces
// The drivers on a transposed normalized matrix (ml.py:199-254 with T = Mᵀ) get T·w and Tᵀ·p from
// the factorized operators; what is left per iteration is point-wise over the n-long vectors:
//   mode 0 (logistic): p = y / (1 + exp(tw)), loss_i = log1p(exp(-|y·tw|)) + max(-y·tw, 0)  (ml.py:207-211)
//   mode 1 (least squares): p = tw - y, loss_i = p²                                       (ml.py:247-249)
// Block partials of the loss are written per CTA and summed in CTA order by the last CTA
// (deterministic); trace[it] gets the sum.
__global__ void __launch_bounds__(256) glm_pointwise_kernel(const double* __restrict__ tw,
                                                            const double* __restrict__ y, int64_t n, int mode,
                                                            double* __restrict__ p, double* partials,
                                                            unsigned* counter, double* trace, int it) {
  __shared__ double red[256];
  __shared__ bool last;
  double loss = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double t = tw[i], yy = y[i];
    if (mode == 0) {
      p[i] = yy / (1.0 + exp(t));
      const double m = yy * t;
      loss += log1p(exp(-fabs(m))) + fmax(-m, 0.0);
    } else {
      const double r = t - yy;
      p[i] = r;
      loss += r * r;
    }
  }
  red[threadIdx.x] = loss;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = red[0];
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double s = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) s += partials[b];
    trace[it] = s;
    *counter = 0u;
  }
}

size_t glm_pointwise_workspace_bytes(int num_sms) { return static_cast<size_t>(num_sms) * 4 * 8 + 256; }

cudaError_t launch_glm_pointwise(const double* tw, const double* y, int64_t n, int mode, double* p, double* trace,
                                 int it, void* ws, cudaStream_t st, int num_sms) {
  const int grid = num_sms * 4;
  double* partials = static_cast<double*>(ws);
  unsigned* counter = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + static_cast<size_t>(grid) * 8);
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  glm_pointwise_kernel<<<grid, 256, 0, st>>>(tw, y, n, mode, p, partials, counter, trace, it);
  FB_LAUNCHED();
  return cudaGetLastError();
}

// y += alpha·x; *diverged (start at -1) latches the first iteration whose y holds a non-finite value
// (the reference checks np.isfinite(w).all() after every update, ml.py:213, 252).
__global__ void __launch_bounds__(256) axpy_check_kernel(double alpha, const double* __restrict__ x,
                                                         double* __restrict__ y, int64_t n, int it, int* diverged) {
  bool bad = false;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = y[i] + alpha * x[i];
    y[i] = v;
    bad |= !isfinite(v);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicCAS(diverged, -1, it);
}

cudaError_t launch_axpy_check(double alpha, const double* x, double* y, int64_t n, int it, int* diverged,
                              cudaStream_t st, int num_sms) {
  if (n <= 0) return cudaSuccess;
  axpy_check_kernel<<<grid_for(n, 256 * 4, 8, num_sms), 256, 0, st>>>(alpha, x, y, n, it, diverged);
  FB_LAUNCHED();
  return cudaGetLastError();
}

}  // namespace fb
