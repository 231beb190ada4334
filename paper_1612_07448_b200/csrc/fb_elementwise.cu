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

}  // namespace fb
