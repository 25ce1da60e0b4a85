// Shared helpers for the l1-filtering PCP kernels (sm_100a).
//
// Every C-ABI entry point returns an int status (L1F_OK or a negative code) and
// records a human-readable message retrievable through l1f_last_error(); no C++
// exception crosses the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <float.h>
#include <string>

#include "../../include/l1pcp_b200.h"

namespace l1f {

void set_error(const char* fmt, ...);

#define L1F_CUDA_TRY(expr)                                                        \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      ::l1f::set_error("%s:%d: %s: %s", __FILE__, __LINE__, #expr,                \
                       cudaGetErrorString(_e));                                   \
      return L1F_ERR_CUDA;                                                        \
    }                                                                             \
  } while (0)

#define L1F_CHECK_LAUNCH() L1F_CUDA_TRY(cudaGetLastError())

#define L1F_REQUIRE(cond, code, ...)                                              \
  do {                                                                            \
    if (!(cond)) {                                                                \
      ::l1f::set_error(__VA_ARGS__);                                              \
      return (code);                                                              \
    }                                                                             \
  } while (0)

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

int num_sms();
int64_t option(int key);  // l1f_set_option values (L1F_OPT_*), defaults when unset

template <typename T> struct Limits;
template <> struct Limits<float> {
  __host__ __device__ static constexpr float tiny() { return FLT_MIN; }
  __host__ __device__ static constexpr float inf() { return __builtin_huge_valf(); }
};
template <> struct Limits<double> {
  __host__ __device__ static constexpr double tiny() { return DBL_MIN; }
  __host__ __device__ static constexpr double inf() { return __builtin_huge_val(); }
};

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float  tabs(float v)  { return fabsf(v); }
__device__ __forceinline__ double tabs(double v) { return fabs(v); }
__device__ __forceinline__ float  tmax(float a, float b)   { return fmaxf(a, b); }
__device__ __forceinline__ double tmax(double a, double b) { return fmax(a, b); }

// FP64 reciprocal and square root from the hardware estimates with Newton steps (within an ulp of
// IEEE; off the division / sqrt subroutines, which cost ~10x more issue slots)
__device__ __forceinline__ double rcp_nr2(double x) {
  if (!(fabs(x) > 4.0 * DBL_MIN)) return 1.0 / x;  // the estimate flushes subnormals
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-x, r, 2.0);
  return r * fma(-x, r, 2.0);
}
__device__ __forceinline__ double sqrt_nr(double x) {  // x > 0 normal
  if (!(x > 4.0 * DBL_MIN) || x > 1e300) return sqrt(x);
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-0.5 * x * r, r, 1.5);
  r = r * fma(-0.5 * x * r, r, 1.5);
  const double s = x * r;
  return fma(0.5 * r, fma(-s, s, x), s);  // one correction of the root itself
}
// Householder reflector scalars of (alpha, x) with ||x||^2 = xnorm2 > 0 (LAPACK dlarfg without
// the rescaling loop): beta = -sign(alpha) ||(alpha, x)||, tau = (beta - alpha) / beta,
// v = x / (alpha - beta) (returned as its scale)
__device__ __forceinline__ void householder_scalars(double alpha, double xnorm2, double& beta, double& tau,
                                                    double& scale) {
  beta = -copysign(sqrt_nr(fma(alpha, alpha, xnorm2)), alpha);
  tau = (beta - alpha) * rcp_nr2(beta);
  scale = rcp_nr2(alpha - beta);
}

// sign(w) * max(|w| - t, 0), the reference's soft threshold
// (pkg/src/l1pcp/matcore.py:66-70; per-unit use at l1reg.py:97).
template <typename T>
__device__ __forceinline__ T shrink(T w, T t) {
  T m = tabs(w) - t;
  m = m > T(0) ? m : T(0);
  return w > T(0) ? m : (w < T(0) ? -m : T(0));
}

}  // namespace l1f
