// C-ABI housekeeping: error strings, version, device query and the FP32 FMA-throughput
// probe used as the filter kernel's roofline denominator.
#include "common.cuh"

#include <cstdarg>
#include <cstdio>

namespace l1f {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// keep freed stream-ordered allocations in the default pool (the default release threshold of
// 0 returns them to the driver at every synchronisation and re-maps them on the next call)
static void keep_pool_memory(int dev) {
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

// process-wide option table (l1f_set_option); index = L1F_OPT_* key
static constexpr int kNumOptions = 13;
static int64_t g_options[kNumOptions] = {0, 0, 1, 0, 1, 1, 1, 1, 10000, 0, 2, 1, 1};

int64_t option(int key) {
  return (key > 0 && key < kNumOptions) ? __atomic_load_n(&g_options[key], __ATOMIC_RELAXED) : 0;
}

int num_sms() {
  static int cached = 0;
  if (!cached) {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) {
      cached = v;
      keep_pool_memory(dev);
    }
    else
      cached = 148;
  }
  return cached;
}

// 8 independent FMA chains per thread, operands in registers; 2 FLOP per FMA.
__global__ void __launch_bounds__(256) fma_probe_kernel(int iters, float* sink) {
  float a0 = threadIdx.x * 1e-7f, a1 = a0 + 1e-7f, a2 = a0 + 2e-7f, a3 = a0 + 3e-7f;
  float a4 = a0 + 4e-7f, a5 = a0 + 5e-7f, a6 = a0 + 6e-7f, a7 = a0 + 7e-7f;
  const float b = 0.999999f, c = 1e-9f * (blockIdx.x + 1);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
      a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
    }
  }
  const float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678f) sink[blockIdx.x] = s;  // keeps the chains alive
}

__global__ void __launch_bounds__(256) fma_probe_f64_kernel(int iters, double* sink) {
  double a0 = threadIdx.x * 1e-7, a1 = a0 + 1e-7, a2 = a0 + 2e-7, a3 = a0 + 3e-7;
  double a4 = a0 + 4e-7, a5 = a0 + 5e-7, a6 = a0 + 6e-7, a7 = a0 + 7e-7;
  const double b = 0.999999, c = 1e-9 * (blockIdx.x + 1);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) sink[blockIdx.x] = s;  // keeps the chains alive
}

}  // namespace l1f

using namespace l1f;

extern "C" const char* l1f_last_error(void) { return g_err; }

extern "C" int l1f_set_option(int key, int64_t value) {
  L1F_REQUIRE(key > 0 && key < kNumOptions, L1F_ERR_ARG, "set_option: unknown option %d", key);
  L1F_REQUIRE(key != L1F_OPT_WAIT_TIMEOUT_MS || value >= 0, L1F_ERR_ARG, "set_option: timeout must be >= 0");
  __atomic_store_n(&g_options[key], value, __ATOMIC_RELAXED);
  return L1F_OK;
}

extern "C" int l1f_get_option(int key, int64_t* value_host) {
  L1F_REQUIRE(key > 0 && key < kNumOptions && value_host, L1F_ERR_ARG, "get_option: unknown option %d", key);
  *value_host = option(key);
  return L1F_OK;
}
extern "C" int l1f_version(void) { return 10000; }

extern "C" int l1f_sm_count(int* out_host) {
  int dev = 0, v = 0;
  L1F_CUDA_TRY(cudaGetDevice(&dev));
  L1F_CUDA_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
  *out_host = v;
  return L1F_OK;
}

extern "C" int l1f_fma_peak_probe(int32_t iters, float* sink, double* flops_host, void* stream) {
  L1F_REQUIRE(iters > 0, L1F_ERR_ARG, "iters must be positive");
  const int blocks = num_sms() * 8;  // 8 x 256 threads = 64 warps per SM
  fma_probe_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(iters, sink);
  L1F_CHECK_LAUNCH();
  *flops_host = 2.0 * 8.0 * 16.0 * (double)iters * 256.0 * (double)blocks;
  return L1F_OK;
}

extern "C" int l1f_fma_peak_probe_f64(int32_t iters, double* sink, double* flops_host, void* stream) {
  L1F_REQUIRE(iters > 0, L1F_ERR_ARG, "iters must be positive");
  const int blocks = num_sms() * 8;
  fma_probe_f64_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(iters, sink);
  L1F_CHECK_LAUNCH();
  *flops_host = 2.0 * 8.0 * 16.0 * (double)iters * 256.0 * (double)blocks;
  return L1F_OK;
}
