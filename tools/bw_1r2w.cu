// Achievable HBM bandwidth for 1 read + 2 writes per element (the reconstruction's traffic), vs copy.
#include <cstdio>
__global__ void r1w2(const float4* __restrict__ a, float4* __restrict__ b, float4* __restrict__ c, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcs(a + i);
    __stcs(b + i, v);
    __stcs(c + i, make_float4(-v.x, -v.y, -v.z, -v.w));
  }
}
__global__ void r1w1(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}
__global__ void r1w2_plain(const float4* __restrict__ a, float4* __restrict__ b, float4* __restrict__ c, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = a[i];
    b[i] = v;
    c[i] = make_float4(-v.x, -v.y, -v.z, -v.w);
  }
}
int main() {
  const size_t n = 768000000ull / 4;  // float4 elements: 768M floats (cfg4)
  float4 *a, *b, *c;
  cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16); cudaMalloc(&c, n * 16);
  cudaMemset(a, 0, n * 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int grid : {148 * 4, 148 * 8, 148 * 16, 148 * 64}) {
    for (int mode = 0; mode < 3; ++mode) {
      for (int w = 0; w < 2; ++w) {
        if (mode == 0) r1w2<<<grid, 256>>>(a, b, c, n); else if (mode == 1) r1w1<<<grid, 256>>>(a, b, n); else r1w2_plain<<<grid, 256>>>(a, b, c, n);
      }
      cudaEventRecord(e0);
      for (int it = 0; it < 5; ++it) {
        if (mode == 0) r1w2<<<grid, 256>>>(a, b, c, n); else if (mode == 1) r1w1<<<grid, 256>>>(a, b, n); else r1w2_plain<<<grid, 256>>>(a, b, c, n);
      }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
      const double bytes = (mode == 1 ? 2.0 : 3.0) * n * 16;
      printf("grid %5d %-10s %.3f ms  %.0f GB/s\n", grid, mode == 0 ? "1r2w cs" : mode == 1 ? "copy cs" : "1r2w plain", ms, bytes / ms / 1e6);
    }
  }
  return 0;
}
