// Microbenchmark: tcgen05 bf16 MMA rate (M=128, K=16, N=96) for the dictionary operand in
// each smem layout, read K-major (phase a: D[r][n] = sum_t A[r][t] B[t][n]) and MN-major from
// the same bytes (phase c: D[t][n] = sum_r A[r][t] V[r][n]).  Checks the products exactly
// (small integers) and prints cycles per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1108_5359_b200/csrc tools/umma_swizzle_rate.cu -o tools/umma_swizzle_rate.bin
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "umma.cuh"

using namespace l1f::umma;

constexpr int R = 128, T = 128, N = 96;  // dictionary rows x columns; MMA N
constexpr int NT = 128;

// mode: 0 none, 1 SW32, 2 SW64, 3 SW128 (row bytes n = 16 << mode... none uses core matrices)
__host__ __device__ inline int rowbytes(int mode) { return mode == 1 ? 32 : mode == 2 ? 64 : 128; }
__host__ __device__ inline int a_off(int mode, int r, int t) {  // byte offset of A[r][t]
  if (mode == 0) return ((r / 8) * (T / 8) + t / 8) * 128 + (r % 8) * 16 + (t % 8) * 2;
  const int n = rowbytes(mode), E = n / 2;
  const int sw = mode == 1 ? ((r % 8) >> 2) : mode == 2 ? ((r % 8) >> 1) : (r % 8);
  return (t / E) * (R * n) + (r / 8) * (8 * n) + (r % 8) * n + ((((t % E) / 8) ^ sw) * 16) + (t % 8) * 2;
}
__host__ __device__ inline int b_off(int k, int n) {  // B (K x N) MN-major, no swizzle
  return (k / 8) * (N / 8 * 128) + (n / 8) * 128 + (k % 8) * 16 + (n % 8) * 2;
}
__device__ inline uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, int mode) {
  uint64_t d = desc_noswz(addr, lbo, sbo);
  const uint64_t lt = mode == 0 ? 0 : mode == 1 ? 6 : mode == 2 ? 4 : 2;
  return d | (lt << 61);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t d, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
               ::"r"(d), "l"(da), "l"(db), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(a), "r"(parity) : "memory");
  } while (!done);
}

// phase 0: K-major read (M = r, K = t, B = Bt[t][n]); phase 1: MN-major read (M = t, K = r, B = V[r][n])
__global__ void __launch_bounds__(NT, 1) kern(const float* A, const float* B, float* D, int mode, int phase, int reps,
                                             long long* cyc) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* base = raw + (1024 - (__cvta_generic_to_shared(raw) & 1023)) % 1024;
  __nv_bfloat16* a = reinterpret_cast<__nv_bfloat16*>(base);
  __nv_bfloat16* b = reinterpret_cast<__nv_bfloat16*>(base + R * T * 2);
  __shared__ unsigned long long bar;
  __shared__ uint32_t tmem;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < R * T; e += NT) {
    const int r = e / T, t = e % T;
    a[a_off(mode, r, t) / 2] = __float2bfloat16_rn(A[e]);
  }
  for (int e = tid; e < 128 * N; e += NT) {
    const int k = e / N, n = e % N;
    b[b_off(k, n) / 2] = __float2bfloat16_rn(B[e]);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(&tmem, 128);
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t td = tmem;
  if (tid == 0) {
    const uint32_t aa = saddr(a), ba = saddr(b);
    const int n = rowbytes(mode), E = n / 2;
    uint64_t da[8], db[8];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      db[ks] = desc_noswz(ba + (uint32_t)(2 * ks) * (N / 8 * 128), N / 8 * 128, 128);
      if (phase == 0) {
        if (mode == 0) da[ks] = desc(aa + ks * 256, 128, (T / 8) * 128, 0);
        else da[ks] = desc(aa + (uint32_t)((16 * ks) / E) * (R * n) + (uint32_t)((16 * ks) % E) * 2, 16, 8 * n, mode);
      } else {
        if (mode == 0) da[ks] = desc(aa + (uint32_t)(2 * ks) * (T / 8) * 128, (T / 8) * 128, 128, 0);
        else da[ks] = desc(aa + (uint32_t)(2 * ks) * (8 * n), R * n, 8 * n, mode);
      }
    }
    const uint32_t id = idesc_bf16(128, N, phase, 1);
    fence_after();
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) mma_bf16(td, da[ks], db[ks], id, (rep | ks) != 0);
    }
    commit(&bar);
    mbar_wait(saddr(&bar), 0);
    long long t1 = clock64();
    cyc[0] = t1 - t0;
  }
  __syncthreads();
  fence_after();
  float v[16];
  for (int c = 0; c < N; c += 16) {
    ld16(td + ((uint32_t)(32 * warp) << 16) + c, v);
    ld_wait();
    for (int i = 0; i < 16; ++i) D[(32 * warp + tid % 32) * N + c + i] = v[i];
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(td, 128);
}

int main() {
  std::vector<float> A(R * T), B(128 * N);
  srand(1);
  for (auto& x : A) x = (float)(rand() % 5 - 2);
  for (auto& x : B) x = (float)(rand() % 5 - 2);
  float *dA, *dB, *dD;
  long long* dc;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, 128 * N * 4);
  cudaMalloc(&dc, 8);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = R * T * 2 + 128 * N * 2 + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[4] = {"none", "sw32", "sw64", "sw128"};
  std::vector<float> D(128 * N);
  for (int phase = 0; phase < 2; ++phase)
    for (int mode = 0; mode < 4; ++mode) {
      kern<<<1, NT, smem>>>(dA, dB, dD, mode, phase, 1, dc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
          float ref = 0.f;
          for (int k = 0; k < 128; ++k) ref += phase == 0 ? A[m * T + k] * B[k * N + n] : A[k * T + m] * B[k * N + n];
          if (ref != D[m * N + n]) ++bad;
        }
      long long best = 1LL << 62;
      for (int it = 0; it < 5; ++it) {
        kern<<<1, NT, smem>>>(dA, dB, dD, mode, phase, 64, dc);
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        if (c < best) best = c;
      }
      printf("phase %c  A %-5s %s-major: mismatches %d, %.1f cycles/MMA (M=128 N=%d K=16)\n", phase ? 'c' : 'a',
             names[mode], phase ? "MN" : "K", bad, (double)best / (64 * 8), N);
    }
  return 0;
}
