// bf16 (kind::f16) no-swizzle K-major / MN-major check, and MMA timing for small N
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_bf16.h>
#include "umma.cuh"
using namespace l1f::umma;

__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t d, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
               ::"r"(d), "l"(da), "l"(db), "r"(id), "r"(acc) : "memory");
}
// A: 128 x 16 (M x K), B: 16 x 32 (K x N)
struct __align__(1024) Sm { __nv_bfloat16 a[128 * 16]; __nv_bfloat16 b[32 * 16]; float big[16384]; unsigned long long bar; uint32_t tmem; };

__device__ void waitbar(Sm& sm, uint32_t ph) {
  uint32_t done = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(saddr(&sm.bar)), "r"(ph) : "memory");
  } while (!done);
}

template <int N, int NACC, bool BF>
__device__ __forceinline__ void issue(uint32_t tmem, uint64_t da0, uint64_t db0) {
#pragma unroll
  for (int i = 0; i < 48; ++i) {
    const uint64_t da = da0 + (uint64_t)(((i % 8) * 256) >> 4), db = db0 + (uint64_t)(((i % 8) * 256) >> 4);
    const uint32_t d = tmem + (uint32_t)((i % NACC) * N);
    if (BF) mma_bf16(d, da, db, idesc_bf16(128, N, 0, 0), i >= NACC);
    else mma_tf32(d, da, db, idesc_tf32(128, N, 0, 0), i >= NACC);
  }
}

__global__ void kern(const float* A, const float* B, float* D, int mode, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char raw[];
  Sm& sm = *reinterpret_cast<Sm*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~(uintptr_t)1023);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const bool a_mn = mode == 2, b_mn = mode == 1;
  for (int e = tid; e < 128 * 16; e += 128) {
    const int r = e / 16, t = e % 16;  // A[r][t]
    int off;
    if (a_mn) off = ((r / 8) + (t / 8) * 16) * 64 + (t % 8) * 8 + (r % 8);   // MN groups(8 rows) SBO=128B, K groups LBO=2048B
    else off = ((r / 8) * 2 + t / 8) * 64 + (r % 8) * 8 + (t % 8);            // K-major: M groups SBO=256B, K groups LBO=128B
    sm.a[off] = __float2bfloat16(A[e]);
  }
  for (int e = tid; e < 16 * 32; e += 128) {
    const int t = e / 32, s = e % 32;  // B[t][s]
    int off;
    if (b_mn) off = ((s / 8) + (t / 8) * 4) * 64 + (t % 8) * 8 + (s % 8);     // MN groups SBO=128B, K groups LBO=512B
    else off = ((s / 8) * 2 + t / 8) * 64 + (s % 8) * 8 + (t % 8);            // K-major: N groups SBO=256B, K LBO=128B
    sm.b[off] = __float2bfloat16(B[e]);
  }
  for (int e = tid; e < 16384; e += 128) sm.big[e] = 0.001f * (e % 97);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&sm.bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(&sm.tmem, 512);
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = sm.tmem;
  uint32_t ph = 0;
  if (mode <= 2) {
    if (tid == 0) {
      const uint64_t da = a_mn ? desc_noswz(saddr(sm.a), 2048, 128) : desc_noswz(saddr(sm.a), 128, 256);
      const uint64_t db = b_mn ? desc_noswz(saddr(sm.b), 512, 128) : desc_noswz(saddr(sm.b), 128, 256);
      mma_bf16(tmem, da, db, idesc_bf16(128, 32, a_mn, b_mn), 0u);
      commit(&sm.bar);
    }
    waitbar(sm, 0);
    fence_after();
    float v[16];
    for (int h = 0; h < 2; ++h) {
      ld16(tmem + ((uint32_t)(32 * warp) << 16) + 16 * h, v);
      ld_wait();
      for (int j = 0; j < 16; ++j) D[(32 * warp + lane) * 32 + 16 * h + j] = v[j];
    }
  } else {
    long long total = 0;
    const uint64_t da0 = desc_noswz(saddr(sm.big), 128, 256), db0 = desc_noswz(saddr(sm.big) + 8192, 128, 256);
    for (int rep = 0; rep < 50; ++rep) {
      long long t0 = clock64();
      if (tid == 0) {
        switch (mode) {
          case 3: issue<32, 1, false>(tmem, da0, db0); break;
          case 4: issue<64, 1, false>(tmem, da0, db0); break;
          case 5: issue<128, 1, false>(tmem, da0, db0); break;
          case 6: issue<256, 1, false>(tmem, da0, db0); break;
          case 7: issue<32, 3, false>(tmem, da0, db0); break;
          case 8: issue<32, 1, true>(tmem, da0, db0); break;
          case 9: issue<128, 1, true>(tmem, da0, db0); break;
        }
        commit(&sm.bar);
      }
      waitbar(sm, ph);
      ph ^= 1;
      total += clock64() - t0;
    }
    if (tid == 0) cyc[0] = total / 50;
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  std::vector<float> A(128 * 16), B(16 * 32), D(128 * 32);
  for (int i = 0; i < 128 * 16; ++i) A[i] = (float)((i * 7) % 13) - 6.f;
  for (int i = 0; i < 16 * 32; ++i) B[i] = (float)((i * 5) % 11) - 5.f;
  float *dA, *dB, *dD; long long* dc;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4); cudaMalloc(&dc, 8);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = sizeof(Sm) + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"bf16 K/K", "bf16 B MN", "bf16 A MN", "tf32 N32 1acc", "tf32 N64", "tf32 N128", "tf32 N256", "tf32 N32 3acc", "bf16 N32 K16", "bf16 N128 K16"};
  for (int mode = 0; mode < 10; ++mode) {
    cudaMemset(dD, 0xff, D.size() * 4);
    kern<<<1, 128, smem>>>(dA, dB, dD, mode, dc);
    cudaError_t e = cudaDeviceSynchronize();
    if (mode <= 2) {
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int r = 0; r < 128; ++r)
        for (int s = 0; s < 32; ++s) {
          double ref = 0;
          for (int t = 0; t < 16; ++t) ref += (double)A[r * 16 + t] * B[t * 32 + s];
          if (std::abs(D[r * 32 + s] - ref) > 1e-3) ++bad;
        }
      printf("%s: %s bad=%d D[0][0..2]=%g %g %g\n", names[mode], cudaGetErrorString(e), bad, D[0], D[1], D[2]);
    } else {
      long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
      printf("%s: %s  %lld cycles / 48 MMAs = %.1f per MMA\n", names[mode], cudaGetErrorString(e), c, c / 48.0);
    }
  }
  return 0;
}
