// Microtest: tcgen05.mma kind::f16 with the A operand in TMEM (M = 128 lanes, K = 16 bf16 packed
// two per 32-bit column: lane m, column c = {A[m][2c], A[m][2c+1]}), B from shared memory (K-major).
#include <cstdio>
#include <vector>
#include <cuda_bf16.h>
#include "umma.cuh"
using namespace l1f::umma;
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
struct __align__(128) Sm { __nv_bfloat16 b[32 * 16]; unsigned long long bar; uint32_t tmem; };
__global__ void kern(const float* A, const float* B, float* D, int mode) {
  extern __shared__ __align__(128) unsigned char raw[];
  Sm& sm = *reinterpret_cast<Sm*>(raw);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int e = tid; e < 16 * 32; e += 128) {  // B[t][s], K-major core: 8 slots x 8 k
    const int t = e / 32, s = e % 32;
    sm.b[((s / 8) * 2 + t / 8) * 64 + (s % 8) * 8 + (t % 8)] = __float2bfloat16(B[e]);
  }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&sm.bar))); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (warp == 0) tmem_alloc(&sm.tmem, 64);
  fence_async_smem(); fence_before(); __syncthreads(); fence_after();
  const uint32_t tmem = sm.tmem;
  // A into TMEM columns [32, 40): lane = row (warp w -> lanes 32w..), column c packs k = 2c, 2c + 1
  {
    const int m = 32 * warp + lane;
    uint32_t v[8];
    for (int c = 0; c < 8; ++c) {
      const int k0 = mode == 0 ? 2 * c : c, k1 = mode == 0 ? 2 * c + 1 : c + 8;
      __nv_bfloat162 p = __floats2bfloat162_rn(A[m * 16 + k0], A[m * 16 + k1]);
      v[c] = *reinterpret_cast<uint32_t*>(&p);
    }
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 ::"r"(tmem + 32 + ((uint32_t)(32 * warp) << 16)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]),
                 "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  fence_before(); __syncthreads(); fence_after();
  if (tid == 0) {
    const uint64_t db = desc_noswz(saddr(sm.b), 128, 256);
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }"
                 ::"r"(tmem), "r"(tmem + 32), "l"(db), "r"(idesc_bf16(128, 32, 0, 0)), "r"(0u) : "memory");
    commit(&sm.bar);
  }
  uint32_t done = 0;
  do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(saddr(&sm.bar)), "r"(0) : "memory"); } while (!done);
  fence_after();
  float v[16];
  for (int h = 0; h < 2; ++h) {
    ld16(tmem + 16 * h + ((uint32_t)(32 * warp) << 16), v); ld_wait();
    for (int j = 0; j < 16; ++j) D[(32 * warp + lane) * 32 + 16 * h + j] = v[j];
  }
  fence_before(); __syncthreads(); fence_after();
  if (warp == 0) tmem_dealloc(tmem, 64);
}
int main() {
  std::vector<float> A(128 * 16), B(16 * 32), D(128 * 32);
  for (int i = 0; i < 128 * 16; ++i) A[i] = (float)((i * 7) % 13) - 6.f;
  for (int i = 0; i < 16 * 32; ++i) B[i] = (float)((i * 5) % 11) - 5.f;
  float *dA, *dB, *dD; cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 2; ++mode) {
    kern<<<1, 128, sizeof(Sm) + 128>>>(dA, dB, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 128; ++r) for (int s = 0; s < 32; ++s) {
      double ref = 0; for (int t = 0; t < 16; ++t) ref += (double)A[r * 16 + t] * B[t * 32 + s];
      if (std::abs(D[r * 32 + s] - ref) > 1e-3) ++bad;
    }
    printf("mode %d (%s): %s bad=%d D[0][0..2]=%g %g %g\n", mode, mode == 0 ? "pairs (2c,2c+1)" : "(c, c+8)", cudaGetErrorString(e), bad, D[0], D[1], D[2]);
  }
  return 0;
}
