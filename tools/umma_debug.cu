// Debug variants for the no-swizzle UMMA layouts (see umma_layout_test.cu)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "umma.cuh"
using namespace l1f::umma;
constexpr int TS = 32;
struct __align__(1024) Sm { float a[128 * 8 * 4]; float b[32 * 8 * 4]; float pad[2048]; unsigned long long bar; uint32_t tmem; };

__global__ void kern(const float* A, const float* B, float* D, int mode) {
  extern __shared__ __align__(128) unsigned char raw[];
  Sm& sm = *reinterpret_cast<Sm*>(raw);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  // A: 128 rows x 8 k, K-major no-swizzle: block (rg, kg) at (rg * 2 + kg) * 32 floats
  const bool a_mn = mode >= 5 && mode != 7;
  const bool swz = mode >= 7;
  for (int e = tid; e < 128 * 8; e += 128) {
    const int r = e / 8, t = e % 8;
    if (mode == 8) sm.a[(r / 32) * 256 + t * 32 + ((((r % 32) / 4) ^ t) * 4) + (r % 4)] = A[e];  // MN SW128
    else if (a_mn) sm.a[(r / 4) * 32 + t * 4 + (r % 4)] = A[e];  // MN-major: core 4 rows x 8 k
    else sm.a[((r / 8) * 2 + t / 4) * 32 + (r % 8) * 4 + (t % 4)] = A[e];
  }
  for (int e = tid; e < 32 * 8; e += 128) {
    const int t = e / TS, s = e % TS;  // B[t][s]
    if (mode == 7)  // MN-major SW128: row t of 128 B holds 32 slots, 16-B chunks XOR t
      sm.b[t * 32 + (((s / 4) ^ t) * 4) + (s % 4)] = B[e];
    else if (mode == 2 || mode >= 5)  // K-major: core matrix 8 slots x 4 k: block (sg, kg) at (sg * 2 + kg) * 32
      sm.b[((s / 8) * 2 + t / 4) * 32 + (s % 8) * 4 + (t % 4)] = B[e];
    else            // MN-major: core 4 slots x 8 k: block sg at sg * 32
      sm.b[(s / 4) * 32 + t * 4 + (s % 4)] = B[e];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&sm.bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(&sm.tmem, 32);
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = sm.tmem;
  if (mode == 0) {
    uint32_t v[16];
    for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(1000.f * warp + lane + 0.01f * j);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(tmem + ((uint32_t)(32 * warp) << 16)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]),
                 "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]),
                 "r"(v[14]), "r"(v[15]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  } else {
    if (tid == 0) {
      uint64_t da = desc_noswz(saddr(sm.a), 128, 256);
      if (mode == 5) da = desc_noswz(saddr(sm.a), 4096, 128);
      if (mode == 6) da = desc_noswz(saddr(sm.a), 128, 4096);
      uint64_t db = desc_noswz(saddr(sm.b), 128, 256);
      if (mode == 1) db = desc_noswz(saddr(sm.b), 1024, 128);
      if (mode == 3) db = desc_noswz(saddr(sm.b), 128, 1024);
      if (mode == 4) db = desc_noswz(saddr(sm.b), 128, 128);
      if (mode == 7) db = desc_noswz(saddr(sm.b), 1024, 1024) | ((uint64_t)2 << 61);
      if (mode == 8) da = desc_noswz(saddr(sm.a), 1024, 1024) | ((uint64_t)2 << 61);
      const int bmn = (mode == 1 || mode == 3 || mode == 4 || mode == 7);
      mma_tf32(tmem, da, db, idesc_tf32(128, TS, a_mn ? 1 : 0, bmn), 0u);
      commit(&sm.bar);
    }
    uint32_t done = 0;
    do {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(saddr(&sm.bar)), "r"(0) : "memory");
    } while (!done);
  }
  fence_after();
  float v[16];
  ld16(tmem + ((uint32_t)(32 * warp) << 16), v);
  ld_wait();
  for (int j = 0; j < 16; ++j) D[(32 * warp + lane) * TS + j] = v[j];
  ld16(tmem + ((uint32_t)(32 * warp) << 16) + 16, v);
  ld_wait();
  for (int j = 0; j < 16; ++j) D[(32 * warp + lane) * TS + 16 + j] = v[j];
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc(tmem, 32);
}

int main() {
  std::vector<float> A(128 * 8), B(8 * TS), D(128 * TS);
  for (int i = 0; i < 128 * 8; ++i) A[i] = (float)((i * 7) % 13) - 6.f;
  for (int i = 0; i < 8 * TS; ++i) B[i] = (float)((i * 5) % 11) - 5.f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Sm) + 128);
  for (int mode = 0; mode < 9; ++mode) {
    cudaMemset(dD, 0xff, D.size() * 4);
    kern<<<1, 128, sizeof(Sm) + 128>>>(dA, dB, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 128; ++r)
      for (int s = 0; s < TS; ++s) {
        double ref = 0;
        if (mode == 0) ref = (s < 16) ? 1000.0 * (r / 32) + (r % 32) + 0.01 * s : -1;
        else for (int t = 0; t < 8; ++t) ref += (double)A[r * 8 + t] * B[t * TS + s];
        if (mode == 0 && s >= 16) continue;
        if (std::abs(D[r * TS + s] - ref) > 1e-3) ++bad;
      }
    printf("mode %d: err=%s bad=%d  D[0][0..3]=%g %g %g %g  D[1][0]=%g D[8][0]=%g\n", mode, cudaGetErrorString(e), bad,
           D[0], D[1], D[2], D[3], D[TS], D[8 * TS]);
  }
  return 0;
}
