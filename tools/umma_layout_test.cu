// Microtest for the tensor-core filter's operand layouts and MMA rate (one CTA, 256 threads).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1108_5359_b200/csrc tools/umma_layout_test.cu -o /tmp/umma_test
// Phase a: D_a[row][slot] = sum_t A[row][t] Z[t][slot]   (A K-major, Z MN-major)
// Phase c: D_c[t][slot]   = sum_r A[r][t]   V[r][slot]   (A MN-major from the same bytes, V MN-major)
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "umma.cuh"

using namespace l1f::umma;

constexpr int SL = 128, KP = 112, TS = 32, KG = KP / 4;
constexpr int NTERMS = 3;

__device__ __forceinline__ int a_off(int r, int t) { return ((r / 8) * KG + t / 4) * 32 + (r % 8) * 4 + (t % 4); }
__device__ __forceinline__ int zmn_off(int s, int t) { return (s / 4) * 32 + (t / 8) * 256 + (t % 8) * 4 + (s % 4); }

struct __align__(128) Sm {
  float a_hi[SL * KP], a_lo[SL * KP];
  float z_hi[KP * TS], z_lo[KP * TS];
  float v_hi[SL * TS], v_lo[SL * TS];
  unsigned long long bar;
  uint32_t tmem;
};

__global__ void __launch_bounds__(256, 1) kern(const float* A, const float* Z, const float* V, float* Da, float* Dc,
                                                int reps, long long* cyc) {
  extern __shared__ __align__(128) unsigned char raw[];
  Sm& sm = *reinterpret_cast<Sm*>(raw);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int e = tid; e < SL * KP; e += 256) {
    const int r = e / KP, t = e % KP;
    float h, l;
    split_tf32(A[e], h, l);
    sm.a_hi[a_off(r, t)] = h;
    sm.a_lo[a_off(r, t)] = l;
  }
  for (int e = tid; e < KP * TS; e += 256) {
    const int t = e / TS, s = e % TS;
    float h, l;
    split_tf32(Z[e], h, l);
    sm.z_hi[zmn_off(s, t)] = h;
    sm.z_lo[zmn_off(s, t)] = l;
  }
  for (int e = tid; e < SL * TS; e += 256) {
    const int r = e / TS, s = e % TS;
    float h, l;
    split_tf32(V[e], h, l);
    sm.v_hi[zmn_off(s, r)] = h;
    sm.v_lo[zmn_off(s, r)] = l;
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&sm.bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(&sm.tmem, 64);
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = sm.tmem;
  constexpr uint32_t ID_A = idesc_tf32(128, TS, 0, 1), ID_C = idesc_tf32(128, TS, 1, 1);
  uint32_t phase = 0;
  long long c_a = 0, c_c = 0;
  for (int rep = 0; rep < reps; ++rep) {
    long long t0 = clock64();
    if (tid == 0) {
      const float* ap[2] = {sm.a_hi, sm.a_lo};
      const float* zp[2] = {sm.z_hi, sm.z_lo};
      const int ta[3] = {0, 0, 1}, tb[3] = {0, 1, 0};
      for (int ks = 0; ks < KP / 8; ++ks)
        for (int q = 0; q < NTERMS; ++q) {
          const uint64_t da = desc_noswz(saddr(ap[ta[q]] + (2 * ks) * 32), 128, KG * 128);
          const uint64_t db = desc_noswz(saddr(zp[tb[q]] + ks * 256), 1024, 128);
          mma_tf32(tmem, da, db, ID_A, (ks | q) != 0);
        }
      commit(&sm.bar);
    }
    {
      uint32_t done = 0;
      do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(saddr(&sm.bar)), "r"(phase) : "memory");
      } while (!done);
      phase ^= 1;
    }
    long long t1 = clock64();
    if (tid == 0) {
      const float* ap[2] = {sm.a_hi, sm.a_lo};
      const float* vp[2] = {sm.v_hi, sm.v_lo};
      const int ta[3] = {0, 0, 1}, tb[3] = {0, 1, 0};
      for (int ks = 0; ks < SL / 8; ++ks)
        for (int q = 0; q < NTERMS; ++q) {
          const uint64_t da = desc_noswz(saddr(ap[ta[q]] + ks * KG * 32), KG * 128, 128);
          const uint64_t db = desc_noswz(saddr(vp[tb[q]] + ks * 256), 1024, 128);
          mma_tf32(tmem + 32, da, db, ID_C, (ks | q) != 0);
        }
      commit(&sm.bar);
    }
    {
      uint32_t done = 0;
      do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(saddr(&sm.bar)), "r"(phase) : "memory");
      } while (!done);
      phase ^= 1;
    }
    long long t2 = clock64();
    c_a += t1 - t0;
    c_c += t2 - t1;
  }
  fence_after();
  if (warp < 4) {
    for (int h = 0; h < 2; ++h) {
      float v[16];
      ld16(tmem + ((uint32_t)(32 * warp) << 16) + 16 * h, v);
      ld_wait();
      for (int j = 0; j < 16; ++j) Da[(32 * warp + lane) * TS + 16 * h + j] = v[j];
      ld16(tmem + ((uint32_t)(32 * warp) << 16) + 32 + 16 * h, v);
      ld_wait();
      for (int j = 0; j < 16; ++j) Dc[(32 * warp + lane) * TS + 16 * h + j] = v[j];
    }
  }
  if (tid == 0) { cyc[0] = c_a; cyc[1] = c_c; }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) tmem_dealloc(tmem, 64);
}

int main() {
  std::vector<float> A(SL * KP), Z(KP * TS), V(SL * TS);
  srand(1);
  auto rnd = [] { return (float)rand() / RAND_MAX * 2.f - 1.f; };
  for (auto& x : A) x = rnd() * 0.1f;
  for (auto& x : Z) x = rnd() * 300.f;
  for (auto& x : V) x = rnd() * 20.f;
  float *dA, *dZ, *dV, *dDa, *dDc;
  long long* dc;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dZ, Z.size() * 4); cudaMalloc(&dV, V.size() * 4);
  cudaMalloc(&dDa, SL * TS * 4); cudaMalloc(&dDc, 128 * TS * 4); cudaMalloc(&dc, 16);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dZ, Z.data(), Z.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dV, V.data(), V.size() * 4, cudaMemcpyHostToDevice);
  const int smem = sizeof(Sm) + 128;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 200;
  kern<<<1, 256, smem>>>(dA, dZ, dV, dDa, dDc, reps, dc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> Da(SL * TS), Dc(128 * TS);
  long long cyc[2];
  cudaMemcpy(Da.data(), dDa, Da.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(Dc.data(), dDc, Dc.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(cyc, dc, 16, cudaMemcpyDeviceToHost);
  double ea = 0, na = 0, ec = 0, nc = 0;
  for (int r = 0; r < SL; ++r)
    for (int s = 0; s < TS; ++s) {
      double ref = 0;
      for (int t = 0; t < KP; ++t) ref += (double)A[r * KP + t] * Z[t * TS + s];
      ea += (Da[r * TS + s] - ref) * (Da[r * TS + s] - ref);
      na += ref * ref;
    }
  for (int t = 0; t < KP; ++t)
    for (int s = 0; s < TS; ++s) {
      double ref = 0;
      for (int r = 0; r < SL; ++r) ref += (double)A[r * KP + t] * V[r * TS + s];
      ec += (Dc[t * TS + s] - ref) * (Dc[t * TS + s] - ref);
      nc += ref * ref;
    }
  for (int i = 0; i < 4; ++i) {
    double ref = 0;
    for (int t = 0; t < KP; ++t) ref += (double)A[i * KP + t] * Z[t * TS + 0];
    double ref1 = 0;
    for (int t = 0; t < KP; ++t) ref1 += (double)A[0 * KP + t] * Z[t * TS + i];
    printf("Da[%d][0]=%g ref %g | Da[0][%d]=%g ref %g | Dc[%d][0]=%g\n", i, Da[i * TS], ref, i, Da[i], ref1, i, Dc[i * TS]);
  }
  printf("phase a rel err %.3e   phase c rel err %.3e\n", sqrt(ea / na), sqrt(ec / nc));
  printf("cycles per phase (incl. commit/wait): a %.0f (%d MMAs), c %.0f (%d MMAs)\n", (double)cyc[0] / reps,
         NTERMS * KP / 8, (double)cyc[1] / reps, NTERMS * SL / 8);
  return 0;
}
