// Latency of a GPU-wide all-to-all exchange of one value per block per step (the tridiagonalisation's
// per-column wait): 148 blocks x 256 threads; per step lane 0 of warp 0 stores its slot
// (release or relaxed), warp 0 polls every block's slot, bar.sync.  Variants: release store,
// relaxed store + fence, plus optional extra per-step global stores (rowbuf-like traffic).
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
constexpr unsigned long long S = 0xffffffffffffffffull;
template <int MODE>
__global__ void __launch_bounds__(256, 1) xchg(unsigned long long* slots, int steps, double* junk, int extra, long long* out) {
  const int G = gridDim.x, b = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) {
    unsigned long long* col = slots + (size_t)i * G;
    for (int x = threadIdx.x; x < extra; x += 256) junk[(size_t)b * extra + x] = i;  // other stores before
    __syncthreads();
    if (warp == 0) {
      if (lane == 0) {
        unsigned long long v = (unsigned long long)(i + 1);
        if (MODE == 0) asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(col + b), "l"(v) : "memory");
        else { __threadfence(); asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(col + b), "l"(v) : "memory"); }
      }
      unsigned long long pv[8];
      for (int k = 0; k < 8; ++k) { pv[k] = 0; if (lane + 32 * k < G) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(pv[k]) : "l"(col + lane + 32 * k) : "memory"); }
      bool miss;
      do {
        miss = false;
        for (int k = 0; k < 8; ++k) if (lane + 32 * k < G && pv[k] == S) { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(pv[k]) : "l"(col + lane + 32 * k) : "memory"); miss |= pv[k] == S; }
      } while (__any_sync(0xffffffffu, miss));
      __threadfence();
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[b] = clock64() - t0;
}
// counter barrier: thread 0 red.release.add on one counter per step, spins with ld.acquire (MODE 2)
// or relaxed loads + fence (MODE 3); MODE 4: cooperative_groups grid.sync()
template <int MODE>
__global__ void __launch_bounds__(256, 1) ctr(unsigned* cnt, int steps, double* junk, int extra, long long* out) {
  const int G = gridDim.x, b = blockIdx.x;
  for (int i = 0; i < steps; ++i) {
    for (int x = threadIdx.x; x < extra; x += 256) junk[(size_t)b * extra + x] = i;
    if (MODE == 4) { cg::this_grid().sync(); continue; }
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt + i) : "memory");
      unsigned v;
      do {
        if (MODE == 2) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt + i) : "memory");
        else asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt + i) : "memory");
      } while (v < (unsigned)G);
      if (MODE == 3) __threadfence();
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[b] = 0;
}
int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int steps = 2000;
  unsigned long long* slots; double* junk; long long* out;
  cudaMalloc(&slots, sizeof(unsigned long long) * steps * nsm);
  cudaMalloc(&junk, sizeof(double) * nsm * 4096);
  cudaMalloc(&out, sizeof(long long) * nsm);
  for (int mode = 0; mode < 2; ++mode)
    for (int extra : {0, 16, 1024}) {
      cudaMemset(slots, 0xff, sizeof(unsigned long long) * steps * nsm);
      cudaEvent_t a, c; cudaEventCreate(&a); cudaEventCreate(&c);
      void* args[] = {&slots, (void*)&steps, &junk, &extra, &out};
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel(mode == 0 ? (void*)xchg<0> : (void*)xchg<1>, nsm, 256, args, 0, 0);
      cudaEventRecord(c); cudaEventSynchronize(c);
      float ms; cudaEventElapsedTime(&ms, a, c);
      printf("mode %s extra %4d: %.3f us per step (%s)\n", mode == 0 ? "release" : "fence+relaxed", extra, ms * 1e3 / steps, cudaGetErrorString(cudaGetLastError()));
    }
  unsigned* cnt; cudaMalloc(&cnt, sizeof(unsigned) * steps);
  for (int mode = 2; mode <= 4; ++mode)
    for (int extra : {0, 1024}) {
      cudaMemset(cnt, 0, sizeof(unsigned) * steps);
      cudaEvent_t a, c; cudaEventCreate(&a); cudaEventCreate(&c);
      void* args[] = {&cnt, (void*)&steps, &junk, &extra, &out};
      void* fn = mode == 2 ? (void*)ctr<2> : mode == 3 ? (void*)ctr<3> : (void*)ctr<4>;
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel(fn, nsm, 256, args, 0, 0);
      cudaEventRecord(c); cudaEventSynchronize(c);
      float ms; cudaEventElapsedTime(&ms, a, c);
      printf("counter mode %d extra %4d: %.3f us per step (%s)\n", mode, extra, ms * 1e3 / steps, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
