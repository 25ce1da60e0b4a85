// TMA read-rate probe for the reconstruction's M stream: 148 persistent CTAs walk 128 x 128 fp32
// tiles of a rows x cols matrix (same raster as recon_tc), loading each tile as four 32-column
// boxes (SWIZZLE_128B) through a ring of NB buffers with a prefetch distance of NB - 2 boxes;
// one thread consumes (touches) each box.  Variants: box rows, L2 promotion, boxes per issue.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/tma_read_rate.cu -o tools/tma_read_rate.bin -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(void* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(void* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(void* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(sa(b)), "r"(parity) : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* map, int x, int y, void* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(sa(dst)), "l"(map), "r"(x), "r"(y), "r"(sa(bar)) : "memory");
}

constexpr int NB = 8;
__global__ void __launch_bounds__(128, 1) stream(const __grid_constant__ CUtensorMap tm, int ntm, int ntn, int brows,
                                               float* sink) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* buf = raw + (1024 - (sa(raw) & 1023)) % 1024;
  __shared__ unsigned long long full[NB];
  const uint32_t box_bytes = 32 * 4 * brows;
  const int sub = 128 / brows;  // boxes per 32-column chunk
  if (threadIdx.x == 0) {
    for (int i = 0; i < NB; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int ntiles = ntm * ntn;
  const int per_cta = (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int nboxes = per_cta * 4 * sub;
  auto coords = [&](int b, int& x, int& y) {
    const int tl = b / (4 * sub), rem = b % (4 * sub), cc = rem / sub, sr = rem % sub;
    const int t = blockIdx.x + tl * gridDim.x;
    const int per_group = 8 * ntn, gq = t / per_group, r = t % per_group;
    const int gs = min(8, ntm - gq * 8);
    const int tmi = gq * 8 + r % gs, tni = r / gs;
    x = tni * 128 + cc * 32;
    y = tmi * 128 + sr * brows;
  };
  const int pf = NB - 2;
  for (int b = 0; b < pf && b < nboxes; ++b) {
    int x, y;
    coords(b, x, y);
    mbar_expect(&full[b % NB], box_bytes);
    tma_load(buf + (size_t)(b % NB) * box_bytes, &tm, x, y, &full[b % NB]);
  }
  float acc = 0.f;
  for (int b = 0; b < nboxes; ++b) {
    if (b + pf < nboxes) {
      int x, y;
      coords(b + pf, x, y);
      const int s = (b + pf) % NB;
      mbar_expect(&full[s], box_bytes);
      tma_load(buf + (size_t)s * box_bytes, &tm, x, y, &full[s]);
    }
    mbar_wait(&full[b % NB], (b / NB) & 1);
    acc += reinterpret_cast<const float*>(buf + (size_t)(b % NB) * box_bytes)[0];
  }
  if (acc == 12345.f) sink[0] = acc;
}

// L2-resident stream: every CTA loads boxes of bw fp32 columns x 128 rows from a small matrix
__global__ void __launch_bounds__(128, 1) stream_l2(const __grid_constant__ CUtensorMap tm, int rows, int cols, int bw,
                                                  int nboxes, float* sink) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* buf = raw + (1024 - (sa(raw) & 1023)) % 1024;
  __shared__ unsigned long long full[NB];
  const uint32_t box_bytes = bw * 4 * 128;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NB; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int nx = cols / bw, ny = rows / 128;
  auto coords = [&](int b, int& x, int& y) {
    const int q = (b + (int)blockIdx.x * 7) % (nx * ny);
    x = (q % nx) * bw;
    y = (q / nx) * 128;
  };
  const int pf = NB - 2;
  for (int b = 0; b < pf; ++b) {
    int x, y;
    coords(b, x, y);
    mbar_expect(&full[b % NB], box_bytes);
    tma_load(buf + (size_t)(b % NB) * box_bytes, &tm, x, y, &full[b % NB]);
  }
  float acc = 0.f;
  for (int b = 0; b < nboxes; ++b) {
    if (b + pf < nboxes) {
      int x, y;
      coords(b + pf, x, y);
      const int s = (b + pf) % NB;
      mbar_expect(&full[s], box_bytes);
      tma_load(buf + (size_t)s * box_bytes, &tm, x, y, &full[s]);
    }
    mbar_wait(&full[b % NB], (b / NB) & 1);
    acc += reinterpret_cast<const float*>(buf + (size_t)(b % NB) * box_bytes)[0];
  }
  if (acc == 12345.f) sink[0] = acc;
}

int main() {
  const int rows = 20000, cols = 20000;
  float* M;
  cudaMalloc(&M, sizeof(float) * (size_t)rows * cols);
  cudaMemset(M, 0, sizeof(float) * (size_t)rows * cols);
  float* sink;
  cudaMalloc(&sink, 4);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int ntm = (rows + 127) / 128, ntn = (cols + 127) / 128;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const CUtensorMapL2promotion promos[3] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
  const char* pn[3] = {"none", "128B", "256B"};
  for (int brows : {128, 64, 32})
    for (int p = 0; p < 3; ++p) {
      CUtensorMap tm;
      cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
      cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
      cuuint32_t box[2] = {32, (cuuint32_t)brows};
      cuuint32_t es[2] = {1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, M, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, promos[p], CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const int smem = NB * 32 * 4 * brows + 1024;
      cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(a);
        stream<<<sms, 128, smem>>>(tm, ntm, ntn, brows, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep && ms < best) best = ms;
      }
      const cudaError_t e = cudaGetLastError();
      printf("box 32 x %3d, L2 promotion %-4s, %d buffers (prefetch %d): %.3f ms, %.0f GB/s %s\n", brows, pn[p], NB,
             NB - 2, best, (double)rows * cols * 4 / best / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  {  // L2-resident operand stream (4096 x 128 fp32 = 2 MB)
    const int r2 = 4096, c2 = 128;
    for (int bw : {16, 32}) {
      CUtensorMap tm;
      cuuint64_t dims[2] = {(cuuint64_t)c2, (cuuint64_t)r2};
      cuuint64_t strides[1] = {(cuuint64_t)c2 * 4};
      cuuint32_t box[2] = {(cuuint32_t)bw, 128};
      cuuint32_t es[2] = {1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, M, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          bw == 16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const int smem = NB * bw * 4 * 128 + 1024;
      cudaFuncSetAttribute(stream_l2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      const int nboxes = (int)((64ll << 20) / (bw * 4 * 128));  // 64 MB per CTA
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        stream_l2<<<sms, 128, smem>>>(tm, r2, c2, bw, nboxes, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep && ms < best) best = ms;
      }
      const double bytes = (double)nboxes * bw * 4 * 128;
      printf("L2-resident boxes of %d fp32 x 128 rows (%d-byte rows): %.1f GB/s per SM, %.1f B/cycle at 1.965 GHz\n",
             bw, bw * 4, bytes / best / 1e6, bytes / (best * 1e-3) / 1.965e9);
    }
  }
  return 0;
}
