// Tensor-core reconstruction L = Af Bf^T, S = M - L (K4 for k > 16) on tcgen05.
//
// Reference: nystrom_complete + assemble + s = m - l (pkg/src/l1pcp/l1filter.py:137-167,253) in the
// unified rank-k form L[i][j] = Af[i] . Bf[j] (see l1f_build_factors).  FP32 accuracy from FP16
// tensor cores by a two-piece split: every factor row is scaled by a power of two 2^e (max |x| 2^e
// in [2^13, 2^14)), and x 2^e = h + l with h = fp16(x 2^e) and l = fp16(x 2^e - h), 22 significant
// bits in all.  L = (Ah Bh^T + Ah Bl^T + Al Bh^T) 2^-ea 2^-eb is accumulated in FP32 in TMEM (the
// dropped Al Bl^T term is ~2^-22 relative; the parity gate is 1e-4); the power-of-two scales are
// exact.  Same accuracy class as 3xTF32 at the FP16 rate (twice TF32) and half the operand bytes
// per K, so a K chunk of 32 costs what 16 did in TF32: half the MMA time and half the operand-
// pipeline round trips per tile.  The split runs once per call (split_factor_kernel).
//
// Persistent CTAs (one per SM), 12 warps (2, 3 idle):
//   warp 0      TMA producer: fp16 chunks Ah, Al (128 x 32) and Bh, Bl (128 x 32), SWIZZLE_64B, K-major
//   warp 1      TMEM allocation + MMA issuer (one thread): 6 tcgen05.mma.kind::f16 per chunk
//   warps 4-11  epilogue: tcgen05.ld (row x 16 columns per thread), scales, M via TMA, S = M - L,
//               L and S staged in shared memory and written with TMA stores
// Two 128x128 FP32 accumulators in TMEM (256 columns) overlap the MMA of tile t+1 with the
// epilogue of tile t; four operand stages overlap loads and MMAs.  Edges are handled by TMA (zero
// fill on load, clipping on store).  12 B of DRAM traffic per output entry.
#include "common.cuh"

#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

namespace l1f {
namespace rtc {

constexpr int BM = 128, BN = 128, BK = 32;      // K chunk of 32 fp16 = 64-byte rows (SWIZZLE_64B)
// pipeline depths (template parameters): operand stages (TMA -> MMA) and M buffers (prefetch
// distance NMB - 2 chunks); measured (tools/run_recon_variants.sh): 3 stages + 6 M buffers for
// k <= 128, 4 + 4 above (the operand pipeline needs the depth once K grows)
constexpr int NTHREADS = 384;
constexpr int EPI0 = 4;   // first epilogue warp
constexpr int EPI = 256;  // epilogue threads: warps 4-11, two per TMEM lane quarter (16 columns each)
constexpr uint32_t OP_BYTES = BM * BK * 2;      // 8 KB: one 128 x 32 fp16 operand box
constexpr uint32_t CHUNK_BYTES = BM * 32 * 4;   // 16 KB: one 128 x 32 fp32 epilogue box (SWIZZLE_128B)
#ifndef L1F_RTC_GROUP
#define L1F_RTC_GROUP 8
#endif
constexpr int GROUP = L1F_RTC_GROUP;            // row tiles per raster group (L2 reuse of Bf)
constexpr int kScaleExp = 14;                   // max |x| 2^e in [2^13, 2^14)

template <int STAGES, int NMB>
struct Smem {
  // every buffer is a multiple of 1024 bytes (swizzle atoms)
  uint8_t a_hi[STAGES][OP_BYTES];
  uint8_t a_lo[STAGES][OP_BYTES];
  uint8_t b_hi[STAGES][OP_BYTES];
  uint8_t b_lo[STAGES][OP_BYTES];
  uint8_t mbuf[NMB][CHUNK_BYTES];  // M chunk, overwritten in place by S before its TMA store
  uint8_t lbuf[2][CHUNK_BYTES];
  unsigned long long full[STAGES], empty[STAGES];
  unsigned long long tfull[2], tempty[2];
  unsigned long long mfull[NMB];
  alignas(16) float colscale[2][BN];  // 2^-eb of the tile's columns, by tile parity
  uint32_t tmem_base;
  double red[2][8];
};

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(void* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_arrive(void* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(void* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
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
__device__ __forceinline__ void tma_store(const CUtensorMap* map, int x, int y, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];"
               ::"l"(map), "r"(x), "r"(y), "r"(sa(src)) : "memory");
}
__device__ __forceinline__ void tma_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tma_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void tma_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// UMMA shared-memory descriptor: K-major, SWIZZLE_64B (64-byte rows), 8-row groups 512 B apart
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);   // start address
  d |= (uint64_t)1 << 16;                  // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;         // stride byte offset: 8 rows x 64 B
  d |= (uint64_t)1 << 46;                  // descriptor version (Blackwell)
  d |= (uint64_t)4 << 61;                  // SWIZZLE_64B
  return d;
}
// instruction descriptor: D f32, A/B f16, K-major both, M = 128, N = 128
constexpr uint32_t kIdesc = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
               ::"r"(tmem_d), "l"(da), "l"(db), "r"(kIdesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_commit(void* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(bar))
               : "memory");
}

struct Sched {
  int ntm, ntn, ntiles;
  __device__ void tile(int t, int& tm, int& tn) const {
    const int per_group = GROUP * ntn;
    const int g = t / per_group, r = t - g * per_group;
    const int gs = min(GROUP, ntm - g * GROUP);
    tm = g * GROUP + r % gs;
    tn = r / gs;
  }
};

template <int STAGES, int NMB>
__global__ void __launch_bounds__(NTHREADS, 1)
recon_tc_kernel(const __grid_constant__ CUtensorMap tmAh, const __grid_constant__ CUtensorMap tmAl,
                const __grid_constant__ CUtensorMap tmBh, const __grid_constant__ CUtensorMap tmBl,
                const __grid_constant__ CUtensorMap tmM, const __grid_constant__ CUtensorMap tmL,
                const __grid_constant__ CUtensorMap tmS, const float* __restrict__ inv_a,
                const float* __restrict__ inv_b, int64_t m, int64_t n, int kchunks, Sched sch, int has_m, int has_l,
                int has_s, double* __restrict__ part) {
  extern __shared__ uint8_t smem_raw[];
  constexpr int MPF = NMB - 2;
  using SmemT = Smem<STAGES, NMB>;
  SmemT& sm = *reinterpret_cast<SmemT*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&sm.full[s], 1); mbar_init(&sm.empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&sm.tfull[a], 1); mbar_init(&sm.tempty[a], EPI); }
    for (int b = 0; b < NMB; ++b) mbar_init(&sm.mfull[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // 256 TMEM columns: two 128-column FP32 accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(sa(&sm.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // ================= TMA producer
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < sch.ntiles; t += gridDim.x) {
        int tm, tn;
        sch.tile(t, tm, tn);
        for (int kc = 0; kc < kchunks; ++kc, ++it) {
          const int s = it % STAGES, ph = (it / STAGES) & 1;
          mbar_wait(&sm.empty[s], ph ^ 1);
          mbar_expect_arrive(&sm.full[s], 4 * OP_BYTES);
          tma_load(sm.a_hi[s], &tmAh, kc * BK, tm * BM, &sm.full[s]);
          tma_load(sm.b_hi[s], &tmBh, kc * BK, tn * BN, &sm.full[s]);
          tma_load(sm.a_lo[s], &tmAl, kc * BK, tm * BM, &sm.full[s]);
          tma_load(sm.b_lo[s], &tmBl, kc * BK, tn * BN, &sm.full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer
    int it = 0, ti = 0;
    for (int t = blockIdx.x; t < sch.ntiles; t += gridDim.x, ++ti) {
      const int acc = ti & 1, aph = (ti >> 1) & 1;
      mbar_wait(&sm.tempty[acc], aph ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t d = tmem + (uint32_t)(acc * BN);
      for (int kc = 0; kc < kchunks; ++kc, ++it) {
        const int s = it % STAGES, ph = (it / STAGES) & 1;
        mbar_wait(&sm.full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (lane == 0) {
          const uint32_t ah = sa(sm.a_hi[s]), bh = sa(sm.b_hi[s]), al = sa(sm.a_lo[s]), bl = sa(sm.b_lo[s]);
#pragma unroll
          for (int j = 0; j < BK / 16; ++j) {
            const uint32_t off = 32u * j;  // 16 fp16 = 32 bytes along K inside the 64-byte swizzle atom
            mma_f16(d, smem_desc(ah + off), smem_desc(bh + off), (kc | j) ? 1u : 0u);
            mma_f16(d, smem_desc(ah + off), smem_desc(bl + off), 1u);
            mma_f16(d, smem_desc(al + off), smem_desc(bh + off), 1u);
          }
          mma_commit(&sm.empty[s]);                         // stage free when these MMAs retire
          if (kc == kchunks - 1) mma_commit(&sm.tfull[acc]);  // accumulator ready
        }
        __syncwarp();
      }
    }
  } else if (warp >= EPI0) {
    // ================= epilogue (256 threads, TMEM lane quarter = warp % 4)
    const int ew = warp - EPI0, q = warp & 3, half = ew >> 2;
    const int row = 32 * q + lane;  // row of the tile owned by this thread (columns half * 16 .. + 16)
    const bool leader = threadIdx.x == 32 * EPI0;
    double r2 = 0.0, m2 = 0.0;
    int ti = 0, g = 0;
    // chunk g -> (tile, column chunk); prefetch M of chunk g+1 while g is processed
    auto chunk_coords = [&](int gg, int& x, int& y) -> bool {
      const int tloc = gg / (BN / 32), cc = gg % (BN / 32);
      const int t = blockIdx.x + tloc * gridDim.x;
      if (t >= sch.ntiles) return false;
      int tm, tn;
      sch.tile(t, tm, tn);
      x = tn * BN + cc * 32;
      y = tm * BM;
      return true;
    };
    if (leader && has_m) {  // M of the first chunks
      for (int gg = 0; gg < MPF; ++gg) {
        int x, y;
        if (chunk_coords(gg, x, y)) {
          mbar_expect_arrive(&sm.mfull[gg], CHUNK_BYTES);
          tma_load(sm.mbuf[gg], &tmM, x, y, &sm.mfull[gg]);
        }
      }
    }
    for (int t = blockIdx.x; t < sch.ntiles; t += gridDim.x, ++ti) {
      int tm, tn;
      sch.tile(t, tm, tn);
      const int acc = ti & 1, aph = (ti >> 1) & 1;
      const int64_t gi = (int64_t)tm * BM + row;
      const float sca = gi < m ? inv_a[gi] : 0.f;  // 2^-ea of this row
      {
        const int et = threadIdx.x - 32 * EPI0;
        const int64_t gj = (int64_t)tn * BN + et;
        if (et < BN) sm.colscale[ti & 1][et] = gj < n ? inv_b[gj] : 0.f;  // read after the next named barrier
      }
      mbar_wait(&sm.tfull[acc], aph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int cc = 0; cc < BN / 32; ++cc, ++g) {
        const int mb = g % NMB, lb = g & 1;
        uint32_t v[16];
        const uint32_t taddr = tmem + (uint32_t)(acc * BN + cc * 32 + 16 * half) + ((uint32_t)(32 * q) << 16);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (cc == BN / 32 - 1) {  // accumulator fully read: release it to the MMA warp
          asm volatile("tcgen05.fence::before_thread_sync;");
          mbar_arrive(&sm.tempty[acc]);
        }
        if (leader) {
          // stores of chunk g-2 (lbuf[lb], its M buffer) have finished reading shared memory
          tma_wait_read1();
          if (has_m) {  // prefetch M of chunk g+MPF into the buffer freed above
            int x, y;
            if (chunk_coords(g + MPF, x, y)) {
              const int nb = (g + MPF) % NMB;
              mbar_expect_arrive(&sm.mfull[nb], CHUNK_BYTES);
              tma_load(sm.mbuf[nb], &tmM, x, y, &sm.mfull[nb]);
            }
          }
        }
        if (has_m) mbar_wait(&sm.mfull[mb], (g / NMB) & 1);
        named_bar(1, EPI);
        // 16-byte chunk j of this row sits at position j ^ (row & 7) (SWIZZLE_128B)
        float4* mrow = reinterpret_cast<float4*>(sm.mbuf[mb] + row * 128);
        float4* lrow = reinterpret_cast<float4*>(sm.lbuf[lb] + row * 128);
        // sum(M^2) of this row's 32 entries in FP32, folded into the double once per chunk; the
        // residual partial of (M - L) - S is identically 0 (S is stored as the fp32 M - L)
        float macc = 0.f;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = 4 * half + jj, p = j ^ (row & 7);
          const float4 c4 = *reinterpret_cast<const float4*>(&sm.colscale[ti & 1][cc * 32 + 4 * j]);
          const float4 l4 = make_float4(__uint_as_float(v[4 * jj]) * sca * c4.x,
                                        __uint_as_float(v[4 * jj + 1]) * sca * c4.y,
                                        __uint_as_float(v[4 * jj + 2]) * sca * c4.z,
                                        __uint_as_float(v[4 * jj + 3]) * sca * c4.w);
          if (has_l) lrow[p] = l4;
          if (has_m) {
            const float4 m4 = mrow[p];
            mrow[p] = make_float4(m4.x - l4.x, m4.y - l4.y, m4.z - l4.z, m4.w - l4.w);  // S in place of M
            macc = fmaf(m4.x, m4.x, fmaf(m4.y, m4.y, fmaf(m4.z, m4.z, fmaf(m4.w, m4.w, macc))));
          }
        }
        m2 += (double)macc;
        fence_async_smem();
        named_bar(1, EPI);
        if (leader) {
          const int x = tn * BN + cc * 32, y = tm * BM;
          if (has_l) tma_store(&tmL, x, y, sm.lbuf[lb]);
          if (has_s && has_m) tma_store(&tmS, x, y, sm.mbuf[mb]);
          tma_commit();
        }
      }
    }
    if (leader) tma_wait_all();
    // per-CTA residual partials (deterministic)
    r2 = warp_sum(r2);
    m2 = warp_sum(m2);
    if (lane == 0) { sm.red[0][ew] = r2; sm.red[1][ew] = m2; }
    named_bar(1, EPI);
    if (leader && part) {
      double a = 0, c = 0;
      for (int i = 0; i < 8; ++i) { a += sm.red[0][i]; c += sm.red[1][i]; }
      part[2 * blockIdx.x] = a;
      part[2 * blockIdx.x + 1] = c;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

// two-piece FP16 split of a rows x k factor into rows x kp (kp % 32 == 0, zero padded): one warp
// per row; x 2^e = h + l with max |x| 2^e in [2^13, 2^14), inv[row] = 2^-e (1 for a zero row)
__global__ void split_factor_kernel(const float* __restrict__ src, int64_t rows, int k, int64_t lds, int kp,
                                    __half* __restrict__ hi, __half* __restrict__ lo, float* __restrict__ inv) {
  const int lane = threadIdx.x % 32;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
    const float* x = src + r * lds;
    float mx = 0.f;
    for (int t = lane; t < k; t += 32) mx = fmaxf(mx, fabsf(x[t]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int ex = 0;
    if (mx > 0.f) frexpf(mx, &ex);  // mx = f 2^ex, f in [0.5, 1)
    const int e = mx > 0.f ? kScaleExp - ex : 0;
    for (int t = lane; t < kp; t += 32) {
      const float v = t < k ? ldexpf(x[t], e) : 0.f;
      const __half h = __float2half_rn(v);
      hi[r * kp + t] = h;
      lo[r * kp + t] = __float2half_rn(v - __half2float(h));
    }
    if (lane == 0) inv[r] = ldexpf(1.f, -e);
  }
}

__global__ void sum_parts_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double a = 0, b = 0;
    for (int i = 0; i < n; ++i) { a += part[2 * i]; b += part[2 * i + 1]; }
    out[0] = a;
    out[1] = b;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2D fp32 (or fp16) tensor (rows x cols, row pitch ld elements), box_cols x 128 boxes
static bool make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_cols,
                     CUtensorMapSwizzle swz, bool f16 = false) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * (f16 ? 2 : 4))};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, 128};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace rtc
}  // namespace l1f

// tcgen05 path of l1f_reconstruct for float, k > 16; returns L1F_ERR_UNSUPPORTED when it cannot run
int l1f_reconstruct_tc(int64_t m, int64_t n, int k, const float* Af, int64_t ldaf, const float* Bf, int64_t ldbf,
                       const float* M, int64_t ldm, float* L, int64_t ldl, float* S, int64_t lds, double* resid_sq,
                       cudaStream_t st) {
  using namespace l1f;
  using namespace l1f::rtc;
  const char* env = getenv("L1F_RECON_TC");
  if (env && env[0] == '0') return L1F_ERR_UNSUPPORTED;
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  if ((M && (!al16(M) || ldm % 4)) || (L && (!al16(L) || ldl % 4)) || (S && (!al16(S) || lds % 4)))
    return L1F_ERR_UNSUPPORTED;
  if (m >= INT32_MAX || n >= INT32_MAX || !encode_fn()) return L1F_ERR_UNSUPPORTED;
  const int kp = (int)ceil_div(k, BK) * BK;
  __half *ah = nullptr, *al = nullptr, *bh = nullptr, *bl = nullptr;
  float *ia = nullptr, *ib = nullptr;
  double* part = nullptr;
  const int grid = num_sms();
  L1F_CUDA_TRY(cudaMallocAsync(&ah, sizeof(__half) * (size_t)m * kp * 2, st));
  L1F_CUDA_TRY(cudaMallocAsync(&bh, sizeof(__half) * (size_t)n * kp * 2, st));
  const int64_t m4 = ceil_div(m, 4) * 4;  // inv_b 16-byte aligned (float4 loads)
  L1F_CUDA_TRY(cudaMallocAsync(&ia, sizeof(float) * (size_t)(m4 + n), st));
  L1F_CUDA_TRY(cudaMallocAsync(&part, sizeof(double) * 2 * grid, st));
  al = ah + (size_t)m * kp;
  bl = bh + (size_t)n * kp;
  ib = ia + m4;
  split_factor_kernel<<<grid * 4, 256, 0, st>>>(Af, m, k, ldaf, kp, ah, al, ia);
  split_factor_kernel<<<grid * 4, 256, 0, st>>>(Bf, n, k, ldbf, kp, bh, bl, ib);
  CUtensorMap tAh, tAl, tBh, tBl, tM, tL, tS;
  const auto W = CU_TENSOR_MAP_SWIZZLE_128B, W64 = CU_TENSOR_MAP_SWIZZLE_64B;
  bool ok = make_map(&tAh, ah, m, kp, kp, BK, W64, true) && make_map(&tAl, al, m, kp, kp, BK, W64, true) &&
            make_map(&tBh, bh, n, kp, kp, BK, W64, true) && make_map(&tBl, bl, n, kp, kp, BK, W64, true);
  const void* dummy = ia;  // any 16-byte aligned device pointer for unused maps
  ok = ok && make_map(&tM, M ? (const void*)M : dummy, M ? m : 1, M ? n : 32, M ? ldm : 32, 32, W);
  ok = ok && make_map(&tL, L ? (const void*)L : dummy, L ? m : 1, L ? n : 32, L ? ldl : 32, 32, W);
  ok = ok && make_map(&tS, S ? (const void*)S : dummy, S ? m : 1, S ? n : 32, S ? lds : 32, 32, W);
  int rc = L1F_OK;
  if (!ok) {
    set_error("reconstruct: cuTensorMapEncodeTiled failed");
    rc = L1F_ERR_UNSUPPORTED;
  } else {
    Sched sch;
    sch.ntm = (int)ceil_div(m, BM);
    sch.ntn = (int)ceil_div(n, BN);
    sch.ntiles = sch.ntm * sch.ntn;
    const int g = std::min(grid, sch.ntiles);
    // L1F_RECON_TC_MASK (diagnostics): bit 0 drops M, bit 1 drops L, bit 2 drops S
    const char* mk = getenv("L1F_RECON_TC_MASK");
    const int mask = mk ? atoi(mk) : 0;
    static bool attr_set[2] = {false, false};
    auto run = [&](auto kern, size_t smem, int which) {
      if (!attr_set[which]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_set[which] = true;
      }
      kern<<<g, NTHREADS, smem, st>>>(tAh, tAl, tBh, tBl, tM, tL, tS, ia, ib, m, n, kp / BK, sch,
                                      M != nullptr && !(mask & 1), L != nullptr && !(mask & 2),
                                      S != nullptr && !(mask & 4), part);
    };
    if (kp <= 128) run(recon_tc_kernel<3, 6>, sizeof(Smem<3, 6>) + 1024, 0);
    else run(recon_tc_kernel<4, 4>, sizeof(Smem<4, 4>) + 1024, 1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      set_error("reconstruct (tcgen05): launch failed: %s", cudaGetErrorString(e));
      rc = L1F_ERR_CUDA;
    } else if (resid_sq && M) {
      sum_parts_kernel<<<1, 32, 0, st>>>(part, g, resid_sq);
    }
  }
  cudaFreeAsync(ah, st);
  cudaFreeAsync(bh, st);
  cudaFreeAsync(ia, st);
  cudaFreeAsync(part, st);
  return rc;
}
