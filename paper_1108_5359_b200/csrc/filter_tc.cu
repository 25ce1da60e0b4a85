// Tensor-core ADM filter (K3 v3): the resident-state cluster kernel of filter_resident.cu with both
// contractions of every ADM iteration on tcgen05.
//
// Reference: _solve_block, pkg/src/l1pcp/l1reg.py:59-137 (per-unit ADM for min ||x - A z||_1).
// Per pass (one ADM iteration of the 32 unit slots of a cluster) a CTA owning SL = 128 dictionary
// rows computes
//   phase a   az[row][slot]  = sum_t A[row][t] z[t][slot]     tcgen05.mma M=128 (rows) N=32 K=k
//   phase b   the elementwise ADM update of filter_resident.cu (cancellation-free residual)
//   phase c   zp[t][slot]    = sum_row A[row][t] v[row][slot]  tcgen05.mma M=128 (t)    N=32 K=128
// and the cluster sums zp over its CTAs through DSMEM as in filter_resident.cu.
//
// FP32 accuracy from BF16 tensor cores: every operand is split into three bf16 pieces
// x = x0 + x1 + x2 (each the bf16 rounding of the remainder; 24 significant bits) and the
// products with i + j <= 2 are accumulated in FP32 in TMEM (6 MMAs per K step; the dropped terms
// are ~2^-26 relative).  bf16 because tcgen05 reads bf16 operands in MN-major layout (TF32 only
// K-major): the dictionary's no-swizzle core matrices (8 rows x 8 columns, 16-byte rows) are
// K-major for phase a (M = rows) and MN-major for phase c (M = columns), so ONE resident copy of A
// (3 pieces, 6 B per element) serves both contractions.
//
// Roles: warp 1 (one thread) issues the MMAs; warp 0 takes the per-slot decisions while phase a runs;
// all 16 warps do phase b (warp w: TMEM lanes 32 (w % 4) .. +31 = rows, slots 8 (w / 4) .. +7).
#include "common.cuh"
#include "umma.cuh"

#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace l1f {
namespace tcf {

constexpr int TS = 32;        // unit slots per cluster (MMA N)
constexpr int SL = 128;       // dictionary rows per CTA (MMA M of phase a)
constexpr int NT = 512;       // threads per CTA (4 warps per TMEM lane quarter)
constexpr int TSP = TS + 4;   // padded fp32 z row (conflict-free TMEM -> smem stores)
constexpr int RING = 4;
constexpr int kStallIters = 20;      // STAGNATION_ITERS, l1reg.py:34
constexpr float kStallEps = 1e-12f;  // STAGNATION_EPS, l1reg.py:33
constexpr uint32_t TMEM_COLS = 64;   // phase a: cols [0, 32); phase c: cols [32, 64)

struct Params {
  int s, k, cluster, rs;
  int64_t n_units, ldx, ldz, lde;
  int max_iter;
  double tol, rho, beta0, beta_max;
};

struct Slots {
  int unit[TS], it[TS], stalled[TS], state[TS], finish[TS], src[TS];
  float beta_cur[TS], beta_next[TS], inv_next[TS], beta_max[TS], thresh[TS], prev_res[TS], res[TS];
  float ring_sc[RING];
  long long ring_u[RING];
  long long head, tail, pf_from, pf_to;
  alignas(16) float4 prm[TS];  // phase-b parameters per slot: beta_it, 1/beta_{it+1}, zero-az flag
  alignas(8) unsigned long long bar_p, bar_r, bar_a, bar_c;
  uint32_t tmem, fmask;
  uint8_t code[TS];
};

template <int KP>
struct Geo {
  static constexpr int KG = KP / 8;                         // 8-column groups of A
  static constexpr int KZ = KP + 16;                        // fp32 z rows (room for C * ceil(KP / C))
  static constexpr size_t a_piece = (size_t)SL * KP;       // bf16 elements per piece
  static constexpr size_t z_piece = (size_t)KP * TS;
  static constexpr size_t v_piece = (size_t)SL * TS;
  // bf16 operands first (their MMA over-reads past the last piece land in bf16 data), then fp32
  static constexpr size_t off_a = 0;
  static constexpr size_t off_z = off_a + 3 * a_piece * 2;
  static constexpr size_t off_v = off_z + 3 * z_piece * 2;
  static constexpr size_t off_z0 = off_v + 3 * v_piece * 2;       // fp32 z ping
  static constexpr size_t off_z1 = off_z0 + (size_t)KZ * TSP * 4;  // fp32 z pong
  static constexpr size_t off_zin = off_z1 + (size_t)KZ * TSP * 4; // peers' partials of my slice
  static constexpr size_t off_rpart = off_zin + (size_t)KZ * TSP * 4;
  static constexpr size_t off_ring = off_rpart + (size_t)4 * TS * 4;
  static constexpr size_t off_rall = off_ring + (size_t)RING * SL * 4;
  static constexpr size_t smem_bytes = off_rall + (size_t)16 * TS * 4;
  static_assert(KP % 16 == 0 && KP <= 128, "KP: multiple of 16, at most 128 (one phase-c M tile)");
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t peer_addr(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(void* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(umma::saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(void* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(umma::saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(void* bar, uint32_t parity) {
  const uint32_t a = umma::saddr(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(a), "r"(parity) : "memory");
  } while (!done);
}
__device__ __forceinline__ void st_async16(uint32_t peer_dst, const void* src16, uint32_t peer_bar) {
  const uint4 v = *reinterpret_cast<const uint4*>(src16);
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
               ::"r"(peer_dst), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(peer_bar) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const float* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(umma::saddr(dst)), "l"(src), "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t d, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
               ::"r"(d), "l"(da), "l"(db), "r"(id), "r"(acc) : "memory");
}

// x = p0 + p1 + p2, each the bf16 rounding of the remaining part
__device__ __forceinline__ void split3(float x, __nv_bfloat16& p0, __nv_bfloat16& p1, __nv_bfloat16& p2) {
  p0 = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(p0);
  p1 = __float2bfloat16_rn(r1);
  p2 = __float2bfloat16_rn(r1 - __bfloat162float(p1));
}
__device__ __forceinline__ uint32_t pack2(__nv_bfloat16 lo, __nv_bfloat16 hi) {
  return (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
}
// 8 consecutive fp32 -> three 16-byte rows of bf16 pieces
__device__ __forceinline__ void split8_store(const float (&v)[8], __nv_bfloat16* d0, __nv_bfloat16* d1,
                                             __nv_bfloat16* d2) {
  uint32_t w0[4], w1[4], w2[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat16 a0, a1, a2, b0, b1, b2;
    split3(v[2 * i], a0, a1, a2);
    split3(v[2 * i + 1], b0, b1, b2);
    w0[i] = pack2(a0, b0);
    w1[i] = pack2(a1, b1);
    w2[i] = pack2(a2, b2);
  }
  *reinterpret_cast<uint4*>(d0) = make_uint4(w0[0], w0[1], w0[2], w0[3]);
  *reinterpret_cast<uint4*>(d1) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
  *reinterpret_cast<uint4*>(d2) = make_uint4(w2[0], w2[1], w2[2], w2[3]);
}

// products (i, j) of the 3-piece split kept: i + j <= 2
__host__ __device__ constexpr int term_a(int t) { return t == 2 || t == 4 ? 1 : t == 5 ? 2 : 0; }
__host__ __device__ constexpr int term_b(int t) { return t == 1 || t == 4 ? 1 : t == 3 ? 2 : 0; }

template <int KP>
__global__ void __launch_bounds__(NT, 1)
adm_tc_kernel(const float* __restrict__ X, const float* __restrict__ A, int64_t lda, const float* __restrict__ scale,
              Params P, float* __restrict__ Z, float* __restrict__ E, int32_t* __restrict__ iters,
              float* __restrict__ res_out, uint8_t* __restrict__ status, long long* __restrict__ prof) {
  using Gm = Geo<KP>;
  constexpr int KG = Gm::KG;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __nv_bfloat16* aop = reinterpret_cast<__nv_bfloat16*>(smem_raw + Gm::off_a);  // [3][SL*KP]
  __nv_bfloat16* zop = reinterpret_cast<__nv_bfloat16*>(smem_raw + Gm::off_z);  // [3][KP*TS]
  __nv_bfloat16* vop = reinterpret_cast<__nv_bfloat16*>(smem_raw + Gm::off_v);  // [3][SL*TS]
  float* zbuf0 = reinterpret_cast<float*>(smem_raw + Gm::off_z0);               // [KZ][TSP]
  float* zbuf1 = reinterpret_cast<float*>(smem_raw + Gm::off_z1);
  float* zin = reinterpret_cast<float*>(smem_raw + Gm::off_zin);
  float* rpart = reinterpret_cast<float*>(smem_raw + Gm::off_rpart);            // [4][TS]
  float* ring_x = reinterpret_cast<float*>(smem_raw + Gm::off_ring);            // [RING][SL]
  float* rall = reinterpret_cast<float*>(smem_raw + Gm::off_rall);              // [16][TS]
  __shared__ Slots ss;

  cg::cluster_group cluster = cg::this_cluster();
  const int C = P.cluster;
  const int crank = C > 1 ? (int)cluster.block_rank() : 0;
  const int cid = blockIdx.x / C, nclusters = gridDim.x / C;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int row_base = crank * SL;
  const float tol = (float)P.tol, rho = (float)P.rho;
  const int rs = P.rs;  // rows of z reduced by each CTA

  // ---- resident dictionary rows, 3 bf16 pieces: core matrix (row group rg, column group cg) at
  //      (rg * KG + cg) * 64 elements, element (r % 8) * 8 + (t % 8)
  for (int e = tid; e < SL * KP; e += NT) {
    const int r = e / KP, t = e - r * KP;
    const int row = row_base + r;
    const float a = (row < P.s && t < P.k) ? A[(int64_t)row * lda + t] : 0.f;
    __nv_bfloat16 p0, p1, p2;
    split3(a, p0, p1, p2);
    const size_t off = (size_t)((r >> 3) * KG + (t >> 3)) * 64 + (r & 7) * 8 + (t & 7);
    aop[off] = p0;
    aop[Gm::a_piece + off] = p1;
    aop[2 * Gm::a_piece + off] = p2;
  }
  for (int e = tid; e < (int)(3 * Gm::z_piece); e += NT) zop[e] = __float2bfloat16_rn(0.f);

  // phase b mapping: TMEM lane quarter q (rows 32q .. 32q+31), slots [8 h, 8 h + 8)
  const int q = warp & 3, h = warp >> 2;
  const int lrow = 32 * q + lane;
  const int grow = row_base + lrow;
  const int slot0 = 8 * h;

  float xr[8], yr[8], lr[8];

  auto cand = [&](long long j) -> long long { return (long long)cid + j * (long long)nclusters; };
  auto prefetch = [&]() {
    for (long long j = ss.pf_from; j < ss.pf_to; ++j) {
      const int e = (int)(j % RING);
      const long long u = cand(j);
      const bool ok = u < P.n_units;
      for (int r = tid; r < SL; r += NT)
        cp_async4(ring_x + (size_t)e * SL + r, X + (ok ? u : 0) * P.ldx + (ok && row_base + r < P.s ? row_base + r : 0),
                  ok && row_base + r < P.s);
      if (tid == 0) {
        ss.ring_u[e] = u;
        cp_async4(&ss.ring_sc[e], scale + (ok ? u : 0), ok);
      }
    }
  };
  auto install_unit = [&](int slot, long long u, float sc, int src) {
    const float b0 = P.beta0 > 0 ? (float)P.beta0 : 1.f / sc;
    ss.unit[slot] = (int)u;
    ss.state[slot] = 1;
    ss.it[slot] = 0;
    ss.stalled[slot] = 0;
    ss.src[slot] = src;
    ss.beta_cur[slot] = b0;
    ss.beta_next[slot] = b0;
    ss.inv_next[slot] = 1.f / b0;
    ss.beta_max[slot] = P.beta_max > 0 ? (float)P.beta_max : 1e7f * b0;
    ss.thresh[slot] = tol * sc;
    ss.prev_res[slot] = Limits<float>::inf();
  };
  auto claim_into = [&](int slot) {
    for (;;) {
      if (ss.head < ss.tail) {
        const int e = (int)(ss.head % RING);
        const long long u = ss.ring_u[e];
        ss.head++;
        if (u >= P.n_units) break;
        if (ss.ring_sc[e] > 0.f) { install_unit(slot, u, ss.ring_sc[e], e); return; }
      } else {
        const long long u = cand(ss.head);
        ss.head++;
        ss.tail = ss.head;
        if (u >= P.n_units) break;
        const float sc = scale[u];
        if (sc > 0.f) { install_unit(slot, u, sc, -1); return; }
      }
    }
    ss.state[slot] = 0;
    ss.unit[slot] = -1;
  };
  // warp 0, lane = slot: phase-b parameters of this pass (after the decision and the claims)
  auto publish = [&](int slot) {
    const bool live = ss.state[slot] == 1;
    const bool zero_az = !live || ss.it[slot] == 0;  // fresh or empty slot: A z_0 = 0
    ss.prm[slot] = live ? make_float4(ss.beta_cur[slot], ss.inv_next[slot], zero_az ? 1.f : 0.f, 0.f)
                        : make_float4(0.f, 0.f, 1.f, 0.f);
  };
  auto load_slot = [&](int j) {
    const int slot = slot0 + j;
    const bool live = ss.state[slot] == 1;
    const int src = ss.src[slot];
    const int64_t u = live ? ss.unit[slot] : 0;
    float x = 0.f;
    if (live && grow < P.s) x = src >= 0 ? ring_x[(size_t)src * SL + lrow] : X[u * P.ldx + grow];
    xr[j] = x;
    yr[j] = 0.f;
    lr[j] = 0.f;
  };

  if (tid == 0) {
    ss.head = 0; ss.tail = 0; ss.pf_from = 0; ss.pf_to = RING;
    mbar_init(&ss.bar_p, 1);
    mbar_init(&ss.bar_r, 1);
    mbar_init(&ss.bar_a, 1);
    mbar_init(&ss.bar_c, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) umma::tmem_alloc(&ss.tmem, TMEM_COLS);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = ss.tmem;
  prefetch();
  cp_async_wait_all();
  __syncthreads();
  if (tid == 0) {
    ss.tail = RING;
    for (int sl = 0; sl < TS; ++sl) { claim_into(sl); ss.finish[sl] = 0; }
    ss.fmask = 0;
    ss.pf_from = ss.tail;
    ss.pf_to = ss.head + RING;
    if (ss.pf_to < ss.pf_from) ss.pf_to = ss.pf_from;
  }
  __syncthreads();
  if (warp == 0) publish(lane);
#pragma unroll
  for (int j = 0; j < 8; ++j) load_slot(j);
  umma::fence_async_smem();  // dictionary and zero z operands visible to the tensor core
  __syncthreads();
  if (tid == 0) ss.tail = ss.pf_to;
  prefetch();
  if (C > 1) cluster.sync();  // peers' mbarriers initialised before any DSMEM traffic

  // MMA descriptors (no swizzle): A K-major for phase a (LBO: next 8 columns, SBO: next 8 rows),
  // A MN-major for phase c (SBO: next 8 columns = M, LBO: next 8 rows = K); z and v MN-major
  // (SBO: next 8 slots, LBO: next 8 rows of K).
  const uint32_t a_addr = umma::saddr(aop), z_addr = umma::saddr(zop), v_addr = umma::saddr(vop);
  constexpr uint32_t ID_A = idesc_bf16(128, TS, 0, 1);
  constexpr uint32_t ID_C = idesc_bf16(128, TS, 1, 1);

  uint32_t phase = 0, ph_a = 0, ph_c = 0;
  // fp32 z ping-pong: phase c of this pass writes (partial, then reduced) z_{it+1} into wbuf; the
  // other buffer holds z_it, whose bf16 pieces phase a reads.  The decision at the start of the
  // next pass outputs z of finished units from the buffer that pass is about to write (read
  // before its phase c).
  float* wbuf = zbuf0;
  bool first = true;
  const bool pf = prof != nullptr && blockIdx.x == 0 && tid == 64;  // profile: one thread of CTA 0
  long long tp[9];
  auto stamp = [&](int i) { if (pf) tp[i] = clock64(); };
  for (;;) {
    stamp(0);
    // ========== phase a on the tensor core: az = A_rows z  (z operand holds z_it); issued by warp 1
    //            so that warp 0's decision runs while the MMAs are issued and executed
    if (warp == 1 && lane == 0) {
      umma::fence_after();
#pragma unroll 1
      for (int ks = 0; ks < KP / 16; ++ks) {
#pragma unroll
        for (int tt = 0; tt < 6; ++tt) {
          const uint32_t aa = a_addr + (uint32_t)(term_a(tt) * Gm::a_piece * 2) + (uint32_t)(2 * ks) * 128u;
          const uint32_t bb = z_addr + (uint32_t)(term_b(tt) * Gm::z_piece * 2) + (uint32_t)(2 * ks) * 512u;
          mma_bf16(tmem, umma::desc_noswz(aa, 128, KG * 128), umma::desc_noswz(bb, 512, 128), ID_A,
                   (ks | tt) != 0);
        }
      }
      umma::commit(&ss.bar_a);
    }
    __syncwarp();
    // ========== warp 0: decision of the previous pass, outputs, refill claims (overlaps phase a)
    if (warp == 0 && !first) {
      const int slot = lane;
      bool fin = false;
      float r = 0.f;
      for (int c = 0; c < C; ++c) r = fmaxf(r, rall[c * TS + slot]);
      if (ss.state[slot] == 1) {
        if (ss.it[slot] > 0) {
          const float prev = ss.prev_res[slot];
          const float rel = fabsf(r - prev) / fmaxf(r, Limits<float>::tiny());
          ss.stalled[slot] = (rel < kStallEps) ? ss.stalled[slot] + 1 : 0;
          ss.prev_res[slot] = r;
          if (r <= ss.thresh[slot]) { fin = true; ss.code[slot] = L1F_UNIT_OK; }
          else if (ss.stalled[slot] >= kStallIters) { fin = true; ss.code[slot] = L1F_UNIT_STALLED; }
          else if (ss.it[slot] >= P.max_iter) { fin = true; ss.code[slot] = L1F_UNIT_MAXITER; }
        }
        if (!fin) {
          ss.it[slot] += 1;
          const float bc = ss.beta_next[slot];
          ss.beta_cur[slot] = bc;
          float bn = rho * bc;  // beta = min(rho * beta, beta_max), l1reg.py:128
          if (bn > ss.beta_max[slot]) bn = ss.beta_max[slot];
          ss.beta_next[slot] = bn;
          ss.inv_next[slot] = 1.f / bn;
        }
      }
      ss.res[slot] = r;
      ss.finish[slot] = fin;
      const unsigned fmask = __ballot_sync(0xffffffffu, fin);
      if (crank == 0) {  // the finished iteration's z is the previous pass's reduced z
        const float* zprev = wbuf;  // z of the finished iteration (overwritten by this pass's phase c)
        for (unsigned mm = fmask; mm; mm &= mm - 1) {
          const int sl = __ffs(mm) - 1;
          const int64_t u = ss.unit[sl];
          for (int t = lane; t < P.k; t += 32) Z[u * P.ldz + t] = zprev[t * TSP + sl];
          if (lane == 0) {
            if (iters) iters[u] = ss.it[sl];
            if (res_out) res_out[u] = ss.res[sl];
            if (status) status[u] = ss.code[sl];
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        for (unsigned mm = fmask; mm; mm &= mm - 1) claim_into(__ffs(mm) - 1);
        ss.pf_from = ss.tail > ss.head ? ss.tail : ss.head;
        ss.pf_to = ss.head + RING;
        ss.tail = ss.pf_to;
        ss.fmask = fmask;
      }
      __syncwarp();
      publish(lane);
    }

    // ========== az from TMEM
    mbar_wait(&ss.bar_a, ph_a);
    ph_a ^= 1;
    stamp(1);
    umma::fence_after();
    float az[8];
    umma::ld8(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)slot0, az);
    umma::ld_wait();
    if (!__syncthreads_or(tid < TS && ss.state[tid] == 1)) break;
    first = false;
    stamp(2);
    {
      const uint32_t fm = (ss.fmask >> slot0) & 0xFFu;
      if (fm) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (fm & (1u << j)) load_slot(j);
      }
    }

    // ========== phase b: elementwise ADM update (reformulated residual), v -> bf16 pieces
    if (E != nullptr && grow < P.s) {  // e_it = x - l of live, non-fresh slots (numpy API path only)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (ss.prm[slot0 + j].z == 0.f) E[(int64_t)ss.unit[slot0 + j] * P.lde + grow] = xr[j] - lr[j];
    }
    float rmax[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 pr = ss.prm[slot0 + j];  // beta_it, 1/beta_{it+1}, zero-az flag
      const float tn = pr.y;
      const float x = xr[j];
      const float azv = pr.z != 0.f ? 0.f : az[j];
      const float r = lr[j] - azv;          // r_it = x - A z_it - e_it (0 for fresh and empty slots)
      rmax[j] = fabsf(r);
      const float y = fmaf(pr.x, r, yr[j]);  // y_{it+1} = y_it + b_it r_it
      const float yb = y * tn;
      const float w = (x - azv) + yb;
      const bool sup = fabsf(w) > tn;
      const float sgt = w > 0.f ? tn : -tn;
      lr[j] = sup ? (azv - yb) + sgt : x;
      az[j] = sup ? azv + sgt : x + yb;     // v = (x - e) + y / b
      yr[j] = y;
    }
    // v operand: MN-major core matrices (row group rg, slot group sg) at (rg * 4 + sg) * 64
    {
      const size_t off = (size_t)((lrow >> 3) * 4 + h) * 64 + (lrow & 7) * 8;
      split8_store(az, vop + off, vop + Gm::v_piece + off, vop + 2 * Gm::v_piece + off);
    }
    // per-slot max|r| over this warp's 32 rows: reduce-scatter butterfly (8 values over 32 lanes)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool up = lane & 16;
      const float send = up ? rmax[i] : rmax[i + 4];
      const float keep = up ? rmax[i + 4] : rmax[i];
      rmax[i] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, 16));
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const bool up = lane & 8;
      const float send = up ? rmax[i] : rmax[i + 2];
      const float keep = up ? rmax[i + 2] : rmax[i];
      rmax[i] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, 8));
    }
    {
      const bool up = lane & 4;
      const float send = up ? rmax[0] : rmax[1];
      const float keep = up ? rmax[1] : rmax[0];
      rmax[0] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, 4));
      rmax[0] = fmaxf(rmax[0], __shfl_xor_sync(0xffffffffu, rmax[0], 2));
      rmax[0] = fmaxf(rmax[0], __shfl_xor_sync(0xffffffffu, rmax[0], 1));
    }
    // lane holds slot slot0 + 4 b4 + 2 b3 + b2 (bits of the lane)
    if ((lane & 3) == 0) rpart[q * TS + slot0 + (lane >> 2)] = rmax[0];
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();

    stamp(3);
    // ========== phase c on the tensor core: zp = A_rows^T v
    if (warp == 1 && lane == 0) {
      umma::fence_after();
#pragma unroll 1
      for (int ks = 0; ks < SL / 16; ++ks) {
#pragma unroll
        for (int tt = 0; tt < 6; ++tt) {
          const uint32_t aa = a_addr + (uint32_t)(term_a(tt) * Gm::a_piece * 2) + (uint32_t)(2 * ks) * (KG * 128u);
          const uint32_t bb = v_addr + (uint32_t)(term_b(tt) * Gm::v_piece * 2) + (uint32_t)(2 * ks) * 512u;
          mma_bf16(tmem + 32, umma::desc_noswz(aa, KG * 128, 128), umma::desc_noswz(bb, 512, 128), ID_C,
                   (ks | tt) != 0);
        }
      }
      umma::commit(&ss.bar_c);
    }
    __syncwarp();
    prefetch();  // ring entries claimed above were consumed by load_slot
    if (tid < TS) {  // CTA-local max|r| per slot
      float m = fmaxf(fmaxf(rpart[tid], rpart[TS + tid]), fmaxf(rpart[2 * TS + tid], rpart[3 * TS + tid]));
      rall[crank * TS + tid] = m;
    }
    mbar_wait(&ss.bar_c, ph_c);
    ph_c ^= 1;
    stamp(4);
    umma::fence_after();
    {
      float zp[8];
      umma::ld8(tmem + ((uint32_t)(32 * q) << 16) + 32u + (uint32_t)slot0, zp);
      umma::ld_wait();
      const int t = lrow;  // TMEM lane = dictionary column
      if (t < KP) {
        float* dst = wbuf + (size_t)t * TSP + slot0;
        *reinterpret_cast<float4*>(dst) = make_float4(zp[0], zp[1], zp[2], zp[3]);
        *reinterpret_cast<float4*>(dst + 4) = make_float4(zp[4], zp[5], zp[6], zp[7]);
      }
    }
    umma::fence_before();
    __syncthreads();

    stamp(5);
    // ========== cluster reduction: partial slices -> owners, reduced slices + max|r| -> all
    if (C > 1) {
      const int slice_chunks = rs * TSP / 4;
      const uint32_t bar_p = umma::saddr(&ss.bar_p), bar_r = umma::saddr(&ss.bar_r);
      if (tid == 0) {
        mbar_arm(&ss.bar_p, (uint32_t)((C - 1) * rs * TSP * 4));
        uint32_t br = 0;
        for (int c = 0; c < C; ++c) {
          if (c == crank) continue;
          const int vc = max(0, min(rs, KP - c * rs));
          br += (uint32_t)(vc * 192 + TS * 4 + (crank == 0 ? vc * 128 : 0));
        }
        mbar_arm(&ss.bar_r, br);
      }
      for (int idx = tid; idx < (C - 1) * slice_chunks; idx += NT) {
        const int d = idx / slice_chunks, ch = idx - d * slice_chunks;
        const int owner = d < crank ? d : d + 1;
        const float* src = wbuf + (size_t)owner * rs * TSP + (size_t)ch * 4;
        const uint32_t dst = peer_addr(umma::saddr(zin + (size_t)crank * rs * TSP + (size_t)ch * 4), owner);
        st_async16(dst, src, peer_addr(bar_p, owner));
      }
      mbar_wait(&ss.bar_p, phase);
      // owner: sum my slice of z_{it+1} (fp32 into wbuf for rank 0's outputs) and split it into the
      // bf16 pieces of the phase-a operand; then push the pieces to every peer's z operand, the
      // fp32 slice to rank 0, and my per-slot max|r| to every peer
      const int r0 = crank * rs;
      const int vmine = max(0, min(rs, KP - r0));
      for (int e = tid; e < vmine * 4; e += NT) {
        const int row = e >> 2, sg = e & 3, t = r0 + row;
        float v8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v8[i] = 0.f;
        for (int c = 0; c < C; ++c) {
          const float* src = (c == crank) ? wbuf + (size_t)t * TSP + 8 * sg : zin + ((size_t)c * rs + row) * TSP + 8 * sg;
          const float4 a = *reinterpret_cast<const float4*>(src), b = *reinterpret_cast<const float4*>(src + 4);
          v8[0] += a.x; v8[1] += a.y; v8[2] += a.z; v8[3] += a.w;
          v8[4] += b.x; v8[5] += b.y; v8[6] += b.z; v8[7] += b.w;
        }
        float* dst = wbuf + (size_t)t * TSP + 8 * sg;
        *reinterpret_cast<float4*>(dst) = make_float4(v8[0], v8[1], v8[2], v8[3]);
        *reinterpret_cast<float4*>(dst + 4) = make_float4(v8[4], v8[5], v8[6], v8[7]);
        const size_t off = (size_t)((t >> 3) * 4 + sg) * 64 + (t & 7) * 8;
        split8_store(v8, zop + off, zop + Gm::z_piece + off, zop + 2 * Gm::z_piece + off);
      }
      __syncthreads();
      const int pc = vmine * 12, fc = vmine * 8, npush = pc + TS / 4 + fc;
      for (int idx = tid; idx < (C - 1) * npush; idx += NT) {
        const int d = idx / npush, ch = idx - d * npush;
        const int peer = d < crank ? d : d + 1;
        const void* src;
        uint32_t bar = bar_r;
        if (ch < pc) {  // bf16 piece chunk: (piece, row, slot group)
          const int piece = ch / (vmine * 4), rem = ch - piece * vmine * 4;
          const int t = r0 + (rem >> 2), sg = rem & 3;
          src = zop + (size_t)piece * Gm::z_piece + (size_t)((t >> 3) * 4 + sg) * 64 + (t & 7) * 8;
        } else if (ch < pc + TS / 4) {
          src = rall + (size_t)crank * TS + (size_t)(ch - pc) * 4;
        } else {
          if (peer != 0) continue;
          const int fch = ch - pc - TS / 4;
          src = wbuf + (size_t)(r0 + (fch >> 3)) * TSP + (size_t)(fch & 7) * 4;
        }
        st_async16(peer_addr(umma::saddr(src), peer), src, peer_addr(bar, peer));
      }
      mbar_wait(&ss.bar_r, phase);
      phase ^= 1;
    } else {
      for (int e = tid; e < KP * (TS / 8); e += NT) {
        const int t = e >> 2, sg = e & 3;
        const float* src = wbuf + (size_t)t * TSP + 8 * sg;
        const float4 lo = *reinterpret_cast<const float4*>(src), hi = *reinterpret_cast<const float4*>(src + 4);
        const float v8[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
        const size_t off = (size_t)((t >> 3) * 4 + sg) * 64 + (t & 7) * 8;
        split8_store(v8, zop + off, zop + Gm::z_piece + off, zop + 2 * Gm::z_piece + off);
      }
    }
    stamp(6);
    cp_async_wait_all();
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();  // z operand, reduced z, rall and the prefetched ring visible to all
    stamp(7);
    wbuf = (wbuf == zbuf0) ? zbuf1 : zbuf0;
    stamp(8);
    if (pf) {
      for (int i = 1; i < 9; ++i) prof[i] += tp[i] - tp[i - 1];
      prof[0] += 1;
    }
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  if (warp == 0) umma::tmem_dealloc(tmem, TMEM_COLS);
  if (C > 1) cluster.sync();
}

// per-unit ||x||_inf; outputs of dead units (scale 0) and of max_iter <= 0 (l1reg.py:74-75,130-135)
__global__ void unit_scale_kernel(const float* __restrict__ X, Params P, float* __restrict__ scale, float* __restrict__ Z,
                                  float* __restrict__ E, int32_t* __restrict__ iters, float* __restrict__ res,
                                  uint8_t* __restrict__ status) {
  const int lane = threadIdx.x % 32;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t u = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; u < P.n_units; u += warps) {
    const float* x = X + u * P.ldx;
    float m = 0.f;
    for (int i = lane; i < P.s; i += 32) m = fmaxf(m, fabsf(x[i]));
    m = warp_max(m);
    if (lane == 0) scale[u] = m;
    const bool dead = !(m > 0.f);
    if (dead || P.max_iter <= 0) {
      for (int t = lane; t < P.k; t += 32) Z[u * P.ldz + t] = 0.f;
      if (E)
        for (int i = lane; i < P.s; i += 32) E[u * P.lde + i] = 0.f;
      if (lane == 0) {
        if (iters) iters[u] = dead ? 0 : P.max_iter;
        if (res) res[u] = dead ? 0.f : Limits<float>::inf();
        if (status) status[u] = dead ? L1F_UNIT_ZERO : L1F_UNIT_MAXITER;
      }
    }
  }
}

template <int KP>
int launch(const float* X, int64_t ldx, int s, int64_t n_units, const float* A, int64_t lda, int k, double tol,
           double rho, double beta0, double beta_max, int max_iter, float* Z, int64_t ldz, float* E, int64_t lde,
           int32_t* iters, float* res, uint8_t* status, void* workspace, size_t ws_bytes, cudaStream_t st, bool query,
           size_t* need) {
  using Gm = Geo<KP>;
  const int C = (int)ceil_div(s, SL);
  const size_t scale_bytes = (sizeof(float) * (size_t)(n_units > 0 ? n_units : 1) + 255) & ~(size_t)255;
  if (query) { *need = scale_bytes; return L1F_OK; }
  auto kern = adm_tc_kernel<KP>;
  static bool configured = false;
  if (!configured) {
    L1F_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Gm::smem_bytes));
    L1F_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    configured = true;
  }
  void* owned = nullptr;
  if (!workspace) {
    L1F_CUDA_TRY(cudaMallocAsync(&owned, scale_bytes, st));
    workspace = owned;
  } else {
    L1F_REQUIRE(ws_bytes >= scale_bytes, L1F_ERR_ARG, "filter: workspace too small");
  }
  Params P;
  P.s = s; P.k = k; P.cluster = C; P.rs = (int)ceil_div(KP, C);
  P.n_units = n_units; P.ldx = ldx; P.ldz = ldz; P.lde = lde; P.max_iter = max_iter;
  P.tol = tol; P.rho = rho; P.beta0 = beta0; P.beta_max = beta_max;
  float* scale = (float*)workspace;
  int rc = L1F_OK;
  unit_scale_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n_units, 8), 65535), 256, 0, st>>>(X, P, scale, Z, E, iters,
                                                                                              res, status);
  if (cudaGetLastError() != cudaSuccess) rc = L1F_ERR_CUDA;
  if (rc == L1F_OK && max_iter > 0) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(NT, 1, 1);
    cfg.dynamicSmemBytes = Gm::smem_bytes;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(C, 1, 1);
    int max_clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1)
      max_clusters = std::max(1, num_sms() / C);
    const int64_t want = ceil_div(n_units, TS);
    const int nclusters = (int)std::min<int64_t>(max_clusters, std::max<int64_t>(1, want));
    cfg.gridDim = dim3((unsigned)(nclusters * C), 1, 1);
    static long long* prof = nullptr;
    const char* pe = getenv("L1F_TC_PROF");
    if (pe && pe[0] == '1' && !prof) {
      cudaMallocManaged(&prof, 16 * sizeof(long long));
      memset(prof, 0, 16 * sizeof(long long));
    }
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, X, A, lda, (const float*)scale, P, Z, E, iters, res, status, prof);
    if (prof) {
      cudaStreamSynchronize(st);
      const char* names[9] = {"passes", "a:mma+decision", "syncthreads_or", "phase b", "c:mma wait", "zp->smem",
                              "reduction", "cp wait+sync", "convert"};
      fprintf(stderr, "[tc prof] KP=%d C=%d", KP, C);
      for (int i = 0; i < 9; ++i)
        fprintf(stderr, " %s=%.0f", names[i], i ? (double)prof[i] / (double)prof[0] : (double)prof[0]);
      fprintf(stderr, "\n");
      memset(prof, 0, 16 * sizeof(long long));
    }
    if (e != cudaSuccess) {
      set_error("filter (tensor core, KP=%d C=%d): launch failed: %s", KP, C, cudaGetErrorString(e));
      rc = L1F_ERR_CUDA;
    }
  } else if (rc != L1F_OK) {
    set_error("filter: prologue launch failed");
  }
  if (owned) cudaFreeAsync(owned, st);
  return rc;
}

}  // namespace tcf
}  // namespace l1f

// dispatch used by filter.cu (float only): L1F_ERR_UNSUPPORTED when the shape does not fit;
// L1F_FILTER_TC=0 disables the tensor-core kernel
int l1f_tc_dispatch(const float* X, int64_t ldx, int s, int64_t n_units, const float* A, int64_t lda, int k,
                    double tol, double rho, double beta0, double beta_max, int max_iter, float* Z, int64_t ldz,
                    float* E, int64_t lde, int32_t* iters, float* res, uint8_t* status, void* workspace,
                    size_t ws_bytes, cudaStream_t st, bool query, size_t* need) {
  const char* env = getenv("L1F_FILTER_TC");
  if (env && env[0] == '0') return L1F_ERR_UNSUPPORTED;
  const int kp = (int)l1f::ceil_div(k, 16) * 16;
  if (k <= 16 || kp > 128 || s > 16 * l1f::tcf::SL) return L1F_ERR_UNSUPPORTED;
#define L1F_TC(KP)                                                                                               \
  case KP:                                                                                                       \
    return l1f::tcf::launch<KP>(X, ldx, s, n_units, A, lda, k, tol, rho, beta0, beta_max, max_iter, Z, ldz, E, lde, \
                                iters, res, status, workspace, ws_bytes, st, query, need)
  switch (kp) {
    L1F_TC(32);
    L1F_TC(48);
    L1F_TC(64);
    L1F_TC(80);
    L1F_TC(96);
    L1F_TC(112);
    L1F_TC(128);
  }
#undef L1F_TC
  return L1F_ERR_UNSUPPORTED;
}
