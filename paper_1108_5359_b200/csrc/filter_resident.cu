// Resident-state ADM filter kernel (K3 v2) — the hot path of l1 filtering.
//
// Same problem and per-unit semantics as filter.cu (reference: _solve_block,
// pkg/src/l1pcp/l1reg.py:59-137), re-laid out so that nothing but the small z vectors
// moves during the iterations:
//
//  * a thread-block CLUSTER of C CTAs owns TS = 32 unit slots; CTA c keeps rows
//    [c*SL, (c+1)*SL) of the dictionary A (s x k) resident in shared memory ("A4" layout:
//    16-byte cells holding 4 consecutive rows of one column, quad stride KP+1 cells, so
//    phase a reads 4 rows and phase c reads 4 columns with one conflict-free LDS.128);
//  * each thread keeps the ADM state (x, y, l = x - e) of a 4-row x 4-slot tile in
//    registers across iterations;
//  * one ADM iteration of every slot per pass:
//      phase a  az = A_rows z_it                 (4x4 register tile over k)
//      phase b  r_it, y_{it+1}, e_{it+1} (as l), v; per-slot max|r|
//      phase c  z_part = A_rows^T v              (16k x 32-slot warp tiles, row groups)
//      cluster  z_{it+1} = sum_c z_part_c, res = max_c (DSMEM), decision, refill;
//  * the residual is formed without cancelling the large corrupted entries: with
//    l = x - e, r = x - Az - e = l - Az, and on the shrink support l = Az - y/b + sign(w)/b
//    (exact algebra), so FP32 resolves r far below ulp(max|x|);
//  * units are assigned to clusters round-robin and slots refill as units converge; a
//    unit's arithmetic depends only on the unit, never on its slot, cluster or GPU.
#include "common.cuh"

#include <algorithm>
#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace l1f {
namespace resident {

constexpr int TS = 32;
constexpr int kStallIters = 20;       // STAGNATION_ITERS, l1reg.py:34
constexpr double kStallEps = 1e-12;   // STAGNATION_EPS, l1reg.py:33

template <typename T> struct Vec4;
template <> struct Vec4<float> {
  __device__ static __forceinline__ void ld(const float* p, float (&v)[4]) {
    float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
  __device__ static __forceinline__ void st(float* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <> struct Vec4<double> {
  __device__ static __forceinline__ void ld(const double* p, double (&v)[4]) {
    double2 a = *reinterpret_cast<const double2*>(p), b = *reinterpret_cast<const double2*>(p + 2);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
  __device__ static __forceinline__ void st(double* p, const double (&v)[4]) {
    *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    *reinterpret_cast<double2*>(p + 2) = make_double2(v[2], v[3]);
  }
};

struct Params {
  int s, k, ka, cluster;
  int64_t n_units, ldx, ldz, lde;
  int max_iter;
  double tol, rho, beta0, beta_max;
};

constexpr int RING = 4;  // prefetched upcoming units per cluster

template <typename T>
struct Slots {
  int unit[TS], it[TS], stalled[TS], state[TS], finish[TS], src[TS];
  T beta_cur[TS], beta_next[TS], inv_next[TS], beta_max[TS], thresh[TS], prev_res[TS], res[TS];
  T ring_sc[RING];
  long long ring_u[RING];
  long long head, tail, pf_from, pf_to;  // candidate cursor of this cluster (identical in all its CTAs)
  alignas(8) unsigned long long bar_p, bar_r;  // mbarriers of the DSMEM z reduction
  uint8_t code[TS];
};

constexpr int pow2_floor(int v) { return v >= 16 ? 16 : v >= 8 ? 8 : v >= 4 ? 4 : v >= 2 ? 2 : 1; }

template <typename T, int KP_, int SL_, int NT_>
struct Geo {
  static constexpr int KP = KP_, SL = SL_, NT = NT_;
  static constexpr int NW = NT / 32;
  static constexpr int NRB = SL / 32;                // 32-row blocks
  static constexpr int QUADS = SL / 4;
  static constexpr int QS = KP + 1;                  // cells per quad (odd -> conflict free)
  static constexpr int KT = KP / 16;                 // phase-c k tiles
  static constexpr int G = pow2_floor(NW >= KT ? NW / KT : 1);  // phase-c row groups (divide QUADS)
  static constexpr int ITEMS = KT * G;
  static constexpr int IPW = (ITEMS + NW - 1) / NW;
  static constexpr int QPG = QUADS / G;
  static_assert(KP % 16 == 0, "KP must be a multiple of 16");
  static_assert(NW == NRB * 2, "phase a: one warp per (32-row block, 16-slot half)");
  static_assert(QUADS % G == 0, "row groups must split the quads evenly");
  static_assert((QUADS / G) % 8 == 0, "phase c walks quads in blocks of 8");
  static constexpr size_t a4_elems = (size_t)QUADS * QS * 4;
  static constexpr size_t z_elems = (size_t)KP * TS;
  static constexpr size_t zg_elems = (G > 1 ? (size_t)(G - 1) : 0) * z_elems;
  static constexpr size_t v_elems = (size_t)SL * TS;
  static constexpr size_t r_elems = (size_t)NRB * TS;
  static constexpr size_t ring_elems = (size_t)RING * SL;
  static constexpr size_t rall_elems = (size_t)16 * TS;
  // a4 | zc | zn (= reduced z) | zin (peer partials) | zg | vs | rpart | ring_x | rall
  static constexpr size_t smem_bytes =
      sizeof(T) * (a4_elems + 3 * z_elems + zg_elems + v_elems + r_elems + ring_elems + rall_elems);
};

// swizzled 16-byte chunk of V row `row` holding slots [4c, 4c+3]
__device__ __forceinline__ int vchunk(int row, int c) { return c ^ ((row >> 2) & 7); }

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t peer_addr(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(void* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(void* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(void* bar, uint32_t parity) {
  const uint32_t a = smem_addr(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(a), "r"(parity) : "memory");
  } while (!done);
}
// 16-byte asynchronous store into a peer CTA's shared memory, completing bytes on its mbarrier
__device__ __forceinline__ void st_async16(uint32_t peer_dst, const void* src16, uint32_t peer_bar) {
  const uint4 v = *reinterpret_cast<const uint4*>(src16);
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
               ::"r"(peer_dst), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(peer_bar) : "memory");
}
// element-sized asynchronous global->shared copy (zero-filled when !valid)
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* dst, const T* src, bool valid) {
  static_assert(sizeof(T) == 4 || sizeof(T) == 8, "4- or 8-byte elements");
  if (sizeof(T) == 4)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(valid ? 4 : 0)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <typename T, int KP, int SL, int NT>
__global__ void __launch_bounds__(NT, 1)
adm_resident_kernel(const T* __restrict__ X, const T* __restrict__ A, int64_t lda, const T* __restrict__ scale,
                    Params P, T* __restrict__ Z, T* __restrict__ E, int32_t* __restrict__ iters,
                    T* __restrict__ res_out, uint8_t* __restrict__ status) {
  using Gm = Geo<T, KP, SL, NT>;
  constexpr int QS = Gm::QS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* a4 = reinterpret_cast<T*>(smem_raw);
  T* zc = a4 + Gm::a4_elems;      // z_it used by phase a                       [KP][TS]
  T* zn = zc + Gm::z_elems;       // partial of z_{it+1}, then the reduced z    [KP][TS]
  T* zin = zn + Gm::z_elems;      // peers' partials of this CTA's row slice    [C][KP/C][TS]
  T* zg = zin + Gm::z_elems;      // phase-c row-group partials (groups 1..)    [G-1][KP][TS]
  T* vs = zg + Gm::zg_elems;      // v, swizzled                                [SL][TS]
  T* rpart = vs + Gm::v_elems;    // per-32-row-block slot max|r|               [NRB][TS]
  T* ring_x = rpart + Gm::r_elems;  // x rows of prefetched units             [RING][SL]
  T* rall = ring_x + Gm::ring_elems;  // every CTA's slot max|r|              [16][TS]
  __shared__ Slots<T> ss;

  cg::cluster_group cluster = cg::this_cluster();
  const int C = P.cluster;
  const int crank = C > 1 ? (int)cluster.block_rank() : 0;
  const int cid = blockIdx.x / C, nclusters = gridDim.x / C;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int row_base = crank * SL;
  const T tol = (T)P.tol, rho = (T)P.rho;
  const int rs = KP / C;  // rows of z reduced by each CTA

  // ---- resident dictionary rows: a4[q][t][r] = A[row_base + 4q + r][t]
  for (int e = tid; e < (int)Gm::a4_elems; e += NT) {
    const int r = e & 3, cell = e >> 2, q = cell / QS, t = cell - q * QS;
    const int row = row_base + 4 * q + r;
    a4[e] = (row < P.s && t < P.k) ? A[(int64_t)row * lda + t] : T(0);
  }
  for (int e = tid; e < (int)Gm::z_elems; e += NT) zc[e] = T(0);

  const int rb = warp >> 1, sh = warp & 1;
  const int rq = lane >> 2, sq = lane & 3;
  const int quad = rb * 8 + rq;
  const int lrow0 = 4 * quad;
  const int grow0 = row_base + lrow0;
  const int slot0 = sh * 16 + sq * 4;
  const int kq = lane & 3, sq8 = lane >> 2;

  T xr[4][4], yr[4][4], lr[4][4];  // ADM state [row][slot]

  // candidate j of this cluster is unit cid + j * nclusters
  auto cand = [&](long long j) -> long long { return (long long)cid + j * (long long)nclusters; };
  // all threads: start prefetching candidates [pf_from, pf_to) into the ring
  auto prefetch = [&]() {
    for (long long j = ss.pf_from; j < ss.pf_to; ++j) {
      const int e = (int)(j % RING);
      const long long u = cand(j);
      const bool ok = u < P.n_units;
      for (int r = tid; r < SL; r += NT)
        cp_async_elem(ring_x + (size_t)e * SL + r, X + (ok ? u : 0) * P.ldx + (ok && row_base + r < P.s ? row_base + r : 0),
                  ok && row_base + r < P.s);
      if (tid == 0) {
        ss.ring_u[e] = u;
        cp_async_elem(&ss.ring_sc[e], scale + (ok ? u : 0), ok);
      }
    }
  };
  auto install_unit = [&](int slot, long long u, T sc, int src) {
    const T b0 = P.beta0 > 0 ? (T)P.beta0 : T(1) / sc;
    ss.unit[slot] = (int)u;
    ss.state[slot] = 1;
    ss.it[slot] = 0;
    ss.stalled[slot] = 0;
    ss.src[slot] = src;
    ss.beta_cur[slot] = b0;
    ss.beta_next[slot] = b0;
    ss.inv_next[slot] = T(1) / b0;
    ss.beta_max[slot] = P.beta_max > 0 ? (T)P.beta_max : (T)1e7 * b0;
    ss.thresh[slot] = tol * sc;
    ss.prev_res[slot] = Limits<T>::inf();
  };
  // one thread: next live unit for `slot` (prefetched ring first, then synchronous)
  auto claim_into = [&](int slot) {
    for (;;) {
      if (ss.head < ss.tail) {
        const int e = (int)(ss.head % RING);
        const long long u = ss.ring_u[e];
        ss.head++;
        if (u >= P.n_units) break;
        if (ss.ring_sc[e] > T(0)) { install_unit(slot, u, ss.ring_sc[e], e); return; }
      } else {
        const long long u = cand(ss.head);
        ss.head++;
        ss.tail = ss.head;
        if (u >= P.n_units) break;
        const T sc = scale[u];
        if (sc > T(0)) { install_unit(slot, u, sc, -1); return; }
      }
    }
    ss.state[slot] = 0;
    ss.unit[slot] = -1;
  };
  auto load_slot = [&](int j) {  // (re)initialise this thread's state of slot slot0+j
    const int slot = slot0 + j;
    const bool live = ss.state[slot] == 1;
    const int src = ss.src[slot];
    const int64_t u = live ? ss.unit[slot] : 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = grow0 + i;
      T x = T(0);
      if (live && row < P.s) x = src >= 0 ? ring_x[(size_t)src * SL + lrow0 + i] : X[u * P.ldx + row];
      xr[i][j] = x;
      yr[i][j] = T(0);
      lr[i][j] = T(0);
    }
  };

  if (tid == 0) {
    ss.head = 0; ss.tail = 0; ss.pf_from = 0; ss.pf_to = RING;
    mbar_init(&ss.bar_p, 1);
    mbar_init(&ss.bar_r, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  prefetch();
  cp_async_wait_all();
  __syncthreads();
  if (tid == 0) {
    ss.tail = RING;
    for (int sl = 0; sl < TS; ++sl) { claim_into(sl); ss.finish[sl] = 0; }
    ss.pf_from = ss.tail;
    ss.pf_to = ss.head + RING;
    if (ss.pf_to < ss.pf_from) ss.pf_to = ss.pf_from;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 4; ++j) load_slot(j);
  __syncthreads();
  if (tid == 0) ss.tail = ss.pf_to;
  prefetch();
  if (C > 1) cluster.sync();  // peers' mbarriers initialised before any DSMEM traffic

  uint32_t phase = 0;
  T* zcur = zc;   // z_it read by phase a
  T* znext = zn;  // partial, then reduced, z_{it+1}
  T* zprev = zn;  // z of the previous pass (outputs of units finishing there)
  bool first = true;
  for (;;) {
    // ========== warp 0: decision of the previous pass, outputs, refill claims
    //            (overlaps the other warps' phase a; identical in every CTA)
    if (warp == 0 && !first) {
      const int slot = lane;
      bool fin = false;
      T r = T(0);
      for (int c = 0; c < C; ++c) r = tmax(r, rall[c * TS + slot]);
      if (ss.state[slot] == 1) {
        if (ss.it[slot] > 0) {
          const T prev = ss.prev_res[slot];
          const T rel = tabs(r - prev) / tmax(r, Limits<T>::tiny());
          ss.stalled[slot] = (rel < (T)kStallEps) ? ss.stalled[slot] + 1 : 0;
          ss.prev_res[slot] = r;
          if (r <= ss.thresh[slot]) { fin = true; ss.code[slot] = L1F_UNIT_OK; }
          else if (ss.stalled[slot] >= kStallIters) { fin = true; ss.code[slot] = L1F_UNIT_STALLED; }
          else if (ss.it[slot] >= P.max_iter) { fin = true; ss.code[slot] = L1F_UNIT_MAXITER; }
        }
        if (!fin) {
          ss.it[slot] += 1;
          const T bc = ss.beta_next[slot];
          ss.beta_cur[slot] = bc;
          T bn = rho * bc;  // beta = min(rho * beta, beta_max), l1reg.py:128
          if (bn > ss.beta_max[slot]) bn = ss.beta_max[slot];
          ss.beta_next[slot] = bn;
          ss.inv_next[slot] = T(1) / bn;
        }
      }
      ss.res[slot] = r;
      ss.finish[slot] = fin;
      const unsigned fmask = __ballot_sync(0xffffffffu, fin);
      if (crank == 0) {  // outputs: the finished iteration's z is in zprev
        for (unsigned mm = fmask; mm; mm &= mm - 1) {
          const int sl = __ffs(mm) - 1;
          const int64_t u = ss.unit[sl];
          for (int t = lane; t < P.k; t += 32) Z[u * P.ldz + t] = zprev[t * TS + sl];
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
      }
      __syncwarp();
    }

    // ========== phase a: az[i][j] = sum_t A[row i][t] z_it[t][slot j]  (software pipelined)
    T az[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) az[i][j] = T(0);
    {
      const T* acell = a4 + (size_t)quad * QS * 4;
      const T* zrow = zcur + slot0;
      const int ka = P.ka;  // multiple of 4
      T a0[4], z0[4], a1[4], z1[4];
      Vec4<T>::ld(acell, a0);
      Vec4<T>::ld(zrow, z0);
      Vec4<T>::ld(acell + 4, a1);
      Vec4<T>::ld(zrow + TS, z1);
      for (int t = 0; t < ka; t += 2) {
        T na0[4], nz0[4], na1[4], nz1[4];
        const int tn = t + 2 < ka ? t + 2 : t;  // harmless reload on the last step
        Vec4<T>::ld(acell + 4 * tn, na0);
        Vec4<T>::ld(zrow + tn * TS, nz0);
        Vec4<T>::ld(acell + 4 * tn + 4, na1);
        Vec4<T>::ld(zrow + (tn + 1) * TS, nz1);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) az[i][j] = fma(a0[i], z0[j], az[i][j]);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) az[i][j] = fma(a1[i], z1[j], az[i][j]);
#pragma unroll
        for (int q = 0; q < 4; ++q) { a0[q] = na0[q]; z0[q] = nz0[q]; a1[q] = na1[q]; z1[q] = nz1[q]; }
      }
    }
    if (!__syncthreads_or(tid < TS && ss.state[tid] == 1)) break;
    first = false;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (ss.finish[slot0 + j]) load_slot(j);

    // ========== phase b: elementwise ADM update (reformulated residual), v -> shared
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int slot = slot0 + j;
      const bool live = ss.state[slot] == 1;
      const bool fresh = ss.it[slot] == 0;
      const T bcur = ss.beta_cur[slot], tn = ss.inv_next[slot];
      const int64_t u = ss.unit[slot];
      T m = T(0);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        T v = T(0);
        if (live) {
          const T x = xr[i][j];
          T y = fresh ? T(0) : yr[i][j];
          const T azv = fresh ? T(0) : az[i][j];
          if (!fresh) {
            if (E != nullptr && grow0 + i < P.s) E[u * P.lde + grow0 + i] = x - lr[i][j];  // e_it
            const T r = lr[i][j] - azv;     // r_it = x - A z_it - e_it
            m = tmax(m, tabs(r));
            y = fma(bcur, r, y);            // y_{it+1} = y_it + b_it r_it
          }
          const T yb = y * tn;              // y_{it+1} / b_{it+1}
          const T w = (x - azv) + yb;       // w_{it+1}
          const bool sup = tabs(w) > tn;
          const T sg = w > T(0) ? T(1) : T(-1);
          lr[i][j] = sup ? (azv - yb) + sg * tn : x;  // l = x - shrink(w, 1/b)
          v = sup ? azv + sg * tn : x + yb;           // (x - e) + y/b
          yr[i][j] = y;
        }
        az[i][j] = v;
      }
      m = tmax(m, __shfl_xor_sync(0xffffffffu, m, 4));
      m = tmax(m, __shfl_xor_sync(0xffffffffu, m, 8));
      m = tmax(m, __shfl_xor_sync(0xffffffffu, m, 16));
      if (rq == 0) rpart[rb * TS + slot] = m;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = lrow0 + i;
      T v4[4] = {az[i][0], az[i][1], az[i][2], az[i][3]};
      Vec4<T>::st(vs + (size_t)row * TS + 4 * vchunk(row, slot0 >> 2), v4);
    }
    __syncthreads();
    prefetch();  // ring entries claimed above were consumed by load_slot

    // ========== phase c: z_part[k][slot] = sum_rows A[row][k] v[row][slot]  (pipelined)
#pragma unroll
    for (int ii = 0; ii < Gm::IPW; ++ii) {
      const int item = warp + ii * Gm::NW;
      if (item < Gm::ITEMS) {
        const int kt = item % Gm::KT, g = item / Gm::KT;
        T acc[4][4];  // [k j][slot s]
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int s2 = 0; s2 < 4; ++s2) acc[j][s2] = T(0);
        const int kbase = kt * 16 + kq;
        const int q0 = g * Gm::QPG, q1 = q0 + Gm::QPG;
        // quads in blocks of 8: (q & 7) == qq is compile-time, so is the V swizzle
        for (int qb = q0; qb < q1; qb += 8) {
          const T* acell = a4 + ((size_t)qb * QS + kbase) * 4;
          const T* vblk = vs + (size_t)(4 * qb) * TS;
#pragma unroll
          for (int qq = 0; qq < 8; ++qq) {
            T a[4][4];  // [k j][row r]
#pragma unroll
            for (int j = 0; j < 4; ++j) Vec4<T>::ld(acell + ((size_t)qq * QS + 4 * j) * 4, a[j]);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              T v[4];
              Vec4<T>::ld(vblk + (size_t)(4 * qq + r) * TS + 4 * (sq8 ^ qq), v);
#pragma unroll
              for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int s2 = 0; s2 < 4; ++s2) acc[j][s2] = fma(a[j][r], v[s2], acc[j][s2]);
            }
          }
        }
        T* dst = (g == 0) ? znext : zg + (size_t)(g - 1) * Gm::z_elems;
#pragma unroll
        for (int j = 0; j < 4; ++j) Vec4<T>::st(dst + (size_t)(kbase + 4 * j) * TS + 4 * sq8, acc[j]);
      }
    }
    if (tid < TS) {  // CTA-local max|r| per slot
      T m = T(0);
#pragma unroll
      for (int b = 0; b < Gm::NRB; ++b) m = tmax(m, rpart[b * TS + tid]);
      rall[crank * TS + tid] = m;
    }
    __syncthreads();
    if (Gm::G > 1) {
      for (int e = tid; e < (int)Gm::z_elems; e += NT) {
        T sacc = znext[e];
#pragma unroll
        for (int g = 1; g < Gm::G; ++g) sacc += zg[(size_t)(g - 1) * Gm::z_elems + e];
        znext[e] = sacc;
      }
      if (C > 1) __syncthreads();
    }

    // ========== cluster reduction: partial slices -> owners, reduced slices + max|r| -> all
    if (C > 1) {
      constexpr int CH = 16 / (int)sizeof(T);  // elements per 16-byte chunk
      const int slice_chunks = rs * TS / CH;
      const uint32_t bar_p = smem_addr(&ss.bar_p), bar_r = smem_addr(&ss.bar_r);
      if (tid == 0) {
        mbar_arm(&ss.bar_p, (uint32_t)((C - 1) * rs * TS * sizeof(T)));
        mbar_arm(&ss.bar_r, (uint32_t)((C - 1) * (rs * TS + TS) * sizeof(T)));
      }
      for (int idx = tid; idx < (C - 1) * slice_chunks; idx += NT) {
        const int d = idx / slice_chunks, ch = idx - d * slice_chunks;
        const int owner = d < crank ? d : d + 1;
        const T* src = znext + (size_t)owner * rs * TS + (size_t)ch * CH;
        const uint32_t dst = peer_addr(smem_addr(zin + (size_t)crank * rs * TS + (size_t)ch * CH), owner);
        st_async16(dst, src, peer_addr(bar_p, owner));
      }
      mbar_wait(&ss.bar_p, phase);
      T* mine = znext + (size_t)crank * rs * TS;
      for (int e = tid; e < rs * TS; e += NT) {
        T sacc = T(0);
        for (int c = 0; c < C; ++c) sacc += (c == crank) ? mine[e] : zin[(size_t)c * rs * TS + e];
        mine[e] = sacc;
      }
      __syncthreads();
      const int push_chunks = slice_chunks + TS / CH;
      for (int idx = tid; idx < (C - 1) * push_chunks; idx += NT) {
        const int d = idx / push_chunks, ch = idx - d * push_chunks;
        const int peer = d < crank ? d : d + 1;
        // same offset in the peer: my reduced slice of z, then my slot max|r|
        const T* src = ch < slice_chunks ? mine + (size_t)ch * CH : rall + (size_t)crank * TS + (size_t)(ch - slice_chunks) * CH;
        st_async16(peer_addr(smem_addr(src), peer), src, peer_addr(bar_r, peer));
      }
      mbar_wait(&ss.bar_r, phase);
      phase ^= 1;
    } else if (Gm::G > 1) {
      __syncthreads();
    }
    cp_async_wait_all();
    __syncthreads();  // reduced z, rall and the prefetched ring visible to warp 0
    zprev = zcur;
    zcur = znext;
    znext = zprev;
  }
  if (C > 1) cluster.sync();
}

// per-unit ||x||_inf; outputs of dead units (scale 0) and of max_iter <= 0 (l1reg.py:74-75,130-135)
template <typename T>
__global__ void unit_scale_kernel(const T* __restrict__ X, Params P, T* __restrict__ scale, T* __restrict__ Z,
                                  T* __restrict__ E, int32_t* __restrict__ iters, T* __restrict__ res,
                                  uint8_t* __restrict__ status) {
  const int lane = threadIdx.x % 32;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t u = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; u < P.n_units; u += warps) {
    const T* x = X + u * P.ldx;
    T m = T(0);
    for (int i = lane; i < P.s; i += 32) m = tmax(m, tabs(x[i]));
    m = warp_max(m);
    if (lane == 0) scale[u] = m;
    const bool dead = !(m > T(0));
    if (dead || P.max_iter <= 0) {
      for (int t = lane; t < P.k; t += 32) Z[u * P.ldz + t] = T(0);
      if (E)
        for (int i = lane; i < P.s; i += 32) E[u * P.lde + i] = T(0);
      if (lane == 0) {
        if (iters) iters[u] = dead ? 0 : P.max_iter;
        if (res) res[u] = dead ? T(0) : Limits<T>::inf();
        if (status) status[u] = dead ? L1F_UNIT_ZERO : L1F_UNIT_MAXITER;
      }
    }
  }
}

template <typename T, int KP, int SL, int NT>
int launch(const T* X, int64_t ldx, int s, int64_t n_units, const T* A, int64_t lda, int k, double tol, double rho,
           double beta0, double beta_max, int max_iter, T* Z, int64_t ldz, T* E, int64_t lde, int32_t* iters, T* res,
           uint8_t* status, void* workspace, size_t ws_bytes, cudaStream_t st, bool query, size_t* need) {
  using Gm = Geo<T, KP, SL, NT>;
  const int C = (int)ceil_div(s, SL);
  const size_t scale_bytes = (sizeof(T) * (size_t)(n_units > 0 ? n_units : 1) + 255) & ~(size_t)255;
  if (query) { *need = scale_bytes; return L1F_OK; }
  auto kern = adm_resident_kernel<T, KP, SL, NT>;
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
  P.s = s; P.k = k; P.ka = (int)ceil_div(k, 4) * 4; P.cluster = C;
  P.n_units = n_units; P.ldx = ldx; P.ldz = ldz; P.lde = lde; P.max_iter = max_iter;
  P.tol = tol; P.rho = rho; P.beta0 = beta0; P.beta_max = beta_max;
  T* scale = (T*)workspace;
  int rc = L1F_OK;
  unit_scale_kernel<T><<<(unsigned)std::min<int64_t>(ceil_div(n_units, 8), 65535), 256, 0, st>>>(
      X, P, scale, Z, E, iters, res, status);
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
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, X, A, lda, (const T*)scale, P, Z, E, iters, res, status);
    if (e != cudaSuccess) {
      set_error("filter (resident, KP=%d SL=%d C=%d): launch failed: %s", KP, SL, C, cudaGetErrorString(e));
      rc = L1F_ERR_CUDA;
    }
  } else if (rc != L1F_OK) {
    set_error("filter: prologue launch failed");
  }
  if (owned) cudaFreeAsync(owned, st);
  return rc;
}

}  // namespace resident
}  // namespace l1f

// dispatch used by filter.cu: returns L1F_ERR_UNSUPPORTED when no resident geometry fits
template <typename T>
int l1f_resident_dispatch(const T* X, int64_t ldx, int s, int64_t n_units, const T* A, int64_t lda, int k,
                          double tol, double rho, double beta0, double beta_max, int max_iter, T* Z, int64_t ldz,
                          T* E, int64_t lde, int32_t* iters, T* res, uint8_t* status, void* workspace,
                          size_t ws_bytes, cudaStream_t st, bool query, size_t* need);

#define L1F_RES(TT, KP, SL, NT)                                                                              \
  return l1f::resident::launch<TT, KP, SL, NT>(X, ldx, s, n_units, A, lda, k, tol, rho, beta0, beta_max,    \
                                               max_iter, Z, ldz, E, lde, iters, res, status, workspace,     \
                                               ws_bytes, st, query, need)

template <>
int l1f_resident_dispatch<float>(const float* X, int64_t ldx, int s, int64_t n_units, const float* A, int64_t lda,
                                 int k, double tol, double rho, double beta0, double beta_max, int max_iter,
                                 float* Z, int64_t ldz, float* E, int64_t lde, int32_t* iters, float* res,
                                 uint8_t* status, void* workspace, size_t ws_bytes, cudaStream_t st, bool query,
                                 size_t* need) {
  const int kp = (int)l1f::ceil_div(k, 16) * 16;
  if (k <= 16) return L1F_ERR_UNSUPPORTED;
  if (kp <= 112 && s <= 16 * 256) {
    switch (kp) {
      case 32: L1F_RES(float, 32, 256, 512);
      case 48: L1F_RES(float, 48, 256, 512);
      case 64: L1F_RES(float, 64, 256, 512);
      case 80: L1F_RES(float, 80, 256, 512);
      case 96: L1F_RES(float, 96, 256, 512);
      case 112: L1F_RES(float, 112, 256, 512);
    }
  }
  if (kp <= 224 && s <= 16 * 128) {
    switch (kp) {
      case 32: L1F_RES(float, 32, 128, 256);
      case 48: L1F_RES(float, 48, 128, 256);
      case 64: L1F_RES(float, 64, 128, 256);
      case 80: L1F_RES(float, 80, 128, 256);
      case 96: L1F_RES(float, 96, 128, 256);
      case 112: L1F_RES(float, 112, 128, 256);
      case 128: L1F_RES(float, 128, 128, 256);
      case 144: L1F_RES(float, 144, 128, 256);
      case 160: L1F_RES(float, 160, 128, 256);
      case 176: L1F_RES(float, 176, 128, 256);
      case 192: L1F_RES(float, 192, 128, 256);
      case 208: L1F_RES(float, 208, 128, 256);
      case 224: L1F_RES(float, 224, 128, 256);
    }
  }
  return L1F_ERR_UNSUPPORTED;
}

template <>
int l1f_resident_dispatch<double>(const double* X, int64_t ldx, int s, int64_t n_units, const double* A,
                                  int64_t lda, int k, double tol, double rho, double beta0, double beta_max,
                                  int max_iter, double* Z, int64_t ldz, double* E, int64_t lde, int32_t* iters,
                                  double* res, uint8_t* status, void* workspace, size_t ws_bytes, cudaStream_t st,
                                  bool query, size_t* need) {
  const int kp = (int)l1f::ceil_div(k, 16) * 16;
  if (k <= 16) return L1F_ERR_UNSUPPORTED;
  if (kp <= 96 && s <= 16 * 128) {
    switch (kp) {
      case 32: L1F_RES(double, 32, 128, 256);
      case 48: L1F_RES(double, 48, 128, 256);
      case 64: L1F_RES(double, 64, 128, 256);
      case 80: L1F_RES(double, 80, 128, 256);
      case 96: L1F_RES(double, 96, 128, 256);
    }
  }
  return L1F_ERR_UNSUPPORTED;
}
#undef L1F_RES
