// Column-separable l1 regression by ADM — the hot path of l1 filtering.
//
// Reference: _solve_block (pkg/src/l1pcp/l1reg.py:59-137), driven per 64-column chunk by
// solve_l1reg_columnwise (l1reg.py:163-214) and called by filter_columns / filter_rows
// (l1filter.py:116-134).  Per unit x (length s) against an orthonormal A (s x k):
//   w = x - A z + y/b ; e = shrink(w, 1/b) ; z = A^T (x - e + y/b) ; r = x - A z - e
//   res = max|r| ; stop when res <= tol*||x||_inf or 20 stagnant iterations ; y += b r ;
//   b = min(rho b, b_max)
//
// B200 design:
//  * persistent CTAs, each owning TS = 32 unit SLOTS; a slot whose unit converges is
//    refilled from a global work counter, so lockstep waste is bounded by one iteration
//    per unit instead of max-iterations-per-group;
//  * one pass over the rows of A per ADM iteration: for every 32-row chunk the CTA
//    computes (A z)[rows] for all slots, the elementwise ADM update for those rows, and
//    accumulates the NEXT iteration's A^T v into registers.  A is read once per iteration
//    per 32 units (the reference reads it three times per unit, l1reg.py:96-99);
//  * the per-unit ADM state (y and a double-buffered e) streams through a per-CTA
//    workspace that stays L2-resident; x streams from the unit-major panel;
//  * each unit's arithmetic is independent of its slot, CTA and GPU, so results are
//    bitwise identical for any unit partition (the reference's chunk-invariance contract,
//    l1reg.py:183-186, test_l1reg.py:63-72).
#include "common.cuh"
#include "filter_pair.cuh"

#include <algorithm>
#include <cstdlib>

int l1f_tc_pair_dispatch(const float* X, int64_t ldx, int s, int64_t n_units, const float* A, int64_t lda, int k,
                         double tol, double rho, double beta0, double beta_max, int max_iter, float* Z, int64_t ldz,
                         int32_t* iters, float* res, uint8_t* status, const l1f::tcf::Second& two, cudaStream_t st);

namespace l1f {
namespace filt {

constexpr int TS = 32;   // unit slots per CTA
constexpr int NT = 256;  // threads per CTA
constexpr int RC = 32;   // rows per chunk
constexpr int VS = TS + 4;
constexpr int kStallIters = 20;       // STAGNATION_ITERS, l1reg.py:34
constexpr double kStallEps = 1e-12;   // STAGNATION_EPS, l1reg.py:33

template <typename T>
struct SlotState {
  int unit[TS], it[TS], stalled[TS], state[TS], finish[TS], buf[TS];
  T beta_cur[TS], beta_next[TS], inv_next[TS], beta_max[TS], thresh[TS], prev_res[TS], res[TS];
  uint8_t code[TS];
};

template <typename T> struct V4;
template <> struct V4<float> {
  __device__ static __forceinline__ void load(const float* p, float (&v)[4]) {
    float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
};
template <> struct V4<double> {
  __device__ static __forceinline__ void load(const double* p, double (&v)[4]) {
    double2 a = *reinterpret_cast<const double2*>(p), b = *reinterpret_cast<const double2*>(p + 2);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
};

template <typename T>
__device__ __forceinline__ T recip(T b) { return T(1) / b; }

// L1F_OPT_FILTER_STREAMING forces the streaming kernel (A/B comparisons, tests)
inline bool force_streaming() { return option(L1F_OPT_FILTER_STREAMING) != 0; }

struct Params {
  int s, s_pad, k, kp;
  int64_t n_units, ldx, ldz, lde;
  int max_iter;
  double tol, rho, beta0, beta_max;
};

// ---------------------------------------------------------------- prologue kernels
template <typename T>
__global__ void pad_dictionary_kernel(const T* __restrict__ A, int64_t lda, int s, int k, int s_pad, int kp,
                                      T* __restrict__ Ap) {
  const int64_t total = (int64_t)s_pad * kp;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / kp), t = (int)(e % kp);
    Ap[e] = (r < s && t < k) ? A[(int64_t)r * lda + t] : T(0);
  }
}

// per-unit ||x||_inf (l1reg.py:65); outputs of dead units (scale 0, l1reg.py:74-75) and of
// max_iter <= 0 (l1reg.py:130-135 with an empty loop) are written here.
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

// ---------------------------------------------------------------- the ADM kernel
template <typename T, int KJ>
__global__ void __launch_bounds__(NT, 2)
adm_filter_kernel(const T* __restrict__ X, const T* __restrict__ Ap, const T* __restrict__ scale, Params P,
                  int* __restrict__ queue, T* __restrict__ ws, T* __restrict__ Z, T* __restrict__ E,
                  int32_t* __restrict__ iters, T* __restrict__ res, uint8_t* __restrict__ status) {
  constexpr int KP = 32 * KJ;
  constexpr int AS = KP + 1;  // odd row stride: conflict-free column reads in phase a
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* As = reinterpret_cast<T*>(smem_raw);  // [RC][AS]
  T* zs = As + RC * AS;                    // [KP][TS]
  T* Vs = zs + KP * TS;                    // [RC][VS]
  __shared__ SlotState<T> ss;

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int s = P.s, s_pad = P.s_pad;
  T* ws_y = ws + (int64_t)blockIdx.x * 3 * TS * s_pad;
  T* ws_e0 = ws_y + (int64_t)TS * s_pad;
  T* ws_e1 = ws_e0 + (int64_t)TS * s_pad;
  const T tol = (T)P.tol, rho = (T)P.rho;

  auto refill = [&](int slot) {
    for (;;) {
      const int64_t u = atomicAdd(queue, 1);
      if (u >= P.n_units) { ss.state[slot] = 0; ss.unit[slot] = -1; return; }
      const T sc = scale[u];
      if (!(sc > T(0)) || P.max_iter <= 0) continue;  // handled by unit_scale_kernel
      const T b0 = P.beta0 > 0 ? (T)P.beta0 : recip(sc);
      ss.unit[slot] = (int)u;
      ss.state[slot] = 1;
      ss.it[slot] = 0;
      ss.stalled[slot] = 0;
      ss.buf[slot] = 0;
      ss.beta_cur[slot] = b0;
      ss.beta_next[slot] = b0;
      ss.inv_next[slot] = recip(b0);
      ss.beta_max[slot] = P.beta_max > 0 ? (T)P.beta_max : (T)1e7 * b0;
      ss.thresh[slot] = tol * sc;
      ss.prev_res[slot] = Limits<T>::inf();
      return;
    }
  };

  if (tid < TS) refill(tid);
  for (int e = tid; e < KP * TS; e += NT) zs[e] = T(0);
  __syncthreads();

  // phase-c mapping: k rows {tk + 32 j}, slots {4 tu .. 4 tu + 3}
  const int tk = tid / 8, tu = tid % 8;
  T acc[KJ][4];
#pragma unroll
  for (int j = 0; j < KJ; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[j][q] = T(0);

  const int nchunks = s_pad / RC;
  for (;;) {
    if (!__syncthreads_or(tid < TS && ss.state[tid] == 1)) break;

    T rmax[4] = {T(0), T(0), T(0), T(0)};
    for (int c = 0; c < nchunks; ++c) {
      const int row0 = c * RC;
      __syncthreads();  // previous chunk's phase c is done with As / Vs
      for (int e = tid; e < RC * KP; e += NT) {
        const int r = e / KP, t = e - (e / KP) * KP;
        As[r * AS + t] = Ap[(int64_t)(row0 + r) * KP + t];
      }
      __syncthreads();

      // ---- phase a: (A z)[row] for the 4 slots of this warp; phase b: elementwise ADM
      {
        T az[4] = {T(0), T(0), T(0), T(0)};
        const T* arow = As + lane * AS;
        const T* zcol = zs + 4 * warp;
#pragma unroll 8
        for (int t = 0; t < KP; ++t) {
          const T a = arow[t];
          T z4[4];
          V4<T>::load(zcol + t * TS, z4);
#pragma unroll
          for (int q = 0; q < 4; ++q) az[q] = fma(a, z4[q], az[q]);
        }
        const int i = row0 + lane;
        const bool in = i < s;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int slot = 4 * warp + q;
          T v = T(0);
          if (ss.state[slot] == 1) {
            const int64_t u = ss.unit[slot];
            const int it = ss.it[slot];
            T* ycol = ws_y + (int64_t)slot * s_pad;
            T* e_rd = (ss.buf[slot] ? ws_e1 : ws_e0) + (int64_t)slot * s_pad;
            T* e_wr = (ss.buf[slot] ? ws_e0 : ws_e1) + (int64_t)slot * s_pad;
            const T x = in ? X[u * P.ldx + i] : T(0);
            T y, d;
            if (it == 0) {
              y = T(0);
              d = x;
            } else {
              const T e_old = in ? e_rd[i] : T(0);
              y = in ? ycol[i] : T(0);
              d = x - az[q];
              const T r = d - e_old;
              rmax[q] = tmax(rmax[q], tabs(r));
              y = y + ss.beta_cur[slot] * r;
            }
            const T ib = ss.inv_next[slot];
            const T yb = y * ib;
            const T e = shrink(d + yb, ib);
            v = (x - e) + yb;
            if (in) {
              ycol[i] = y;
              e_wr[i] = e;
            }
          }
          Vs[lane * VS + slot] = v;
        }
      }
      __syncthreads();

      // ---- phase c: acc(k x slots) += A_chunk^T V_chunk  (next iteration's z)
#pragma unroll 4
      for (int r = 0; r < RC; ++r) {
        T v4[4];
        V4<T>::load(Vs + r * VS + 4 * tu, v4);
        const T* arow = As + r * AS + tk;
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
          const T a = arow[32 * j];
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[j][q] = fma(a, v4[q], acc[j][q]);
        }
      }
    }

    // ---- end of pass: per-slot max|r| (warp w owns slots 4w..4w+3 in phase b)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const T m = warp_max(rmax[q]);
      if (lane == 0) ss.res[4 * warp + q] = m;
    }
    __syncthreads();

    // ---- per-slot decision (l1reg.py:100-128)
    if (tid < TS) {
      const int slot = tid;
      ss.finish[slot] = 0;
      if (ss.state[slot] == 1) {
        bool fin = false;
        if (ss.it[slot] > 0) {
          const T r = ss.res[slot];
          const T prev = ss.prev_res[slot];
          const T rel = tabs(r - prev) / tmax(r, Limits<T>::tiny());
          ss.stalled[slot] = (rel < (T)kStallEps) ? ss.stalled[slot] + 1 : 0;
          ss.prev_res[slot] = r;
          const bool ok = r <= ss.thresh[slot];
          if (ok) { fin = true; ss.code[slot] = L1F_UNIT_OK; }
          else if (ss.stalled[slot] >= kStallIters) { fin = true; ss.code[slot] = L1F_UNIT_STALLED; }
          else if (ss.it[slot] >= P.max_iter) { fin = true; ss.code[slot] = L1F_UNIT_MAXITER; }
        }
        if (fin) {
          ss.finish[slot] = 1;
        } else {
          ss.it[slot] += 1;
          const T bc = ss.beta_next[slot];
          ss.beta_cur[slot] = bc;
          T bn = rho * bc;  // beta = min(rho * beta, beta_max), l1reg.py:128
          if (bn > ss.beta_max[slot]) bn = ss.beta_max[slot];
          ss.beta_next[slot] = bn;
          ss.inv_next[slot] = recip(bn);
          ss.buf[slot] ^= 1;
        }
      }
    }
    __syncthreads();

    // ---- outputs of finished units: z (current zs), e (current e buffer)
    for (int slot = warp; slot < TS; slot += NT / 32) {
      if (!ss.finish[slot]) continue;
      const int64_t u = ss.unit[slot];
      for (int t = lane; t < P.k; t += 32) Z[u * P.ldz + t] = zs[t * TS + slot];
      if (E) {
        const T* e_rd = (ss.buf[slot] ? ws_e1 : ws_e0) + (int64_t)slot * s_pad;
        for (int i = lane; i < s; i += 32) E[u * P.lde + i] = e_rd[i];
      }
      if (lane == 0) {
        if (iters) iters[u] = ss.it[slot];
        if (res) res[u] = ss.res[slot];
        if (status) status[u] = ss.code[slot];
      }
    }
    __syncthreads();

    // ---- install next z for continuing slots, zero for finished / empty ones
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int slot = 4 * tu + q;
      const bool keep = ss.state[slot] == 1 && !ss.finish[slot];
#pragma unroll
      for (int j = 0; j < KJ; ++j) {
        zs[(tk + 32 * j) * TS + slot] = keep ? acc[j][q] : T(0);
        acc[j][q] = T(0);
      }
    }
    if (tid < TS && ss.finish[tid]) refill(tid);
    __syncthreads();
  }
}

template <typename T, int KJ>
size_t smem_bytes() {
  constexpr int KP = 32 * KJ;
  return sizeof(T) * ((size_t)RC * (KP + 1) + (size_t)KP * TS + (size_t)RC * VS);
}

template <typename T, int KJ>
int grid_blocks(size_t smem) {
  static int cached = -1;
  if (cached < 0) {
    cudaFuncSetAttribute(adm_filter_kernel<T, KJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, adm_filter_kernel<T, KJ>, NT, smem) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    cached = per_sm * num_sms();
  }
  return cached;
}

struct Layout {
  size_t ap_off, scale_off, queue_off, ws_off, total;
  int grid;
};

template <typename T, int KJ>
Layout layout(int s, int64_t n_units) {
  Layout L;
  const int s_pad = (int)ceil_div(s, RC) * RC, kp = 32 * KJ;
  const int64_t want = ceil_div(n_units, TS);
  int g = grid_blocks<T, KJ>(smem_bytes<T, KJ>());
  if (want < g) g = (int)(want < 1 ? 1 : want);
  L.grid = g;
  auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
  L.ap_off = 0;
  L.scale_off = al(L.ap_off + sizeof(T) * (size_t)s_pad * kp);
  L.queue_off = al(L.scale_off + sizeof(T) * (size_t)(n_units > 0 ? n_units : 1));
  L.ws_off = al(L.queue_off + sizeof(int));
  L.total = al(L.ws_off + sizeof(T) * (size_t)g * 3 * TS * s_pad);
  return L;
}

template <typename T, int KJ>
int run(const T* X, int64_t ldx, int s, int64_t n_units, const T* A, int64_t lda, int k, double tol, double rho,
        double beta0, double beta_max, int max_iter, T* Z, int64_t ldz, T* E, int64_t lde, int32_t* iters, T* res,
        uint8_t* status, void* workspace, size_t ws_bytes, cudaStream_t st, bool query, size_t* need) {
  const size_t smem = smem_bytes<T, KJ>();
  Layout L = layout<T, KJ>(s, n_units);
  if (query) { *need = L.total; return L1F_OK; }
  void* owned = nullptr;
  if (!workspace) {
    L1F_CUDA_TRY(cudaMallocAsync(&owned, L.total, st));
    workspace = owned;
  } else {
    L1F_REQUIRE(ws_bytes >= L.total, L1F_ERR_ARG, "filter: workspace too small (%zu < %zu)", ws_bytes, L.total);
  }
  unsigned char* w = (unsigned char*)workspace;
  Params P;
  P.s = s; P.s_pad = (int)ceil_div(s, RC) * RC; P.k = k; P.kp = 32 * KJ;
  P.n_units = n_units; P.ldx = ldx; P.ldz = ldz; P.lde = lde; P.max_iter = max_iter;
  P.tol = tol; P.rho = rho; P.beta0 = beta0; P.beta_max = beta_max;
  T* Ap = (T*)(w + L.ap_off);
  T* scale = (T*)(w + L.scale_off);
  int* queue = (int*)(w + L.queue_off);
  T* ws = (T*)(w + L.ws_off);
  int rc = L1F_OK;
  do {
    pad_dictionary_kernel<T><<<256, 256, 0, st>>>(A, lda, s, k, P.s_pad, P.kp, Ap);
    if (cudaGetLastError() != cudaSuccess) { rc = L1F_ERR_CUDA; break; }
    unit_scale_kernel<T><<<(unsigned)std::min<int64_t>(ceil_div(n_units, 8), 65535), 256, 0, st>>>(
        X, P, scale, Z, E, iters, res, status);
    if (cudaGetLastError() != cudaSuccess) { rc = L1F_ERR_CUDA; break; }
    if (max_iter <= 0) break;
    if (cudaMemsetAsync(queue, 0, sizeof(int), st) != cudaSuccess) { rc = L1F_ERR_CUDA; break; }
    adm_filter_kernel<T, KJ><<<L.grid, NT, smem, st>>>(X, Ap, scale, P, queue, ws, Z, E, iters, res, status);
    if (cudaGetLastError() != cudaSuccess) { rc = L1F_ERR_CUDA; break; }
  } while (0);
  if (rc != L1F_OK) set_error("filter: kernel launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  if (owned) cudaFreeAsync(owned, st);
  return rc;
}

// ---------------------------------------------------------------- any-k kernel (k > 256)
// One CTA solves one unit at a time; the unit's state (y, e double buffer, v, z, A z) lives in a
// per-CTA workspace, and the dictionary is read from two padded copies in global memory (row-major
// for A^T v, transposed for A z) so both contractions are coalesced.  Same recurrence, same
// sequential FMA order over t (A z) and over rows (A^T v) as the streaming kernel above, so the
// per-unit arithmetic matches it and is independent of the grid.  The refusal of k > 256 it replaces
// was a register limit of the streaming kernel, not of the algorithm (l1reg.py:59-137 takes any k).
constexpr int GT = 256;  // threads per CTA of the any-k kernel

template <typename T>
__global__ void __launch_bounds__(GT)
adm_generic_kernel(const T* __restrict__ X, const T* __restrict__ Ap, const T* __restrict__ At,
                   const T* __restrict__ scale, Params P, T* __restrict__ ws, T* __restrict__ Z, T* __restrict__ E,
                   int32_t* __restrict__ iters, T* __restrict__ res, uint8_t* __restrict__ status) {
  const int s = P.s, k = P.k, kp = P.kp, s_pad = P.s_pad;
  const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
  T* y = ws + (int64_t)blockIdx.x * (4 * (int64_t)s_pad + 2 * (int64_t)kp);
  T* e0 = y + s_pad;
  T* e1 = e0 + s_pad;
  T* v = e1 + s_pad;
  T* z = v + s_pad;
  T* zn = z + kp;
  __shared__ T red[GT / 32];
  __shared__ int fin_s;
  const T tol = (T)P.tol, rho = (T)P.rho;
  for (int64_t u = blockIdx.x; u < P.n_units; u += gridDim.x) {
    const T sc = scale[u];
    if (!(sc > T(0)) || P.max_iter <= 0) continue;  // written by unit_scale_kernel
    const T* x = X + u * P.ldx;
    const T b0 = P.beta0 > 0 ? (T)P.beta0 : recip(sc);
    const T bmax = P.beta_max > 0 ? (T)P.beta_max : (T)1e7 * b0;
    const T thresh = tol * sc;
    T beta_cur = b0, beta_next = b0, inv_next = recip(b0), prev_res = Limits<T>::inf(), r_last = T(0);
    int it = 0, stalled = 0, buf = 0;
    uint8_t code = L1F_UNIT_OK;
    for (int t = tid; t < kp; t += GT) z[t] = T(0);
    __syncthreads();
    for (;;) {
      // phase a + b: rows i
      T rmax = T(0);
      const T* e_rd = buf ? e1 : e0;
      T* e_wr = buf ? e0 : e1;
      for (int i = tid; i < s; i += GT) {
        T az = T(0);
        for (int t = 0; t < kp; ++t) az = fma(At[(int64_t)t * s_pad + i], z[t], az);
        const T xi = x[i];
        T yi, d;
        if (it == 0) {
          yi = T(0);
          d = xi;
        } else {
          d = xi - az;
          const T r = d - e_rd[i];
          rmax = tmax(rmax, tabs(r));
          yi = y[i] + beta_cur * r;
        }
        const T yb = yi * inv_next;
        const T e = shrink(d + yb, inv_next);
        v[i] = (xi - e) + yb;
        y[i] = yi;
        e_wr[i] = e;
      }
      rmax = warp_max(rmax);
      if (lane == 0) red[warp] = rmax;
      __syncthreads();
      if (tid == 0) {
        T m = T(0);
        for (int w = 0; w < GT / 32; ++w) m = tmax(m, red[w]);
        int fin = 0;
        if (it > 0) {
          const T rel = tabs(m - prev_res) / tmax(m, Limits<T>::tiny());
          stalled = (rel < (T)kStallEps) ? stalled + 1 : 0;
          prev_res = m;
          r_last = m;
          if (m <= thresh) { fin = 1; code = L1F_UNIT_OK; }
          else if (stalled >= kStallIters) { fin = 1; code = L1F_UNIT_STALLED; }
          else if (it >= P.max_iter) { fin = 1; code = L1F_UNIT_MAXITER; }
        }
        fin_s = fin;
      }
      __syncthreads();
      // every thread mirrors the scalar schedule (thread 0 owns the decision)
      const int fin = fin_s;
      if (fin) {
        for (int t = tid; t < k; t += GT) Z[u * P.ldz + t] = z[t];
        if (E)
          for (int i = tid; i < s; i += GT) E[u * P.lde + i] = e_rd[i];
        if (tid == 0) {
          if (iters) iters[u] = it;
          if (res) res[u] = r_last;
          if (status) status[u] = code;
        }
        __syncthreads();
        break;
      }
      it += 1;
      beta_cur = beta_next;
      T bn = rho * beta_cur;
      if (bn > bmax) bn = bmax;
      beta_next = bn;
      inv_next = recip(bn);
      buf ^= 1;
      // phase c: z_{it} = A^T v, sequential over rows
      for (int t = tid; t < kp; t += GT) {
        T acc = T(0);
        for (int i = 0; i < s; ++i) acc = fma(Ap[(int64_t)i * kp + t], v[i], acc);
        zn[t] = acc;
      }
      __syncthreads();
      for (int t = tid; t < kp; t += GT) z[t] = zn[t];
      __syncthreads();
    }
  }
}

template <typename T>
__global__ void transpose_dictionary_kernel(const T* __restrict__ A, int64_t lda, int s, int k, int s_pad, int kp,
                                            T* __restrict__ At) {
  const int64_t total = (int64_t)s_pad * kp;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(e / s_pad), r = (int)(e % s_pad);
    At[e] = (r < s && t < k) ? A[(int64_t)r * lda + t] : T(0);
  }
}

template <typename T>
int run_generic(const T* X, int64_t ldx, int s, int64_t n_units, const T* A, int64_t lda, int k, double tol,
                double rho, double beta0, double beta_max, int max_iter, T* Z, int64_t ldz, T* E, int64_t lde,
                int32_t* iters, T* res, uint8_t* status, void* workspace, size_t ws_bytes, cudaStream_t st,
                bool query, size_t* need) {
  const int s_pad = (int)ceil_div(s, RC) * RC, kp = (int)ceil_div(k, 32) * 32;
  const int64_t g64 = std::min<int64_t>(std::max<int64_t>(n_units, 1), (int64_t)num_sms() * 4);
  const int grid = (int)g64;
  auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
  const size_t ap_off = 0;
  const size_t at_off = al(ap_off + sizeof(T) * (size_t)s_pad * kp);
  const size_t scale_off = al(at_off + sizeof(T) * (size_t)s_pad * kp);
  const size_t ws_off = al(scale_off + sizeof(T) * (size_t)(n_units > 0 ? n_units : 1));
  const size_t total = al(ws_off + sizeof(T) * (size_t)grid * (4 * (size_t)s_pad + 2 * (size_t)kp));
  if (query) {
    *need = total;
    return L1F_OK;
  }
  void* owned = nullptr;
  if (!workspace) {
    L1F_CUDA_TRY(cudaMallocAsync(&owned, total, st));
    workspace = owned;
  } else {
    L1F_REQUIRE(ws_bytes >= total, L1F_ERR_ARG, "filter: workspace too small (%zu < %zu)", ws_bytes, total);
  }
  unsigned char* w = (unsigned char*)workspace;
  Params P;
  P.s = s; P.s_pad = s_pad; P.k = k; P.kp = kp;
  P.n_units = n_units; P.ldx = ldx; P.ldz = ldz; P.lde = lde; P.max_iter = max_iter;
  P.tol = tol; P.rho = rho; P.beta0 = beta0; P.beta_max = beta_max;
  T* Ap = (T*)(w + ap_off);
  T* At = (T*)(w + at_off);
  T* scale = (T*)(w + scale_off);
  T* ws = (T*)(w + ws_off);
  int rc = L1F_OK;
  do {
    pad_dictionary_kernel<T><<<256, 256, 0, st>>>(A, lda, s, k, s_pad, kp, Ap);
    transpose_dictionary_kernel<T><<<256, 256, 0, st>>>(A, lda, s, k, s_pad, kp, At);
    unit_scale_kernel<T><<<(unsigned)std::min<int64_t>(ceil_div(n_units, 8), 65535), 256, 0, st>>>(
        X, P, scale, Z, E, iters, res, status);
    if (cudaGetLastError() != cudaSuccess) { rc = L1F_ERR_CUDA; break; }
    if (max_iter <= 0) break;
    adm_generic_kernel<T><<<grid, GT, 0, st>>>(X, Ap, At, scale, P, ws, Z, E, iters, res, status);
    if (cudaGetLastError() != cudaSuccess) { rc = L1F_ERR_CUDA; break; }
  } while (0);
  if (rc != L1F_OK) set_error("filter: kernel launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  if (owned) cudaFreeAsync(owned, st);
  return rc;
}

template <typename T>
int dispatch(const T* X, int64_t ldx, int s, int64_t n_units, const T* A, int64_t lda, int k, double tol,
             double rho, double beta0, double beta_max, int max_iter, T* Z, int64_t ldz, T* E, int64_t lde,
             int32_t* iters, T* res, uint8_t* status, void* workspace, size_t ws_bytes, cudaStream_t st,
             bool query, size_t* need) {
  const int kj = (int)ceil_div(k, 32);
#define L1F_KJ(N)                                                                                      \
  case N:                                                                                              \
    return run<T, N>(X, ldx, s, n_units, A, lda, k, tol, rho, beta0, beta_max, max_iter, Z, ldz, E, lde, \
                     iters, res, status, workspace, ws_bytes, st, query, need);
  switch (kj < 1 ? 1 : kj) {
    L1F_KJ(1) L1F_KJ(2) L1F_KJ(3) L1F_KJ(4) L1F_KJ(5) L1F_KJ(6) L1F_KJ(7) L1F_KJ(8)
    default:  // k > 256: the any-k kernel
      return run_generic<T>(X, ldx, s, n_units, A, lda, k, tol, rho, beta0, beta_max, max_iter, Z, ldz, E, lde,
                            iters, res, status, workspace, ws_bytes, st, query, need);
  }
#undef L1F_KJ
}

}  // namespace filt
}  // namespace l1f

template <typename T>
int l1f_resident_dispatch(const T* X, int64_t ldx, int s, int64_t n_units, const T* A, int64_t lda, int k,
                          double tol, double rho, double beta0, double beta_max, int max_iter, T* Z, int64_t ldz,
                          T* E, int64_t lde, int32_t* iters, T* res, uint8_t* status, void* workspace,
                          size_t ws_bytes, cudaStream_t st, bool query, size_t* need);

template <typename T>
int l1f_small_dispatch(const T* X, int64_t ldx, int s, int64_t n_units, const T* A, int64_t lda, int k, double tol,
                       double rho, double beta0, double beta_max, int max_iter, T* Z, int64_t ldz, T* E, int64_t lde,
                       int32_t* iters, T* res, uint8_t* status, void* workspace, size_t ws_bytes, cudaStream_t st,
                       bool query, size_t* need, l1f::tcf::NotifyHost* nh);

int l1f_tc_dispatch(const float* X, int64_t ldx, int s, int64_t n_units, const float* A, int64_t lda, int k,
                    double tol, double rho, double beta0, double beta_max, int max_iter, float* Z, int64_t ldz,
                    float* E, int64_t lde, int32_t* iters, float* res, uint8_t* status, void* workspace,
                    size_t ws_bytes, cudaStream_t st, bool query, size_t* need, l1f::tcf::NotifyHost* nh);

namespace l1f {
namespace filt {

template <typename T>
int tc_dispatch(const T*, int64_t, int, int64_t, const T*, int64_t, int, double, double, double, double, int, T*,
                int64_t, T*, int64_t, int32_t*, T*, uint8_t*, void*, size_t, cudaStream_t, bool, size_t*) {
  return L1F_ERR_UNSUPPORTED;  // fp64: no tensor-core path
}
template <>
int tc_dispatch<float>(const float* X, int64_t ldx, int s, int64_t n_units, const float* A, int64_t lda, int k,
                       double tol, double rho, double beta0, double beta_max, int max_iter, float* Z, int64_t ldz,
                       float* E, int64_t lde, int32_t* iters, float* res, uint8_t* status, void* workspace,
                       size_t ws_bytes, cudaStream_t st, bool query, size_t* need) {
  return l1f_tc_dispatch(X, ldx, s, n_units, A, lda, k, tol, rho, beta0, beta_max, max_iter, Z, ldz, E, lde, iters,
                         res, status, workspace, ws_bytes, st, query, need, nullptr);
}

// small-k group kernel (filter_small.cu), tensor-core kernel (filter_tc.cu, fp32), resident-state kernel (filter_resident.cu) when a geometry fits, else the streaming kernel
template <typename T>
int select(const T* X, int64_t ldx, int s, int64_t n_units, const T* A, int64_t lda, int k, double tol,
           double rho, double beta0, double beta_max, int max_iter, T* Z, int64_t ldz, T* E, int64_t lde,
           int32_t* iters, T* res, uint8_t* status, void* workspace, size_t ws_bytes, cudaStream_t st,
           bool query, size_t* need) {
  if (!force_streaming()) {
    const int rs = l1f_small_dispatch<T>(X, ldx, s, n_units, A, lda, k, tol, rho, beta0, beta_max, max_iter, Z, ldz,
                                         E, lde, iters, res, status, workspace, ws_bytes, st, query, need, nullptr);
    if (rs != L1F_ERR_UNSUPPORTED) return rs;
    const int rt = tc_dispatch<T>(X, ldx, s, n_units, A, lda, k, tol, rho, beta0, beta_max, max_iter, Z, ldz, E, lde,
                                  iters, res, status, workspace, ws_bytes, st, query, need);
    if (rt != L1F_ERR_UNSUPPORTED) return rt;
    const int rc = l1f_resident_dispatch<T>(X, ldx, s, n_units, A, lda, k, tol, rho, beta0, beta_max, max_iter, Z,
                                            ldz, E, lde, iters, res, status, workspace, ws_bytes, st, query, need);
    if (rc != L1F_ERR_UNSUPPORTED) return rc;
  }
  return dispatch<T>(X, ldx, s, n_units, A, lda, k, tol, rho, beta0, beta_max, max_iter, Z, ldz, E, lde, iters,
                     res, status, workspace, ws_bytes, st, query, need);
}

template <typename T>
int filter_entry(const T* X, int64_t ldx, int32_t s, int64_t n_units, const T* A, int64_t lda, int32_t k, T tol,
                 T rho, T beta0, T beta_max, int32_t max_iter, T* Z, int64_t ldz, T* E, int64_t lde,
                 int32_t* iters, T* res, uint8_t* status, void* workspace, size_t ws_bytes, void* stream) {
  L1F_REQUIRE(s >= 1 && k >= 1 && n_units >= 0, L1F_ERR_ARG, "filter: need s >= 1, k >= 1, n_units >= 0");
  L1F_REQUIRE(ldx >= s && ldz >= k && lda >= k && (!E || lde >= s), L1F_ERR_ARG, "filter: leading dimension too small");
  L1F_REQUIRE(n_units < (int64_t)INT32_MAX, L1F_ERR_UNSUPPORTED, "filter: too many units");
  L1F_REQUIRE(rho > T(1) && tol > T(0), L1F_ERR_ARG, "filter: need rho > 1 and tol > 0");
  if (n_units == 0) return L1F_OK;
  return select<T>(X, ldx, s, n_units, A, lda, k, tol, rho, beta0, beta_max, max_iter, Z, ldz, E, lde, iters,
                     res, status, workspace, ws_bytes, (cudaStream_t)stream, false, nullptr);
}

}  // namespace filt
}  // namespace l1f

using namespace l1f;

extern "C" size_t l1f_filter_workspace_bytes(int dtype, int32_t s, int32_t k, int64_t n_units) {
  size_t need = 0;
  if (s < 1 || k < 1 || n_units < 0) return 0;
  if (dtype == L1F_F32)
    filt::select<float>(nullptr, s, s, n_units, nullptr, k, k, 1e-7, 1.5, 0, 0, 1, nullptr, k, nullptr, s,
                          nullptr, nullptr, nullptr, nullptr, 0, nullptr, true, &need);
  else
    filt::select<double>(nullptr, s, s, n_units, nullptr, k, k, 1e-7, 1.5, 0, 0, 1, nullptr, k, nullptr, s,
                           nullptr, nullptr, nullptr, nullptr, 0, nullptr, true, &need);
  return need;
}

extern "C" int l1f_filter_f32(const float* X, int64_t ldx, int32_t s, int64_t n_units, const float* A, int64_t lda,
                              int32_t k, float tol, float rho, float beta0, float beta_max, int32_t max_iter,
                              float* Z, int64_t ldz, float* E, int64_t lde, int32_t* iters, float* res,
                              uint8_t* status, void* workspace, size_t workspace_bytes, void* stream) {
  return filt::filter_entry<float>(X, ldx, s, n_units, A, lda, k, tol, rho, beta0, beta_max, max_iter, Z, ldz, E,
                                   lde, iters, res, status, workspace, workspace_bytes, stream);
}

extern "C" int l1f_filter_f64(const double* X, int64_t ldx, int32_t s, int64_t n_units, const double* A,
                              int64_t lda, int32_t k, double tol, double rho, double beta0, double beta_max,
                              int32_t max_iter, double* Z, int64_t ldz, double* E, int64_t lde, int32_t* iters,
                              double* res, uint8_t* status, void* workspace, size_t workspace_bytes, void* stream) {
  return filt::filter_entry<double>(X, ldx, s, n_units, A, lda, k, tol, rho, beta0, beta_max, max_iter, Z, ldz, E,
                                    lde, iters, res, status, workspace, workspace_bytes, stream);
}

extern "C" int l1f_filter_pair_f32(const float* X1, int64_t ldx1, int64_t n1, const float* A1, int64_t lda1, float* Z1,
                                   int64_t ldz1, int32_t* iters1, float* res1, uint8_t* status1, const float* X2,
                                   int64_t ldx2, int64_t n2, const float* A2, int64_t lda2, float* Z2, int64_t ldz2,
                                   int32_t* iters2, float* res2, uint8_t* status2, int32_t s, int32_t k, float tol,
                                   float rho, float beta0, float beta_max, int32_t max_iter, int32_t mode,
                                   void* stream) {
  L1F_REQUIRE(s >= 1 && k >= 1 && n1 >= 0 && n2 >= 0, L1F_ERR_ARG, "filter_pair: need s >= 1, k >= 1, n >= 0");
  L1F_REQUIRE((n1 == 0 || (ldx1 >= s && ldz1 >= k && lda1 >= k)) && (n2 == 0 || (ldx2 >= s && ldz2 >= k && lda2 >= k)),
              L1F_ERR_ARG, "filter_pair: leading dimension too small");
  L1F_REQUIRE(n1 < (int64_t)INT32_MAX && n2 < (int64_t)INT32_MAX, L1F_ERR_UNSUPPORTED, "filter_pair: too many units");
  L1F_REQUIRE(rho > 1.f && tol > 0.f, L1F_ERR_ARG, "filter_pair: need rho > 1 and tol > 0");
  L1F_REQUIRE(mode >= 0 && mode <= 2, L1F_ERR_ARG, "filter_pair: mode must be 0, 1 or 2");
  cudaStream_t st = (cudaStream_t)stream;
  if (n1 > 0 && n2 > 0 && !filt::force_streaming()) {
    const tcf::Second two{X2, ldx2, n2, A2, lda2, Z2, ldz2, iters2, res2, status2, mode, nullptr};
    const int rc = l1f_tc_pair_dispatch(X1, ldx1, s, n1, A1, lda1, k, tol, rho, beta0, beta_max, max_iter, Z1, ldz1,
                                        iters1, res1, status1, two, st);
    if (rc != L1F_ERR_UNSUPPORTED) return rc;
  }
  int rc = l1f_filter_f32(X1, ldx1, s, n1, A1, lda1, k, tol, rho, beta0, beta_max, max_iter, Z1, ldz1, nullptr, s,
                          iters1, res1, status1, nullptr, 0, stream);
  if (rc != L1F_OK) return rc;
  return l1f_filter_f32(X2, ldx2, s, n2, A2, lda2, k, tol, rho, beta0, beta_max, max_iter, Z2, ldz2, nullptr, s, iters2,
                        res2, status2, nullptr, 0, stream);
}

extern "C" int l1f_filter_pair_plan_f32(int32_t s, int32_t k, int64_t n1, int64_t n2, int32_t* one_grid) {
  L1F_REQUIRE(s >= 1 && k >= 1 && n1 >= 0 && n2 >= 0 && one_grid, L1F_ERR_ARG, "filter_pair_plan: bad arguments");
  *one_grid = 0;
  if (n1 == 0 || n2 == 0 || filt::force_streaming()) return L1F_OK;
  int plan = 0;
  tcf::Second two{nullptr, s, n2, nullptr, k, nullptr, k, nullptr, nullptr, nullptr, 3, &plan};
  const int rc = l1f_tc_pair_dispatch(nullptr, s, s, n1, nullptr, k, k, 1e-7, 1.5, 0.0, 0.0, 1000, nullptr, k, nullptr,
                                      nullptr, nullptr, two, nullptr);
  if (rc == L1F_OK) *one_grid = plan;
  return rc == L1F_ERR_UNSUPPORTED ? L1F_OK : rc;
}
