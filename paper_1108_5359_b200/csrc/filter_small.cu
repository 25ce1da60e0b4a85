// Small-rank ADM filter kernel (K3, k <= 16): one group of L lanes per unit.
//
// Same per-unit semantics as filter.cu / filter_resident.cu (reference: _solve_block,
// pkg/src/l1pcp/l1reg.py:59-137).  For k <= 16 (configs 1 and 4: s = 100, k = 10) the
// cluster kernel's per-pass barriers cost more than the arithmetic, so each unit is
// solved by an independent group of L lanes (L = 16 or 32):
//  * lane j of a group owns rows {j, j+L, j+2L, ...} (interleaved -> coalesced x loads) and
//    keeps x, y, l = x - e of those rows in registers; z (k values) is replicated in the group;
//  * the dictionary A (s x k) is resident in shared memory, shared by all groups of the CTA;
//  * one ADM iteration per pass, fused per row: az = A[row] . z, the cancellation-free
//    elementwise update (see filter_resident.cu), acc += A[row] * v; then a butterfly
//    all-reduce of acc (bitwise identical in every lane: IEEE addition is commutative) and of
//    max|r|; every lane takes the same stop decision (l1reg.py:100-128);
//  * groups pull units from a global counter; a unit's arithmetic never depends on the group.
#include "common.cuh"
#include "filter_pair.cuh"

#include <algorithm>

namespace l1f {
namespace small {

constexpr int kStallIters = 20;
constexpr double kStallEps = 1e-12;

struct Params {
  int s, k, s_pad;
  int64_t n_units, ldx, ldz, lde;
  int max_iter;
  double tol, rho, beta0, beta_max;
  // progress notification (l1f_rowfilter_reconstruct_small): + 1 to ncnt[nrows[u] >> 7] once
  // z_u is in global memory, + 1 to *nres per started block (null: off)
  const int64_t* nrows = nullptr;
  unsigned* ncnt = nullptr;
  unsigned* nres = nullptr;
};

template <typename T>
__device__ __forceinline__ T shfl_xor(unsigned mask, T v, int o) { return __shfl_xor_sync(mask, v, o); }

// <= 192 registers: two 128-thread blocks plus the 128-thread reconstruction CTA that
// l1f_rowfilter_reconstruct_small runs beside them fit one SM's register file
template <typename T, int KM, int RPL, int L, bool WE>
__global__ void __maxnreg__(192)
adm_small_kernel(const T* __restrict__ X, const T* __restrict__ A, int64_t lda, const T* __restrict__ scale, Params P,
                 int* __restrict__ queue, T* __restrict__ Z, T* __restrict__ E, int32_t* __restrict__ iters,
                 T* __restrict__ res_out, uint8_t* __restrict__ status) {
  constexpr int AST = KM + 1;  // odd row stride: the lanes of a group read distinct banks
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (P.nres && threadIdx.x == 0) atomicAdd(P.nres, 1u);
  T* As = reinterpret_cast<T*>(smem_raw);  // [s_pad][AST], zero padded
  for (int e = threadIdx.x; e < P.s_pad * AST; e += blockDim.x) {
    const int r = e / AST, t = e - (e / AST) * AST;
    As[e] = (r < P.s && t < P.k) ? A[(int64_t)r * lda + t] : T(0);
  }
  __syncthreads();

  const int lane = threadIdx.x % 32;
  const int gl = lane % L;                    // lane within the group
  const int gbase = lane - gl;                // first lane of the group
  // groups of a warp run independently (different units): shuffles use the group's mask
  const unsigned gmask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << gbase);
  const T tol = (T)P.tol, rho = (T)P.rho;

  for (;;) {
    int64_t u = 0;
    if (gl == 0) {
      for (;;) {
        u = atomicAdd(queue, 1);
        if (u >= P.n_units || scale[u] > T(0)) break;  // dead units were written by the prologue
      }
    }
    u = __shfl_sync(gmask, (long long)u, gbase);
    if (u >= P.n_units) break;

    const T sc = scale[u];
    const T b0 = P.beta0 > 0 ? (T)P.beta0 : T(1) / sc;
    const T bmax = P.beta_max > 0 ? (T)P.beta_max : (T)1e7 * b0;
    const T thresh = tol * sc;
    T bcur = b0, bnext = b0, tn = T(1) / b0;

    T x[RPL], y[RPL], l[RPL];
    const T* xu = X + u * P.ldx;
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int row = gl + L * i;
      x[i] = row < P.s ? xu[row] : T(0);
      y[i] = T(0);
      l[i] = T(0);
    }
    T z[KM];
    T prev = Limits<T>::inf(), res = T(0);
    int stalled = 0, it = 0;
    uint8_t code = L1F_UNIT_MAXITER;
    {
      // ---- first pass (z = 0, y = 0): start iteration 1, peeled so the steady-state pass has no
      // "fresh" branches.  Same values as the general pass with A z = 0, y = 0.
      T acc[KM];
#pragma unroll
      for (int t = 0; t < KM; ++t) acc[t] = T(0);
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const T* arow = As + (gl + L * i) * AST;
        const T w = x[i];
        const T sl = w > T(0) ? tn : -tn;
        const T v = tabs(w) > tn ? sl : w;  // = l for the first iteration
        l[i] = v;
#pragma unroll
        for (int t = 0; t < KM; ++t) acc[t] = fma(arow[t], v, acc[t]);
      }
#pragma unroll
      for (int o = L / 2; o > 0; o >>= 1)
#pragma unroll
        for (int t = 0; t < KM; ++t) acc[t] += shfl_xor(gmask, acc[t], o);
      it = 1;
      bcur = bnext;
      T bn = rho * bcur;
      if (bn > bmax) bn = bmax;
      bnext = bn;
      tn = T(1) / bn;
#pragma unroll
      for (int t = 0; t < KM; ++t) z[t] = acc[t];
    }
    for (;;) {
      // ---- one fused pass: finish iteration `it`, start iteration it + 1
      T acc[KM];
#pragma unroll
      for (int t = 0; t < KM; ++t) acc[t] = T(0);
      T m = T(0);
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int row = gl + L * i;
        const T* arow = As + row * AST;
        T a[KM];
#pragma unroll
        for (int t = 0; t < KM; ++t) a[t] = arow[t];
        T azv = T(0);
#pragma unroll
        for (int t = 0; t < KM; ++t) azv = fma(a[t], z[t], azv);
        if (WE && row < P.s) E[u * P.lde + row] = x[i] - l[i];  // e_it
        const T r = l[i] - azv;
        m = tmax(m, tabs(r));
        const T yv = fma(bcur, r, y[i]);
        const T yb = yv * tn;
        const T w = (x[i] - azv) + yb;
        const bool sup = tabs(w) > tn;
        const T sgt = w > T(0) ? tn : -tn;
        l[i] = sup ? (azv - yb) + sgt : x[i];
        const T v = sup ? azv + sgt : x[i] + yb;
        y[i] = yv;
#pragma unroll
        for (int t = 0; t < KM; ++t) acc[t] = fma(a[t], v, acc[t]);
      }
#pragma unroll
      for (int o = L / 2; o > 0; o >>= 1) {
#pragma unroll
        for (int t = 0; t < KM; ++t) acc[t] += shfl_xor(gmask, acc[t], o);
        m = tmax(m, shfl_xor(gmask, m, o));
      }
      bool fin = false;
      {
        const T rel = tabs(m - prev) / tmax(m, Limits<T>::tiny());
        stalled = (rel < (T)kStallEps) ? stalled + 1 : 0;
        prev = m;
        res = m;
        if (m <= thresh) { fin = true; code = L1F_UNIT_OK; }
        else if (stalled >= kStallIters) { fin = true; code = L1F_UNIT_STALLED; }
        else if (it >= P.max_iter) { fin = true; code = L1F_UNIT_MAXITER; }
      }
      if (fin) break;  // z still holds z_it
      it += 1;
      bcur = bnext;
      T bn = rho * bcur;  // beta = min(rho * beta, beta_max), l1reg.py:128
      if (bn > bmax) bn = bmax;
      bnext = bn;
      tn = T(1) / bn;
#pragma unroll
      for (int t = 0; t < KM; ++t) z[t] = acc[t];
    }
    // outputs (z_it, iterations, residual, status)
#pragma unroll
    for (int t = 0; t < KM; ++t)
      if (t % L == gl && t < P.k) Z[u * P.ldz + t] = z[t];
    if (gl == 0) {
      if (iters) iters[u] = it;
      if (res_out) res_out[u] = res;
      if (status) status[u] = code;
    }
    if (P.ncnt) {  // z_u written by the group: count it for the consumer
      __threadfence();
      __syncwarp(gmask);
      if (gl == 0) atomicAdd(&P.ncnt[P.nrows[u] >> 7], 1u);
    }
  }
}

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
      if (P.ncnt) {
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(&P.ncnt[P.nrows[u] >> 7], 1u);
      }
    }
  }
}

template <typename T, int KM, int RPL, int L>
int launch(const T* X, int64_t ldx, int s, int64_t n_units, const T* A, int64_t lda, int k, double tol, double rho,
           double beta0, double beta_max, int max_iter, T* Z, int64_t ldz, T* E, int64_t lde, int32_t* iters, T* res,
           uint8_t* status, void* workspace, size_t ws_bytes, cudaStream_t st, bool query, size_t* need,
           tcf::NotifyHost* nh) {
  const size_t scale_bytes = (sizeof(T) * (size_t)(n_units > 0 ? n_units : 1) + 255) & ~(size_t)255;
  const size_t total = scale_bytes + 256;
  if (query) { *need = total; return L1F_OK; }
  auto kern = E ? adm_small_kernel<T, KM, RPL, L, true> : adm_small_kernel<T, KM, RPL, L, false>;
  const int s_pad = RPL * L;
  const size_t smem = sizeof(T) * (size_t)s_pad * (KM + 1);
  static int bps_cache[2] = {0, 0};
  int& blocks_per_sm = bps_cache[E ? 1 : 0];
  if (!blocks_per_sm) {
    L1F_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // the largest shared-memory carveout: the SMs keep room for a reconstruction CTA beside the
    // filter's blocks (l1f_rowfilter_reconstruct_small); the filter itself uses ~10 KB per block
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, 128, smem) != cudaSuccess ||
        blocks_per_sm < 1)
      blocks_per_sm = 1;
  }
  void* owned = nullptr;
  if (!workspace) {
    L1F_CUDA_TRY(cudaMallocAsync(&owned, total, st));
    workspace = owned;
  } else {
    L1F_REQUIRE(ws_bytes >= total, L1F_ERR_ARG, "filter: workspace too small");
  }
  Params P;
  P.s = s; P.k = k; P.s_pad = s_pad;
  P.n_units = n_units; P.ldx = ldx; P.ldz = ldz; P.lde = lde; P.max_iter = max_iter;
  P.tol = tol; P.rho = rho; P.beta0 = beta0; P.beta_max = beta_max;
  T* scale = (T*)workspace;
  int* queue = (int*)((unsigned char*)workspace + scale_bytes);
  int rc = L1F_OK;
  if (nh) {
    P.nrows = nh->rows;
    P.ncnt = nh->cnt;
    P.nres = nh->resident;
    nh->cluster = 1;
  }
  unit_scale_kernel<T><<<(unsigned)std::min<int64_t>(ceil_div(n_units, 8), 65535), 256, 0, st>>>(
      X, P, scale, Z, E, iters, res, status);
  if (cudaGetLastError() != cudaSuccess) rc = L1F_ERR_CUDA;
  if (rc == L1F_OK && nh && nh->after_prologue && cudaEventRecord(nh->after_prologue, st) != cudaSuccess) rc = L1F_ERR_CUDA;
  if (rc == L1F_OK && max_iter > 0) {
    if (cudaMemsetAsync(queue, 0, sizeof(int), st) != cudaSuccess) rc = L1F_ERR_CUDA;
    const int64_t want_blocks = ceil_div(n_units * L, 128);  // one group per unit at most
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want_blocks, (int64_t)blocks_per_sm * num_sms()));
    if (nh) nh->ctas = grid;
    kern<<<grid, 128, smem, st>>>(X, A, lda, scale, P, queue, Z, E, iters, res, status);
    if (cudaGetLastError() != cudaSuccess) {
      set_error("filter (small-k): launch failed");
      rc = L1F_ERR_CUDA;
    }
  }
  if (owned) cudaFreeAsync(owned, st);
  return rc;
}

}  // namespace small
}  // namespace l1f

template <typename T>
int l1f_small_dispatch(const T* X, int64_t ldx, int s, int64_t n_units, const T* A, int64_t lda, int k, double tol,
                       double rho, double beta0, double beta_max, int max_iter, T* Z, int64_t ldz, T* E, int64_t lde,
                       int32_t* iters, T* res, uint8_t* status, void* workspace, size_t ws_bytes, cudaStream_t st,
                       bool query, size_t* need, l1f::tcf::NotifyHost* nh) {
  if (k > 16) return L1F_ERR_UNSUPPORTED;
#define L1F_SMALL(KM, RPL, L)                                                                                   \
  return l1f::small::launch<T, KM, RPL, L>(X, ldx, s, n_units, A, lda, k, tol, rho, beta0, beta_max, max_iter, \
                                           Z, ldz, E, lde, iters, res, status, workspace, ws_bytes, st, query,  \
                                           need, nh)
  if (k <= 4) {
    if (s <= 64) L1F_SMALL(4, 4, 16);
    if (s <= 128) L1F_SMALL(4, 8, 16);
    if (s <= 256) L1F_SMALL(4, 8, 32);
  } else if (k <= 8) {
    if (s <= 64) L1F_SMALL(8, 4, 16);
    if (s <= 128) L1F_SMALL(8, 8, 16);
    if (s <= 256) L1F_SMALL(8, 8, 32);
  } else if (k <= 10) {  // configs 1 and 4 (k = 10, s = 100): exact width, 8-lane groups
    // 8 lanes x 13 rows for s <= 104 (the configs' s = 100; tools/r2/small_k_ab.py: cfg4 1.10 ms vs
    // 1.23 ms for 16 x 7, 1.60 ms for 32 x 4); L1F_OPT_SMALL_LANES = 16 / 32 selects the others (A/B)
    const int64_t lanes = l1f::option(L1F_OPT_SMALL_LANES);
    if (s <= 112 && lanes == 16) L1F_SMALL(10, 7, 16);
    if (s <= 128 && lanes == 32) L1F_SMALL(10, 4, 32);
    if (s <= 104) L1F_SMALL(10, 13, 8);
    if (s <= 128) L1F_SMALL(10, 8, 16);
    if (s <= 256) L1F_SMALL(10, 8, 32);
  } else if (k <= 12) {
    if (s <= 64) L1F_SMALL(12, 4, 16);
    if (s <= 128) L1F_SMALL(12, 8, 16);
    if (s <= 256) L1F_SMALL(12, 8, 32);
  } else {
    if (s <= 64) L1F_SMALL(16, 4, 16);
    if (s <= 128) L1F_SMALL(16, 8, 16);
    if (s <= 256) L1F_SMALL(16, 8, 32);
  }
#undef L1F_SMALL
  return L1F_ERR_UNSUPPORTED;
}

template int l1f_small_dispatch<float>(const float*, int64_t, int, int64_t, const float*, int64_t, int, double, double,
                                       double, double, int, float*, int64_t, float*, int64_t, int32_t*, float*,
                                       uint8_t*, void*, size_t, cudaStream_t, bool, size_t*,
                                       l1f::tcf::NotifyHost*);
template int l1f_small_dispatch<double>(const double*, int64_t, int, int64_t, const double*, int64_t, int, double,
                                        double, double, double, int, double*, int64_t, double*, int64_t, int32_t*,
                                        double*, uint8_t*, void*, size_t, cudaStream_t, bool, size_t*,
                                        l1f::tcf::NotifyHost*);
