// Eigenpairs of a symmetric matrix above a threshold, hand-written (the Gram step of the large-seed
// SVT, seed.cu svt_gram / svd_gram; reference: the SVD inside svt_with_rank, matcore.py:73-105).
//
//   1. Householder tridiagonalisation T = Q^T G Q (LAPACK dsytd2 'L' order).  Default
//      (tridiag_dsm_kernel, p <= 2000): G resident in the shared memory of all SMs, rows owned per
//      block, one counter barrier per column (see the kernel).  Otherwise (tridiag_kernel): G in
//      L2, two grid-wide barriers per column.
//   2. The k eigenvalues of T above the threshold: a Sturm count gives k, each eigenvalue is
//      bracketed by multisection (one warp per eigenvalue, 32 Sturm counts per round).
//   3. Eigenvectors of T by inverse iteration (tridiagonal LU with partial pivoting, two solves per
//      eigenvalue; one block per eigenvalue with its factors in shared memory), then classical
//      Gram-Schmidt twice inside clusters of nearly equal eigenvalues, normalisation and Rayleigh
//      quotients as the final eigenvalues (one warp per vector).
//   4. Back-transformation Z = Q Y: each vector split over a group of warps and held in
//      registers, the reflector rows streamed through shared memory (cp.async, double-buffered).
// No library call; the host reads k and the eigenvalues once.
#include "common.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <vector>

namespace cg = cooperative_groups;

namespace l1f {
namespace eig {

constexpr int TT = 256;  // threads per block of the tridiagonalisation
constexpr int TW = TT / 32;

__device__ double block_sum_det(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < (int)(blockDim.x / 32); ++w) t += red[w];
  return t;
}

// A: p x p row-major, full symmetric (overwritten).  Outputs d[p], e[p-1], tau[p-1], Vh[p][p]
// (row i: v_i for columns i+1 .. p-1, v_i[i+1] = 1).  pv: p scratch, part: gridDim.x scratch.
// Row r of the trailing block belongs to block r mod gridDim.x; the block's 8 warps split its rows'
// columns into 8 contiguous chunks, so every warp has a few independent loads per lane per phase
// (one L2 round trip) and the row sums of A v reduce in shared memory in a fixed order.  Dynamic
// shared memory: v, w (2 p doubles) and the per-row warp partials.  Two grid barriers per column.
__global__ void __launch_bounds__(TT) tridiag_kernel(double* __restrict__ A, int p, double* __restrict__ d,
                                                   double* __restrict__ e, double* __restrict__ tau_out,
                                                   double* __restrict__ Vh, double* __restrict__ pv,
                                                   double* __restrict__ part) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sv[];  // v: [0, p), w: [p, 2p), warp partials: [2p, 2p + 8 * rows_max)
  double* sw = sv + p;
  double* wp = sv + 2 * p;
  __shared__ double red[TW + 1];
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  const int G = gridDim.x, b = blockIdx.x;
  for (int i = 0; i + 1 < p; ++i) {
    const int c0 = i + 1, len = p - c0;
    const double* rowi = A + (size_t)i * p;
    // row i's tail into shared memory and its norm (every block; the reflector is recomputed
    // identically everywhere)
    double s = 0.0;
    for (int c = c0 + threadIdx.x; c < p; c += TT) {
      const double x = rowi[c];
      sv[c] = x;
      if (c > c0) s = fma(x, x, s);
    }
    const double xnorm2 = block_sum_det(s, red);
    const double alpha = sv[c0];
    double tau = 0.0, beta = alpha, scale = 0.0;
    if (xnorm2 > 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, xnorm2)), alpha);
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    if (b == 0 && threadIdx.x == 0) {
      d[i] = rowi[i];
      e[i] = beta;
      tau_out[i] = tau;
    }
    if (tau == 0.0) {  // H = I: nothing to update (uniform across the grid)
      for (int r = c0 + b * TT + threadIdx.x; r < p; r += G * TT) Vh[(size_t)i * p + r] = r == c0 ? 1.0 : 0.0;
      __syncthreads();
      continue;
    }
    for (int c = c0 + threadIdx.x; c < p; c += TT) sv[c] = c == c0 ? 1.0 : sv[c] * scale;
    __syncthreads();
    // this block's rows r = first, first + G, ...; warp w takes columns [c0 + w*cl, c0 + (w+1)*cl)
    const int first = c0 + ((b - c0 % G) + G) % G;
    const int nrows = first < p ? (p - 1 - first) / G + 1 : 0;
    const int cl = (len + TW - 1) / TW;
    const int ca = c0 + warp * cl, cb = min(p, ca + cl);
    // rows in groups of 8 with independent accumulators: 8 loads in flight per column step
    for (int q0 = 0; q0 < nrows; q0 += 8) {
      double a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = 0.0;
      const double* ar = A + (size_t)(first + q0 * G) * p;
      const size_t rstride = (size_t)G * p;
      const int nu = min(8, nrows - q0);
      for (int c = ca + lane; c < cb; c += 32) {
        const double vc = sv[c];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (u < nu) a[u] = fma(ar[u * rstride + c], vc, a[u]);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double t = warp_sum(a[u]);
        if (lane == 0 && u < nu) wp[(q0 + u) * TW + warp] = t;
      }
    }
    __syncthreads();
    double dot = 0.0;
    for (int q = threadIdx.x; q < nrows; q += TT) {
      const int r = first + q * G;
      double a = 0.0;
      for (int w = 0; w < TW; ++w) a += wp[q * TW + w];
      a *= tau;
      pv[r] = a;
      Vh[(size_t)i * p + r] = sv[r];
      dot = fma(a, sv[r], dot);
    }
    dot = block_sum_det(dot, red);
    if (threadIdx.x == 0) part[b] = dot;
    grid.sync();
    double ps = 0.0;
    for (int x = threadIdx.x; x < G; x += TT) ps += part[x];
    const double pvdot = block_sum_det(ps, red);
    const double K = -0.5 * tau * pvdot;
    for (int c = c0 + threadIdx.x; c < p; c += TT) sw[c] = fma(K, sv[c], pv[c]);
    __syncthreads();
    // A[r][c] -= v[r] w[c] + w[r] v[c]  for this block's rows, warp w on its column chunk
    for (int q0 = 0; q0 < nrows; q0 += 8) {
      const int nu = min(8, nrows - q0);
      double vr[8], wr[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int r = first + (q0 + (u < nu ? u : 0)) * G;
        vr[u] = sv[r];
        wr[u] = sw[r];
      }
      double* ar = A + (size_t)(first + q0 * G) * p;
      const size_t rstride = (size_t)G * p;
      for (int c = ca + lane; c < cb; c += 32) {
        const double vc = sv[c], wc = sw[c];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (u < nu) ar[u * rstride + c] -= fma(vr[u], wc, wr[u] * vc);
      }
    }
    grid.sync();
  }
  if (b == 0 && threadIdx.x == 0) d[p - 1] = A[(size_t)(p - 1) * p + p - 1];
}

// Tridiagonalisation with the matrix resident in the shared memory of the whole GPU (default for
// p up to what 148 SMs hold: p <= 2000).  Block b owns rows b, b + G, b + 2G, ... in its shared
// memory for the whole reduction; each of its 256 threads owns columns tid, tid + 256, ...  Per
// column i every block recomputes the reflector from its register copy of row i (identical values
// and reduction order everywhere: no broadcast), forms y = tau A v for its rows, publishes them
// (per-column slots) with its partial of y.v, waits once on the column's counter (release add,
// acquire spin: 1.3 us measured, tools/r2/xchg_bench.cu — polling per-block slots instead costs
// 4.5 us), then reads y and the partials back (L2), updates its rows and its copy of row i + 1,
// whose values the owner published one column earlier, so that load shares the round trip of y.
// dsytd2 'L' order, as tridiag_kernel; Vh, d, e, tau written by block 0.
#ifdef L1F_EIG_PROF
#define EPROF(slot) do { if (tid == 0 && b == 0) { long long _t = clock64(); eprof[slot] += _t - eprev; eprev = _t; } } while (0)
#else
#define EPROF(slot) do {} while (0)
#endif

constexpr int DSM_T = 256;
constexpr int DSM_W = DSM_T / 32;
constexpr int DSM_R = 16;  // rows per block at most

// ybuf, rowbuf: p x p slots (column i's y; row r's published values); part: p x G slots
template <int CPT, int NTH, int RM>  // RM: rows per block at most (8 or 16)
__global__ void __launch_bounds__(NTH, 1)
tridiag_dsm_kernel(const double* __restrict__ A, int p, double* __restrict__ d, double* __restrict__ e,
                   double* __restrict__ tau_out, double* __restrict__ Vh, double* ybuf, double* part, double* rowbuf,
                   unsigned* cnt) {
  constexpr int NWP = NTH / 32;
  extern __shared__ double As[];  // R x p, row q = global row b + q G
  __shared__ double red[NWP][DSM_R + 1];
  __shared__ double wsum[NWP];
  __shared__ double vq[DSM_R], yq[DSM_R];
  __shared__ double sc[4];
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int R = b < p ? (p - 1 - b) / G + 1 : 0;
  for (int q = 0; q < R; ++q)
    for (int c = tid; c < p; c += NTH) As[(size_t)q * p + c] = A[(size_t)(b + q * G) * p + c];
  double cur[CPT];
  int ownq[CPT];  // this thread's columns that are rows of this block: their index q, else -1
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    const int c = tid + NTH * j;
    cur[j] = c < p ? A[c] : 0.0;
    ownq[j] = (c < p && c >= b && (c - b) % G == 0) ? (c - b) / G : -1;
  }
  __syncthreads();
#ifdef L1F_EIG_PROF
  long long eprof[7] = {0, 0, 0, 0, 0, 0, 0};
  long long eprev = clock64();
#endif
  for (int i = 0; i + 1 < p; ++i) {
    const int c0 = i + 1;
    // ---- reflector from row i (every block, identically)
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int c = tid + NTH * j;
      if (c > c0 && c < p) s = fma(cur[j], cur[j], s);
      if (c == c0) sc[0] = cur[j];
      if (c == i && b == 0) d[i] = cur[j];
    }
    s = warp_sum(s);
    if (lane == 0) wsum[warp] = s;
    __syncthreads();
    const double xnorm2 = warp_sum(lane < NWP ? wsum[lane] : 0.0);  // same tree in every warp
    const double alpha = sc[0];
    double tau = 0.0, beta = alpha, scale = 0.0;
    if (xnorm2 > 0.0) householder_scalars(alpha, xnorm2, beta, tau, scale);
    double v[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int c = tid + NTH * j;
      v[j] = c == c0 ? 1.0 : ((c > c0 && c < p) ? cur[j] * scale : 0.0);
      if (c >= c0 && c < p) {
        if (b == 0) Vh[(size_t)i * p + c] = v[j];
        if (ownq[j] >= 0) vq[ownq[j]] = v[j];
      }
    }
    if (b == 0 && tid == 0) {
      e[i] = beta;
      tau_out[i] = tau;
    }
    EPROF(0);
    // ---- y = tau A v over this block's rows r >= c0
    double acc[RM];
#pragma unroll
    for (int q = 0; q < RM; ++q) {
      acc[q] = 0.0;
      if (q < R && b + q * G >= c0) {
        const double* ar = As + (size_t)q * p;
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
          const int c = tid + NTH * j;
          if (c < p) acc[q] = fma(ar[c], v[j], acc[q]);
        }
      }
    }
    // transpose-reduce: RM values per lane -> lane groups holding one row's warp sum
#pragma unroll
    for (int h = RM / 2; h >= 1; h >>= 1) {
      const int o = h * (32 / RM);  // lane distance 16, 8, ... (RM = 16: 16, 8, 4, 2; RM = 8: 16, 8, 4)
      const bool upper = (lane & o) != 0;
#pragma unroll
      for (int q = 0; q < h; ++q) {
        const double send = upper ? acc[q] : acc[q + h];
        const double keep = upper ? acc[q + h] : acc[q];
        acc[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
#pragma unroll
    for (int o = 32 / RM / 2; o >= 1; o >>= 1) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], o);
    int qrow = 0;
#pragma unroll
    for (int h = RM / 2, o = 16; h >= 1; h >>= 1, o >>= 1) qrow += (lane & o) ? h : 0;
    if ((lane & (32 / RM - 1)) == 0) red[warp][qrow] = acc[0];
    __syncthreads();
    double* ycol = ybuf + (size_t)i * p;
    double* pcol = part + (size_t)i * G;
    EPROF(1);
    if (warp == 0) {
      double pv = 0.0;
      if (lane < RM) {
        const int r = b + lane * G;
        double t = 0.0;
        if (lane < R && r >= c0) {
          for (int w = 0; w < NWP; ++w) t += red[w][lane];
          t *= tau;
          ycol[r] = t;
          pv = t * vq[lane];
        }
        yq[lane] = t;
      }
      pv = warp_sum(pv);
      if (lane == 0) pcol[b] = pv;
      __syncwarp();
      EPROF(5);
      // the column's grid-wide wait: one counter, release add / acquire spin (a barrier over every
      // block's y, partial and the row it published one column earlier)
      if (lane == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt + i) : "memory");
        unsigned arrived;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(arrived) : "l"(cnt + i) : "memory");
        } while (arrived < (unsigned)G);
      }
      __syncwarp();
    }
    __syncthreads();
    EPROF(2);
    // ---- K from every block's partial (warp 0), y and the copy of row c0 for this thread's columns
    if (warp == 0) {
      double t = 0.0;
      for (int x = lane; x < G; x += 32) t += __ldcg(pcol + x);
      t = warp_sum(t);
      if (lane == 0) sc[1] = -0.5 * tau * t;
    }
    double yv[CPT], nx[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int c = tid + NTH * j;
      const bool live = c >= c0 && c < p;
      yv[j] = live ? __ldcg(ycol + c) : 0.0;
      nx[j] = live ? (i == 0 ? A[(size_t)p + c] : __ldcg(rowbuf + (size_t)c0 * p + c)) : 0.0;
    }
    const double yc0 = __ldcg(ycol + c0);
    __syncthreads();
    const double K = sc[1];
    const double wc0 = yc0 + K;
    EPROF(3);
    double w[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) w[j] = fma(K, v[j], yv[j]);
    // ---- rank-2 update of this block's rows and of the copy of row c0
    for (int q = 0; q < R; ++q) {
      const int r = b + q * G;
      if (r < c0) continue;
      const double vr = vq[q], wr = fma(K, vr, yq[q]);
      double* ar = As + (size_t)q * p;
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const int c = tid + NTH * j;
        if (c >= c0 && c < p) ar[c] -= fma(vr, w[j], wr * v[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int c = tid + NTH * j;
      cur[j] = (c >= c0 && c < p) ? nx[j] - fma(1.0, w[j], wc0 * v[j]) : 0.0;
    }
    // ---- publish row i + 2 (current through column i) for the copies at column i + 1
    const int r2 = i + 2;
    if (r2 < p && r2 >= b && (r2 - b) % G == 0) {
      const double* ar = As + (size_t)(r2 / G) * p;
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const int c = tid + NTH * j;
        if (c >= r2 && c < p) rowbuf[(size_t)r2 * p + c] = ar[c];
      }
    }
    EPROF(4);
    // no barrier here: the next column's first __syncthreads orders sc / vq / yq / wsum reuse
  }
#ifdef L1F_EIG_PROF
  if (tid == 0 && b == 0)
    printf("tridiag_dsm p=%d cycles/col: reflector %lld matvec %lld publish %lld wait+K %lld loads %lld update %lld\n", p,
           eprof[0] / (p - 1), eprof[1] / (p - 1), eprof[5] / (p - 1), eprof[2] / (p - 1), eprof[3] / (p - 1), eprof[4] / (p - 1));
#endif
  if (b == 0) {
#pragma unroll
    for (int j = 0; j < CPT; ++j)
      if (tid + NTH * j == p - 1) d[p - 1] = cur[j];
  }
}

// number of eigenvalues of T (d, e2 = e^2) below x (Sturm count), with the hardware reciprocal
// estimate and one Newton step per pivot (relative error ~2^-46, far below the multisection's resolution)
__device__ __forceinline__ int sturm_below_fast(const double* __restrict__ d, const double* __restrict__ e2, int p,
                                                double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0.0;
  for (int j = 1; j < p; ++j) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    r = r * fma(-q, r, 2.0);
    q = fma(-e2[j - 1], r, d[j] - x);
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

// reciprocal from the hardware estimate and two Newton steps (within an ulp of 1 / x; off the
// IEEE division's slow path, which dominates a dependent chain of p steps)
// rcp_nr2: common.cuh

// count of eigenvalues below x with rcp_nr2 pivots (the threshold count of bounds_kernel)
__device__ __forceinline__ int sturm_below_nr2(const double* __restrict__ d, const double* __restrict__ e2, int p,
                                               double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0.0;
  for (int j = 1; j < p; ++j) {
    q = fma(-e2[j - 1], rcp_nr2(q), d[j] - x);
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

struct Bounds {
  double lo, hi, pivmin;
  int k;
};

// Gershgorin bounds, pivmin and k = #(lambda >= thr) (single block)
__global__ void bounds_kernel(const double* __restrict__ d, const double* __restrict__ e, double* __restrict__ e2, int p,
                              double thr_abs, double thr_rel, Bounds* B) {
  __shared__ double red[32];
  __shared__ double shi;
  double lo = 1e300, hi = -1e300, emax = 0.0;
  for (int j = threadIdx.x; j < p; j += blockDim.x) {
    const double el = j > 0 ? fabs(e[j - 1]) : 0.0, er = j + 1 < p ? fabs(e[j]) : 0.0;
    lo = fmin(lo, d[j] - el - er);
    hi = fmax(hi, d[j] + el + er);
    if (j + 1 < p) {
      e2[j] = e[j] * e[j];
      emax = fmax(emax, e2[j]);
    }
  }
  // block min / max (order-independent)
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  }
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32, nw = blockDim.x / 32;
  if (lane == 0) red[warp] = lo;
  __syncthreads();
  if (threadIdx.x == 0) { double t = red[0]; for (int w = 1; w < nw; ++w) t = fmin(t, red[w]); B->lo = t; }
  __syncthreads();
  if (lane == 0) red[warp] = hi;
  __syncthreads();
  if (threadIdx.x == 0) { double t = red[0]; for (int w = 1; w < nw; ++w) t = fmax(t, red[w]); B->hi = t; shi = t; }
  __syncthreads();
  if (lane == 0) red[warp] = emax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = red[0];
    for (int w = 1; w < nw; ++w) t = fmax(t, red[w]);
    const double pivmin = DBL_MIN * fmax(1.0, t);
    B->pivmin = pivmin;
    const double thr = fmax(thr_abs, thr_rel * fmax(fabs(shi), fabs(B->lo)));
    B->lo = thr;  // bracket from the threshold
    B->k = p - sturm_below_nr2(d, e2, p, thr, pivmin);
  }
}

// eigenvalue j (j-th largest, j < k) to a coarse bracket by multisection: one warp per eigenvalue
__global__ void bisect_kernel(const double* __restrict__ d, const double* __restrict__ e2, int p, const Bounds* B,
                              int rounds, double* __restrict__ lam) {
  const int lane = threadIdx.x % 32;
  const int j = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int k = B->k;
  if (j >= k) return;
  const int idx = p - 1 - j;  // ascending index
  const double pivmin = B->pivmin;
  double lo = B->lo, hi = B->hi * (1.0 + 1e-14) + fabs(B->hi) * 1e-14 + pivmin;
  for (int it = 0; it < rounds; ++it) {
    const double x = lo + (hi - lo) * (double)(lane + 1) / 33.0;
    const int c = sturm_below_fast(d, e2, p, x, pivmin);  // eigenvalues below x
    // smallest x with count > idx is the new hi; the largest with count <= idx the new lo
    const unsigned above = __ballot_sync(0xffffffffu, c > idx);
    const int first = above ? __ffs(above) - 1 : 32;
    const double nlo = first == 0 ? lo : lo + (hi - lo) * (double)first / 33.0;
    const double nhi = first == 32 ? hi : lo + (hi - lo) * (double)(first + 1) / 33.0;
    lo = nlo;
    hi = nhi;
    if (hi - lo <= 4e-16 * fmax(fabs(lo), fabs(hi)) + pivmin) break;
  }
  if (lane == 0) lam[j] = 0.5 * (lo + hi);
}

// inverse iteration on T - s I (LU with partial pivoting, LAPACK dgttrf / dgttrs), two solves,
// one thread per eigenvalue.  The per-eigenvalue factors live in scratch interleaved by eigenvalue
// (entry i of eigenvalue j at [i * kp + j]) so a warp's loads and stores are coalesced; Y column j
// (length p, contiguous) receives the normalised vector.
__global__ void inverse_iter_kernel(const double* __restrict__ d, const double* __restrict__ e, int p, const Bounds* B,
                                    const double* __restrict__ lam, double* __restrict__ Y, double* __restrict__ scratch,
                                    int kp) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= B->k) return;
  const double s = lam[j];
  const size_t plane = (size_t)p * kp;
  double* dl = scratch + j;            // multipliers
  double* dd = dl + plane;             // U diagonal
  double* du = dd + plane;             // U first superdiagonal
  double* du2 = du + plane;            // U second superdiagonal
  double* bb = du2 + plane;            // right-hand side / solution
  double* swp = bb + plane;            // row-interchange flags
  auto at = [kp](double* a, int i) -> double& { return a[(size_t)i * kp]; };
  const double eps = 2.220446049250313e-16;
  const double tnorm = fmax(fabs(B->hi), fabs(B->lo)) + 1.0e-300;
  // factor (T - sI) = L U with partial pivoting (dgttrf), carrying the current diagonal and
  // superdiagonal in registers
  double di = d[0] - s, ui = p > 1 ? e[0] : 0.0;
  for (int i = 0; i + 1 < p; ++i) {
    const double sub = e[i];
    const double dn = d[i + 1] - s;
    const double un = i + 2 < p ? e[i + 1] : 0.0;
    if (fabs(di) >= fabs(sub)) {
      const double f = di != 0.0 ? sub / di : 0.0;
      at(dl, i) = f;
      at(dd, i) = di;
      at(du, i) = ui;
      at(du2, i) = 0.0;
      at(swp, i) = 0.0;
      di = dn - f * ui;
      ui = un;
    } else {
      const double f = di / sub;
      at(dl, i) = f;
      at(dd, i) = sub;
      at(du, i) = dn;
      at(du2, i) = un;
      at(swp, i) = 1.0;
      di = ui - f * dn;
      ui = -f * un;
    }
  }
  at(dd, p - 1) = di;
  for (int i = 0; i < p; ++i) {
    double& x = at(dd, i);
    if (fabs(x) < eps * tnorm) x = copysign(eps * tnorm, x == 0.0 ? 1.0 : x);
  }
  for (int i = 0; i < p; ++i) at(bb, i) = 1.0 + 0.5 * sin(0.7 * (double)i + 0.3 * (double)j);
  for (int rep = 0; rep < 2; ++rep) {
    double prev = at(bb, 0);
    for (int i = 0; i + 1 < p; ++i) {  // forward: L with the interchanges
      const double nx = at(bb, i + 1);
      if (at(swp, i) == 0.0) {
        at(bb, i) = prev;
        prev = nx - at(dl, i) * prev;
      } else {
        at(bb, i) = nx;
        prev = prev - at(dl, i) * nx;
      }
    }
    at(bb, p - 1) = prev;
    double x1 = at(bb, p - 1) / at(dd, p - 1);  // back substitution with U
    at(bb, p - 1) = x1;
    double x2 = 0.0;
    if (p > 1) {
      x2 = x1;
      x1 = (at(bb, p - 2) - at(du, p - 2) * x2) / at(dd, p - 2);
      at(bb, p - 2) = x1;
    }
    for (int i = p - 3; i >= 0; --i) {
      const double x0 = (at(bb, i) - at(du, i) * x1 - at(du2, i) * x2) / at(dd, i);
      at(bb, i) = x0;
      x2 = x1;
      x1 = x0;
    }
    double nrm = 0.0;
    for (int i = 0; i < p; ++i) nrm = fma(at(bb, i), at(bb, i), nrm);
    const double inv = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
    for (int i = 0; i < p; ++i) at(bb, i) *= inv;
  }
  double* y = Y + (size_t)j * p;
  for (int i = 0; i < p; ++i) y[i] = at(bb, i);
}

// classical Gram-Schmidt, twice (CGS2), over Y's k columns in descending eigenvalue order: nearly
// equal shifts inside a cluster give nearly parallel vectors; CGS2 keeps the cluster's span and
// makes the basis orthonormal to working precision.  Then the Rayleigh quotients lam[j] = y_j^T T y_j.
// One block (per vector: all dots with the earlier vectors, one barrier, the update, one barrier).
__global__ void cgs2_kernel(double* __restrict__ Y, int p, const Bounds* B, const double* __restrict__ d,
                            const double* __restrict__ e, double* __restrict__ lam) {
  extern __shared__ double sdot[];  // k entries
  __shared__ double red[32];
  const int k = B->k;
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32, nw = blockDim.x / 32;
  // clusters: consecutive eigenvalues closer than 1e-4 ||T||; outside a cluster inverse iteration
  // alone leaves the vectors orthogonal to ~eps ||T|| / gap <= 1e-12 (and already unit length)
  const double gap_tol = 1e-4 * fmax(fabs(B->hi), fabs(B->lo));
  int cstart = 0;
  for (int j = 0; j < k; ++j) {
    if (j > 0 && !(fabs(lam[j - 1] - lam[j]) < gap_tol)) cstart = j;
    if (cstart == j) continue;  // uniform
    double* yj = Y + (size_t)j * p;
    for (int pass = 0; pass < 2; ++pass) {
      for (int i = cstart + warp; i < j; i += nw) {
        const double* yi = Y + (size_t)i * p;
        double s = 0.0;
        for (int r = lane; r < p; r += 32) s = fma(yi[r], yj[r], s);
        s = warp_sum(s);
        if (lane == 0) sdot[i] = s;
      }
      __syncthreads();
      for (int r = threadIdx.x; r < p; r += blockDim.x) {
        double v = yj[r];
        for (int i = cstart; i < j; ++i) v = fma(-sdot[i], Y[(size_t)i * p + r], v);
        yj[r] = v;
      }
      __syncthreads();
    }
    double s = 0.0;
    for (int r = threadIdx.x; r < p; r += blockDim.x) s = fma(yj[r], yj[r], s);
    const double nrm = sqrt(block_sum_det(s, red));
    const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
    for (int r = threadIdx.x; r < p; r += blockDim.x) yj[r] *= inv;
    __syncthreads();
  }
}

// normalisation and Rayleigh quotients lam_j = y_j^T T y_j, one warp per vector
__global__ void rq_kernel(double* __restrict__ Y, int p, const Bounds* B, const double* __restrict__ d,
                          const double* __restrict__ e, double* __restrict__ lam) {
  const int lane = threadIdx.x % 32;
  const int j = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (j >= B->k) return;
  double* yj = Y + (size_t)j * p;
  double s = 0.0;
  for (int r = lane; r < p; r += 32) s = fma(yj[r], yj[r], s);
  const double nrm = sqrt(warp_sum(s));
  const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
  double q = 0.0;
  for (int r = lane; r < p; r += 32) {
    const double yr = yj[r] * inv;
    double ty = d[r] * yr;
    if (r > 0) ty = fma(e[r - 1], yj[r - 1] * inv, ty);
    if (r + 1 < p) ty = fma(e[r], yj[r + 1] * inv, ty);
    q = fma(yr, ty, q);
  }
  q = warp_sum(q);
  __syncwarp();
  for (int r = lane; r < p; r += 32) yj[r] *= inv;
  if (lane == 0) lam[j] = q;
}

// Z column j = Q y_j, Q = H_0 H_1 ... H_{p-2}: H_{p-2} .. H_0 applied in turn; one block per column,
// the column in shared memory, v rows read from global (contiguous)
__global__ void backtransform_kernel(const double* __restrict__ Vh, const double* __restrict__ tau, int p,
                                     const Bounds* B, double* __restrict__ Y) {
  extern __shared__ double sy[];
  __shared__ double red[32];
  const int j = blockIdx.x;
  if (j >= B->k) return;
  double* y = Y + (size_t)j * p;
  for (int c = threadIdx.x; c < p; c += blockDim.x) sy[c] = y[c];
  __syncthreads();
  for (int i = p - 2; i >= 0; --i) {
    const double t = tau[i];
    if (t == 0.0) continue;
    const double* v = Vh + (size_t)i * p;
    double s = 0.0;
    for (int c = i + 1 + threadIdx.x; c < p; c += blockDim.x) s = fma(v[c], sy[c], s);
    s = block_sum_det(s, red) * t;
    for (int c = i + 1 + threadIdx.x; c < p; c += blockDim.x) sy[c] = fma(-s, v[c], sy[c]);
    __syncthreads();
  }
  for (int c = threadIdx.x; c < p; c += blockDim.x) y[c] = sy[c];
}

// inverse iteration as inverse_iter_kernel, one block per eigenvalue with its factors in shared
// memory (a dependent step is a shared-memory access, not an L2 round trip): thread 0 factors and
// solves, the warp writes the normalised vector
__global__ void __launch_bounds__(32) inverse_iter_smem_kernel(const double* __restrict__ d, const double* __restrict__ e,
                                                              int p, const Bounds* B, const double* __restrict__ lam,
                                                              double* __restrict__ Y) {
  extern __shared__ double fsm[];
  const int j = blockIdx.x;
  if (j >= B->k) return;
  double* dl = fsm;
  double* dinv = dl + p;
  double* du = dinv + p;
  double* du2 = du + p;
  double* bb = du2 + p;
  unsigned* sw = (unsigned*)(bb + p);
  __shared__ double s_inv;
  if (threadIdx.x == 0) {
    const double s = lam[j];
    const double eps = 2.220446049250313e-16;
    const double clampv = eps * (fmax(fabs(B->hi), fabs(B->lo)) + 1.0e-300);
    auto inv_pivot = [clampv](double x) {
      if (fabs(x) < clampv) x = copysign(clampv, x == 0.0 ? 1.0 : x);
      return rcp_nr2(x);
    };
    double di = d[0] - s, ui = p > 1 ? e[0] : 0.0;
    unsigned bits = 0;
    for (int i = 0; i + 1 < p; ++i) {
      const double sub = e[i];
      const double dn = d[i + 1] - s;
      const double un = i + 2 < p ? e[i + 1] : 0.0;
      if (fabs(di) >= fabs(sub)) {
        const double f = di != 0.0 ? sub * rcp_nr2(di) : 0.0;
        dl[i] = f; dinv[i] = inv_pivot(di); du[i] = ui; du2[i] = 0.0;
        di = dn - f * ui;
        ui = un;
      } else {
        const double f = di * rcp_nr2(sub);
        dl[i] = f; dinv[i] = inv_pivot(sub); du[i] = dn; du2[i] = un;
        bits |= 1u << (i & 31);
        di = ui - f * dn;
        ui = -f * un;
      }
      if ((i & 31) == 31) { sw[i >> 5] = bits; bits = 0; }
    }
    if (p >= 2 && ((p - 2) & 31) != 31) sw[(p - 2) >> 5] = bits;
    dinv[p - 1] = inv_pivot(di);
    for (int i = 0; i < p; ++i) {  // deterministic start vector in [0.75, 1.25)
      const unsigned h = ((unsigned)i * 2654435761u) ^ ((unsigned)(j + 1) * 2246822519u);
      bb[i] = 0.75 + 0.5 * (double)((h >> 8) & 0xffffu) / 65536.0;
    }
    double inv = 0.0;
    for (int rep = 0; rep < 2; ++rep) {
      if (rep == 1)
        for (int i = 0; i < p; ++i) bb[i] *= inv;
      double prev = bb[0];
      for (int i = 0; i + 1 < p; ++i) {
        const double nx = bb[i + 1];
        const double f = dl[i];
        if (!((sw[i >> 5] >> (i & 31)) & 1u)) {
          bb[i] = prev;
          prev = fma(-f, prev, nx);
        } else {
          bb[i] = nx;
          prev = fma(-f, nx, prev);
        }
      }
      double x1 = prev * dinv[p - 1];
      bb[p - 1] = x1;
      double nrm = x1 * x1, x2 = 0.0;
      if (p > 1) {
        x2 = x1;
        x1 = (bb[p - 2] - du[p - 2] * x2) * dinv[p - 2];
        bb[p - 2] = x1;
        nrm = fma(x1, x1, nrm);
      }
      for (int i = p - 3; i >= 0; --i) {
        const double x0 = (bb[i] - du[i] * x1 - du2[i] * x2) * dinv[i];
        bb[i] = x0;
        nrm = fma(x0, x0, nrm);
        x2 = x1;
        x1 = x0;
      }
      inv = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
    }
    s_inv = inv;
  }
  __syncthreads();
  const double inv = s_inv;
  double* y = Y + (size_t)j * p;
  for (int i = threadIdx.x; i < p; i += 32) y[i] = bb[i] * inv;
}

// back-transformation as backtransform_kernel: BT_VPB eigenvectors per block, each in registers
// and split over a group of BT_GW warps (thread t of the group owns columns t, t + 32 BT_GW, ...).
// The reflector rows stream through shared memory in chunks of rc rows, double-buffered with
// cp.async.  One pass per reflector applies it and forms the next reflector's dot with the updated
// vector (v_{r-1} spans c >= r); the group combines its warps' partials through shared memory
// under one named barrier per reflector.
constexpr int BT_GW = 4;                 // warps per vector
constexpr int BT_VPB = 2;                // vectors per block
constexpr int BT_GT = 32 * BT_GW;        // threads per vector
constexpr int BT_T = BT_GT * BT_VPB;
__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void group_bar(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(BT_GT) : "memory");
}
template <int CM>  // columns per thread: p <= CM * BT_GT (fully unrolled: every load of a pass in flight)
__global__ void __launch_bounds__(BT_T) backtransform_chunk_kernel(const double* __restrict__ Vh,
                                                                  const double* __restrict__ tau, int p,
                                                                  const Bounds* B, double* __restrict__ Y, int rc) {
  extern __shared__ double bt_smem[];
  __shared__ double red[BT_VPB][2][BT_GW];
  const int lane = threadIdx.x & 31;
  const int g = threadIdx.x / BT_GT, t = threadIdx.x % BT_GT, gw = t >> 5;
  const int k = B->k;
  const int j0 = blockIdx.x * BT_VPB;
  if (j0 >= k) return;
  const int j = j0 + g;
  const bool live = j < k;
  double* chunks = bt_smem;  // 2 x rc rows of p
  double* y = Y + (size_t)(live ? j : 0) * p;
  double yr[CM];  // this thread's columns t + BT_GT m of the vector, in registers
#pragma unroll
  for (int m = 0; m < CM; ++m) {
    const int c = t + BT_GT * m;
    yr[m] = (live && c < p) ? y[c] : 0.0;
  }
  const int nrows = p - 1;  // reflectors 0 .. p-2, applied from p-2 down
  const int nch = (nrows + rc - 1) / rc;
  auto stage = [&](int ch) {
    const int hi = p - 2 - ch * rc, lo = max(0, hi - rc + 1);
    double* buf = chunks + (size_t)(ch & 1) * rc * p;
    for (int r = lo; r <= hi; ++r)
      for (int c = r + 1 + threadIdx.x; c < p; c += BT_T)
        cp_async8(buf + (size_t)(r - lo) * p + c, Vh + (size_t)r * p + c);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // group-wide sum of one value per thread (fixed order), parity-buffered slots
  int par = 0;
  auto gsum = [&](double a) {
    a = warp_sum(a);
    if (lane == 0) red[g][par][gw] = a;
    group_bar(g);
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < BT_GW; ++w) s += red[g][par][w];
    par ^= 1;
    return s;
  };
  stage(0);
  __syncthreads();
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) {
      stage(ch + 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    if (live) {
      const int hi = p - 2 - ch * rc, lo = max(0, hi - rc + 1);
      const double* buf = chunks + (size_t)(ch & 1) * rc * p;
      const double tl = lane <= hi - lo ? __ldg(&tau[lo + lane]) : 0.0;  // this chunk's tau (rc <= 32)
      const double* __restrict__ vh = buf + (size_t)(hi - lo) * p;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int m = 0; m < CM; ++m) {
        const int c = t + BT_GT * m;
        const double x = (c > hi && c < p) ? vh[c] * yr[m] : 0.0;
        if (m & 1) a1 += x; else a0 += x;
      }
      double sr = gsum(a0 + a1) * __shfl_sync(0xffffffffu, tl, hi - lo);
      for (int r = hi; r >= lo; --r) {
        const double* __restrict__ vr = buf + (size_t)(r - lo) * p;
        if (r > lo) {
          const double* __restrict__ vn = vr - p;  // v_{r-1}
          double b0 = 0.0, b1 = 0.0;
#pragma unroll
          for (int m = 0; m < CM; ++m) {
            const int c = t + BT_GT * m;
            if (c >= r && c < p) {
              double y0 = yr[m];
              if (c > r) {
                y0 = fma(-sr, vr[c], y0);
                yr[m] = y0;
              }
              if (m & 1) b1 = fma(vn[c], y0, b1); else b0 = fma(vn[c], y0, b0);
            }
          }
          sr = gsum(b0 + b1) * __shfl_sync(0xffffffffu, tl, r - 1 - lo);
        } else {
#pragma unroll
          for (int m = 0; m < CM; ++m) {
            const int c = t + BT_GT * m;
            if (c > r && c < p) yr[m] = fma(-sr, vr[c], yr[m]);
          }
        }
      }
    }
    __syncthreads();  // buffer (ch & 1) is refilled by stage(ch + 2)
  }
  if (live) {
#pragma unroll
    for (int m = 0; m < CM; ++m) {
      const int c = t + BT_GT * m;
      if (c < p) y[c] = yr[m];
    }
  }
}

__global__ void symmetrize_kernel(double* __restrict__ A, int p) {
  // copy the lower triangle (cuBLAS syrk 'L', column-major = upper in row-major view) to a full matrix
  const int64_t total = (int64_t)p * p;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(x / p), c = (int)(x % p);
    if (c < r) A[x] = A[(int64_t)c * p + r];
  }
}

}  // namespace eig
}  // namespace l1f

using namespace l1f;
using namespace l1f::eig;

// Whether the shared-memory-resident tridiagonalisation takes a p x p matrix on this device (every
// block's rows fit in its shared memory: p <= 2000 on 148 SMs)
bool l1f_eig_dsm_applies(int p) {
  int dev = 0, nsm = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (nsm <= 0 || nsm > 256 || p < 2) return false;
  const int rmax = (p + nsm - 1) / nsm;
  const int nw = p > 1024 ? 16 : DSM_W;  // warps of the variant that runs (512 / 256 threads)
  const size_t dsm_static = sizeof(double) * (nw * (DSM_R + 1) + nw + 2 * DSM_R + 4) + 64;
  return rmax <= DSM_R && p <= 2048 && sizeof(double) * (size_t)rmax * p + dsm_static <= (size_t)optin;
}

// Eigenpairs of the symmetric p x p matrix G (column-major lower triangle as cuBLAS syrk leaves it,
// i.e. the row-major upper triangle; G is overwritten) with eigenvalue >= max(thr_abs, thr_rel *
// ||T||_gersh).  Outputs (device): lam[0 .. k) descending, Z (p x k column-major, ld p) eigenvectors.
// *k_host receives k.  Returns L1F_OK / error.
int l1f_eig_sym_above(double* G, int p, double thr_abs, double thr_rel, double* lam, double* Z, int* k_host,
                      cudaStream_t st) {
  if (p < 2) {
    set_error("eig_sym_above: p < 2");
    return L1F_ERR_UNSUPPORTED;
  }
  int dev = 0, coop = 0, nsm = 0;
  L1F_CUDA_TRY(cudaGetDevice(&dev));
  L1F_CUDA_TRY(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  L1F_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  if (!coop) {
    set_error("eig_sym_above: cooperative launch unsupported");
    return L1F_ERR_UNSUPPORTED;
  }
  int per_sm = 0;
  const int grid_target = 2 * nsm;  // two blocks per SM: 16 warps
  const int rows_max = (p + grid_target - 1) / grid_target + 1;
  const size_t tri_smem = sizeof(double) * (2 * (size_t)p + (size_t)TW * rows_max + 8);
  L1F_CUDA_TRY(cudaFuncSetAttribute(tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tri_smem));
  L1F_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tridiag_kernel, TT, tri_smem));
  const int grid = grid_target;  // the shared-memory row partials are sized for this grid
  if (per_sm < 2) {
    set_error("eig_sym_above: occupancy below two blocks per SM");
    return L1F_ERR_UNSUPPORTED;
  }
  void* buf = nullptr;
  const size_t n_d = (size_t)p;
  const size_t bytes = sizeof(double) * (6 * n_d + (size_t)p * p + (size_t)grid + 8 * n_d * (size_t)p / 8 + 64) +
                       sizeof(Bounds) + 64;
  // scratch for inverse iteration: 5 p doubles per eigenvalue (k <= p): allocated separately below
  L1F_CUDA_TRY(cudaMallocAsync(&buf, bytes, st));
  double* w = (double*)buf;
  double* d = w; w += p;
  double* e = w; w += p;
  double* e2 = w; w += p;
  double* tau = w; w += p;
  double* pv = w; w += p;
  double* part = w; w += grid;
  double* Vh = w; w += (size_t)p * p;
  Bounds* B = (Bounds*)(((uintptr_t)(w + 8) + 63) & ~(uintptr_t)63);
  symmetrize_kernel<<<nsm * 4, 256, 0, st>>>(G, p);
  int rc = L1F_OK;
  cudaError_t err = cudaSuccess;
  // shared-memory-resident form when every block's rows fit (p <= 2000 on 148 SMs)
  int optin = 0;
  L1F_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int rmax = (p + nsm - 1) / nsm;
  const size_t dsm_smem = sizeof(double) * (size_t)rmax * p;
  const size_t dsm_static = sizeof(double) * (DSM_W * (DSM_R + 1) + DSM_W + 2 * DSM_R + 4) + 64;
  const bool use_dsm = option(L1F_OPT_SEED_EIG_DSM) != 0 && l1f_eig_dsm_applies(p);
  (void)dsm_static;
  void* dsm_scr = nullptr;
  if (use_dsm) {
    const size_t slots = 2 * (size_t)p * p + (size_t)p * nsm;
    L1F_CUDA_TRY(cudaMallocAsync(&dsm_scr, sizeof(double) * slots + sizeof(unsigned) * (size_t)p, st));
    double* ybuf = (double*)dsm_scr;
    double* rowbuf = ybuf + (size_t)p * p;
    double* dpart = rowbuf + (size_t)p * p;
    unsigned* cnt = (unsigned*)(dpart + (size_t)p * nsm);
    L1F_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned) * (size_t)p, st));
    const double* Ac = G;
    void* dargs[] = {(void*)&Ac, &p, &d, &e, &tau, &Vh, &ybuf, &dpart, &rowbuf, &cnt};
    // 256 threads per block up to p = 1024, 512 beyond (measured, tools/r2/dsm_threads_ab.py: 128
    // threads cost cfg3 +12 %; 512 threads cfg2 +8 %, cfg3 even, cfg5 -5 %)
    const int nth = p > 1024 ? 512 : DSM_T;
    void* fn = nth == 512 ? (rmax <= 8 ? (void*)tridiag_dsm_kernel<4, 512, 8> : (void*)tridiag_dsm_kernel<4, 512, 16>)
               : p <= 2 * DSM_T ? (rmax <= 8 ? (void*)tridiag_dsm_kernel<2, DSM_T, 8> : (void*)tridiag_dsm_kernel<2, DSM_T, 16>)
                                : (rmax <= 8 ? (void*)tridiag_dsm_kernel<4, DSM_T, 8> : (void*)tridiag_dsm_kernel<4, DSM_T, 16>);
    L1F_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm_smem));
    err = cudaLaunchCooperativeKernel(fn, nsm, nth, dargs, dsm_smem, st);
  } else {
    void* args[] = {&G, &p, &d, &e, &tau, &Vh, &pv, &part};
    err = cudaLaunchCooperativeKernel((void*)tridiag_kernel, grid, TT, args, tri_smem, st);
  }
  if (err != cudaSuccess) {
    // not all blocks co-resident (an SM-limited context: MPS / green contexts): the caller takes
    // its library path; anything else is an error
    const bool too_large = err == cudaErrorCooperativeLaunchTooLarge;
    (void)cudaGetLastError();
    set_error("eig_sym_above: tridiagonalisation launch failed: %s", cudaGetErrorString(err));
    rc = too_large ? L1F_ERR_UNSUPPORTED : L1F_ERR_CUDA;
  }
  if (rc == L1F_OK) {
    bounds_kernel<<<1, 256, 0, st>>>(d, e, e2, p, thr_abs, thr_rel, B);
    Bounds hb;
    err = cudaMemcpyAsync(&hb, B, sizeof(Bounds), cudaMemcpyDeviceToHost, st);
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);
    if (err != cudaSuccess) {
      set_error("eig_sym_above: %s", cudaGetErrorString(err));
      rc = L1F_ERR_CUDA;
    } else {
      const int k = hb.k;
      *k_host = k;
      if (k > 0) {
        void* sc = nullptr;
        const int kp = (k + 31) / 32 * 32;
        err = cudaMallocAsync(&sc, sizeof(double) * (size_t)kp * 6 * p, st);
        if (err == cudaSuccess) {
          bisect_kernel<<<(k + 7) / 8, 256, 0, st>>>(d, e2, p, B, 8, lam);
          const size_t inv_smem = sizeof(double) * 5 * (size_t)p + sizeof(unsigned) * ((p + 31) / 32 + 1);
          if (inv_smem <= 200 * 1024) {
            cudaFuncSetAttribute(inverse_iter_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)inv_smem);
            inverse_iter_smem_kernel<<<k, 32, inv_smem, st>>>(d, e, p, B, lam, Z);
          } else {
            inverse_iter_kernel<<<(k + 31) / 32, 32, 0, st>>>(d, e, p, B, lam, Z, (double*)sc, kp);
          }
          cudaFuncSetAttribute(cgs2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(double) * k));
          cgs2_kernel<<<1, 1024, sizeof(double) * (size_t)k, st>>>(Z, p, B, d, e, lam);
          rq_kernel<<<(k + 7) / 8, 256, 0, st>>>(Z, p, B, d, e, lam);
          // the vectors live in registers; the reflector chunks (double-buffered) in shared memory,
          // sized for two blocks per SM
          const int bt_rc = (int)std::min<size_t>(32, (100 * 1024) / (2 * sizeof(double) * p));
          if (bt_rc >= 2 && p <= 16 * BT_GT) {
            const size_t bt_smem = 2 * sizeof(double) * (size_t)bt_rc * p;
            auto fn = p <= 4 * BT_GT ? backtransform_chunk_kernel<4>
                    : p <= 8 * BT_GT ? backtransform_chunk_kernel<8> : backtransform_chunk_kernel<16>;
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bt_smem);
            fn<<<(k + BT_VPB - 1) / BT_VPB, BT_T, bt_smem, st>>>(Vh, tau, p, B, Z, bt_rc);
          } else {
            backtransform_kernel<<<k, 256, sizeof(double) * (size_t)p, st>>>(Vh, tau, p, B, Z);
          }
          err = cudaGetLastError();
          cudaFreeAsync(sc, st);
        }
        if (err != cudaSuccess) {
          set_error("eig_sym_above: %s", cudaGetErrorString(err));
          rc = L1F_ERR_CUDA;
        }
      }
    }
  }
  if (dsm_scr) cudaFreeAsync(dsm_scr, st);
  cudaFreeAsync(buf, st);
  return rc;
}
