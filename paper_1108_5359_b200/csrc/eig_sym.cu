// Eigenpairs of a symmetric matrix above a threshold, hand-written (the Gram step of the large-seed
// SVT, seed.cu svt_gram / svd_gram; reference: the SVD inside svt_with_rank, matcore.py:73-105).
//
//   1. Householder tridiagonalisation T = Q^T G Q (LAPACK dsytd2 'L' order), one cooperative kernel:
//      per column two grid-wide barriers (p = tau A v with partial dot products; then the rank-2
//      update A -= v w^T + w v^T of the trailing block); the full symmetric matrix is kept so rows
//      are contiguous; every block recomputes the reflector redundantly (no extra barrier).
//   2. The k eigenvalues of T above the threshold: a Sturm count gives k, each eigenvalue is
//      bracketed by multisection (one warp per eigenvalue, 32 Sturm counts per round).
//   3. Eigenvectors of T by inverse iteration (tridiagonal LU with partial pivoting, two solves per
//      eigenvalue, one thread each), then modified Gram-Schmidt over the k vectors in descending
//      order (nearly equal shifts of a cluster give nearly parallel vectors: MGS keeps the cluster's
//      span) and Rayleigh quotients as the final eigenvalues.
//   4. Back-transformation Z = Q Y, one warp per eigenvector (reflectors applied in reverse order).
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

// number of eigenvalues of T (d, e2 = e^2) below x
__device__ __forceinline__ int sturm_below(const double* __restrict__ d, const double* __restrict__ e2, int p, double x,
                                           double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0.0;
  for (int j = 1; j < p; ++j) {
    q = (d[j] - x) - e2[j - 1] / q;
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
    B->k = p - sturm_below(d, e2, p, thr, pivmin);
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
    const int c = sturm_below(d, e2, p, x, pivmin);  // eigenvalues below x
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
  // alone leaves the vectors orthogonal to ~eps ||T|| / gap <= 1e-12
  const double gap_tol = 1e-4 * fmax(fabs(B->hi), fabs(B->lo));
  int cstart = 0;
  for (int j = 0; j < k; ++j) {
    if (j > 0 && !(fabs(lam[j - 1] - lam[j]) < gap_tol)) cstart = j;
    double* yj = Y + (size_t)j * p;
    for (int pass = 0; pass < 2 && cstart < j; ++pass) {
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
    double q = 0.0;
    for (int r = threadIdx.x; r < p; r += blockDim.x) {
      double ty = d[r] * yj[r];
      if (r > 0) ty = fma(e[r - 1], yj[r - 1], ty);
      if (r + 1 < p) ty = fma(e[r], yj[r + 1], ty);
      q = fma(yj[r], ty, q);
    }
    q = block_sum_det(q, red);
    if (threadIdx.x == 0) lam[j] = q;
    __syncthreads();
  }
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
  void* args[] = {&G, &p, &d, &e, &tau, &Vh, &pv, &part};
  cudaError_t err = cudaLaunchCooperativeKernel((void*)tridiag_kernel, grid, TT, args, tri_smem, st);
  if (err != cudaSuccess) {
    set_error("eig_sym_above: tridiagonalisation launch failed: %s", cudaGetErrorString(err));
    rc = L1F_ERR_CUDA;
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
          inverse_iter_kernel<<<(k + 31) / 32, 32, 0, st>>>(d, e, p, B, lam, Z, (double*)sc, kp);
          cudaFuncSetAttribute(cgs2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(double) * k));
          cgs2_kernel<<<1, 1024, sizeof(double) * (size_t)k, st>>>(Z, p, B, d, e, lam);
          backtransform_kernel<<<k, 256, sizeof(double) * (size_t)p, st>>>(Vh, tau, p, B, Z);
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
  cudaFreeAsync(buf, st);
  return rc;
}
