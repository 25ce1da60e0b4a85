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
// Dynamic shared memory: v and w of the current step (2 p doubles), so the trailing-matrix streams
// are the only global loads; rows are unrolled 4-deep to keep loads in flight.
__global__ void __launch_bounds__(TT) tridiag_kernel(double* __restrict__ A, int p, double* __restrict__ d,
                                                   double* __restrict__ e, double* __restrict__ tau_out,
                                                   double* __restrict__ Vh, double* __restrict__ pv,
                                                   double* __restrict__ part) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sv[];  // v: [0, p), w: [p, 2p)
  double* sw = sv + p;
  __shared__ double red[TW + 1];
  const int lane = threadIdx.x % 32;
  const int gwarp = blockIdx.x * TW + threadIdx.x / 32, nwarps = gridDim.x * TW;
  for (int i = 0; i + 1 < p; ++i) {
    const double* rowi = A + (size_t)i * p;
    double s = 0.0;
    for (int c = i + 2 + threadIdx.x; c < p; c += TT) s = fma(rowi[c], rowi[c], s);
    const double xnorm2 = block_sum_det(s, red);
    const double alpha = rowi[i + 1];
    double tau = 0.0, beta = alpha, scale = 0.0;
    if (xnorm2 > 0.0) {
      beta = -copysign(sqrt(fma(alpha, alpha, xnorm2)), alpha);
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      d[i] = rowi[i];
      e[i] = beta;
      tau_out[i] = tau;
    }
    if (tau == 0.0) {  // H = I: nothing to update (uniform across the grid)
      for (int c = i + 1 + blockIdx.x * TT + threadIdx.x; c < p; c += gridDim.x * TT)
        Vh[(size_t)i * p + c] = c == i + 1 ? 1.0 : 0.0;
      continue;
    }
    for (int c = i + 1 + threadIdx.x; c < p; c += TT) sv[c] = c == i + 1 ? 1.0 : rowi[c] * scale;
    __syncthreads();
    // p_r = tau * sum_c A[r][c] v[c]  (rows r = i+1 .. p-1, one warp per row), partial p.v
    double dot = 0.0;
    const int c0 = i + 1;
    for (int r = c0 + gwarp; r < p; r += nwarps) {
      const double* ar = A + (size_t)r * p;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int c = c0 + lane;
      for (; c + 96 < p; c += 128) {
        a0 = fma(ar[c], sv[c], a0);
        a1 = fma(ar[c + 32], sv[c + 32], a1);
        a2 = fma(ar[c + 64], sv[c + 64], a2);
        a3 = fma(ar[c + 96], sv[c + 96], a3);
      }
      for (; c < p; c += 32) a0 = fma(ar[c], sv[c], a0);
      double a = warp_sum((a0 + a1) + (a2 + a3)) * tau;
      if (lane == 0) {
        pv[r] = a;
        Vh[(size_t)i * p + r] = sv[r];
        dot = fma(a, sv[r], dot);
      }
    }
    dot = block_sum_det(dot, red);
    if (threadIdx.x == 0) part[blockIdx.x] = dot;
    grid.sync();
    double pvdot = 0.0;
    for (int b = 0; b < (int)gridDim.x; ++b) pvdot += part[b];
    const double K = -0.5 * tau * pvdot;
    for (int c = c0 + threadIdx.x; c < p; c += TT) sw[c] = fma(K, sv[c], pv[c]);
    __syncthreads();
    // A[r][c] -= v[r] w[c] + w[r] v[c],  w = p + K v   (trailing block rows/cols i+1 .. p-1)
    for (int r = c0 + gwarp; r < p; r += nwarps) {
      double* ar = A + (size_t)r * p;
      const double vr = sv[r], wr = sw[r];
      int c = c0 + lane;
      for (; c + 96 < p; c += 128) {
        const double x0 = ar[c], x1 = ar[c + 32], x2 = ar[c + 64], x3 = ar[c + 96];
        ar[c] = x0 - fma(vr, sw[c], wr * sv[c]);
        ar[c + 32] = x1 - fma(vr, sw[c + 32], wr * sv[c + 32]);
        ar[c + 64] = x2 - fma(vr, sw[c + 64], wr * sv[c + 64]);
        ar[c + 96] = x3 - fma(vr, sw[c + 96], wr * sv[c + 96]);
      }
      for (; c < p; c += 32) ar[c] -= fma(vr, sw[c], wr * sv[c]);
    }
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) d[p - 1] = A[(size_t)(p - 1) * p + p - 1];
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
// one thread per eigenvalue; Y column j (length p, contiguous) = the normalised vector
__global__ void inverse_iter_kernel(const double* __restrict__ d, const double* __restrict__ e, int p, const Bounds* B,
                                    const double* __restrict__ lam, double* __restrict__ Y, double* __restrict__ scratch) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= B->k) return;
  const double s = lam[j];
  double* dl = scratch + (size_t)j * 5 * p;  // multipliers
  double* dd = dl + p;                         // U diagonal
  double* du = dd + p;                         // U first superdiagonal
  double* du2 = du + p;                        // U second superdiagonal
  double* y = Y + (size_t)j * p;
  // factor (T - sI) = L U with partial pivoting (dgttrf); the row-interchange flags are kept in y
  // (overwritten by the solution at the end), the right-hand side in the fifth scratch vector
  const double eps = 2.220446049250313e-16;
  const double tnorm = fmax(fabs(B->hi), fabs(B->lo)) + 1.0e-300;
  for (int i = 0; i < p; ++i) {
    dd[i] = d[i] - s;
    du[i] = i + 1 < p ? e[i] : 0.0;
    du2[i] = 0.0;
  }
  for (int i = 0; i + 1 < p; ++i) {
    const double sub = e[i];  // subdiagonal (row i+1, col i)
    if (fabs(dd[i]) >= fabs(sub)) {
      const double f = dd[i] != 0.0 ? sub / dd[i] : 0.0;
      dl[i] = f;
      dd[i + 1] -= f * du[i];
      y[i] = 0.0;  // no interchange
    } else {
      const double f = dd[i] / sub;
      dd[i] = sub;
      dl[i] = f;
      const double t = du[i];
      du[i] = dd[i + 1];
      dd[i + 1] = t - f * dd[i + 1];
      if (i + 2 < p) {
        du2[i] = du[i + 1];
        du[i + 1] = -f * du[i + 1];
      }
      y[i] = 1.0;  // interchange
    }
  }
  for (int i = 0; i < p; ++i)
    if (fabs(dd[i]) < eps * tnorm) dd[i] = copysign(eps * tnorm, dd[i] == 0.0 ? 1.0 : dd[i]);
  // right-hand side: a fixed, deterministic vector
  double* b = du2 + p;
  for (int i = 0; i < p; ++i) b[i] = 1.0 + 0.5 * sin(0.7 * (double)i + 0.3 * (double)j);
  for (int rep = 0; rep < 2; ++rep) {
    // forward: apply L (with interchanges)
    for (int i = 0; i + 1 < p; ++i) {
      if (y[i] == 0.0) {
        b[i + 1] -= dl[i] * b[i];
      } else {
        const double t = b[i];
        b[i] = b[i + 1];
        b[i + 1] = t - dl[i] * b[i + 1];
      }
    }
    // back substitution with U (diag dd, super du, du2)
    double xn = b[p - 1] / dd[p - 1];
    b[p - 1] = xn;
    if (p > 1) {
      b[p - 2] = (b[p - 2] - du[p - 2] * b[p - 1]) / dd[p - 2];
    }
    for (int i = p - 3; i >= 0; --i) b[i] = (b[i] - du[i] * b[i + 1] - du2[i] * b[i + 2]) / dd[i];
    // normalise (and scale to avoid overflow in the next solve)
    double nrm = 0.0;
    for (int i = 0; i < p; ++i) nrm = fma(b[i], b[i], nrm);
    nrm = sqrt(nrm);
    const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
    for (int i = 0; i < p; ++i) b[i] *= inv;
  }
  for (int i = 0; i < p; ++i) y[i] = b[i];
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
  for (int j = 0; j < k; ++j) {
    double* yj = Y + (size_t)j * p;
    for (int pass = 0; pass < 2; ++pass) {
      for (int i = warp; i < j; i += nw) {
        const double* yi = Y + (size_t)i * p;
        double s = 0.0;
        for (int r = lane; r < p; r += 32) s = fma(yi[r], yj[r], s);
        s = warp_sum(s);
        if (lane == 0) sdot[i] = s;
      }
      __syncthreads();
      for (int r = threadIdx.x; r < p; r += blockDim.x) {
        double v = yj[r];
        for (int i = 0; i < j; ++i) v = fma(-sdot[i], Y[(size_t)i * p + r], v);
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

// Z column j = Q y_j, Q = H_0 H_1 ... H_{p-2}: apply H_{p-2} .. H_0 in turn; one warp per column
__global__ void backtransform_kernel(const double* __restrict__ Vh, const double* __restrict__ tau, int p,
                                     const Bounds* B, double* __restrict__ Y) {
  const int lane = threadIdx.x % 32;
  const int j = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (j >= B->k) return;
  double* y = Y + (size_t)j * p;
  for (int i = p - 2; i >= 0; --i) {
    const double t = tau[i];
    if (t == 0.0) continue;
    const double* v = Vh + (size_t)i * p;
    double s = 0.0;
    for (int c = i + 1 + lane; c < p; c += 32) s = fma(v[c], y[c], s);
    s = warp_sum(s) * t;
    for (int c = i + 1 + lane; c < p; c += 32) y[c] = fma(-s, v[c], y[c]);
    __syncwarp();
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
  const size_t tri_smem = sizeof(double) * 2 * (size_t)p;
  L1F_CUDA_TRY(cudaFuncSetAttribute(tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tri_smem));
  L1F_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tridiag_kernel, TT, tri_smem));
  const int64_t want = option(L1F_OPT_EIG_GRID);  // A/B: blocks of the tridiagonalisation (0 = auto)
  int grid = std::max(1, std::min(nsm * std::max(per_sm, 1), std::max(1, (p + TW - 1) / TW)));
  if (want > 0) grid = (int)std::min<int64_t>(want, (int64_t)nsm * std::max(per_sm, 1));
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
        err = cudaMallocAsync(&sc, sizeof(double) * (size_t)k * 5 * p, st);
        if (err == cudaSuccess) {
          bisect_kernel<<<(k + 7) / 8, 256, 0, st>>>(d, e2, p, B, 8, lam);
          inverse_iter_kernel<<<(k + 63) / 64, 64, 0, st>>>(d, e, p, B, lam, Z, (double*)sc);
          cudaFuncSetAttribute(cgs2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(double) * k));
          cgs2_kernel<<<1, 1024, sizeof(double) * (size_t)k, st>>>(Z, p, B, d, e, lam);
          backtransform_kernel<<<(k + 7) / 8, 256, 0, st>>>(Vh, tau, p, B, Z);
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
