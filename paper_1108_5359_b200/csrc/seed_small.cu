// Seed PCP for small blocks, entirely on the device: one persistent CTA runs the whole inexact-ALM
// loop of solve_pcp (pcp_adm.py:90-140) with a hand-written one-sided Jacobi SVD for the singular
// value thresholding (matcore.py:73-105), and a second kernel factors the final seed L
// (recover_seed, l1filter.py:90-113 -> matcore.svd).  No library call and no host round trip: the
// host reads one status record after the loop.  Used when the Jacobi working set (X, V) fits in
// shared memory (square blocks up to 113 x 113: every l1-filtering seed up to rank 11 — configs 1
// and 4, the reference's test and golden sizes; see l1f_seed_small_applies).
//
// One ALM iteration (all in the CTA, data in global memory / L1 / L2):
//   S = shrink((M - L) + Y/b, lam/b);  W = (M - S) + Y/b                  (pcp_adm.py:122-123)
//   X = T V            T = W (m >= n) or W^T (m < n): tall mt x nt, V warm-started from the
//                      previous iteration's right singular vectors (orthogonal nt x nt)
//   one-sided Jacobi on the columns of X, rotating V alongside, until every column pair is
//   orthogonal to eps * sqrt(mt): X = U diag(sigma), T = U diag(sigma) V^T
//   L = sum_{sigma_c > 1/b} x_c (1 - 1/(b sigma_c)) v_c^T  (= U (sigma - 1/b)_+ V^T, matcore.py:96-105)
//   R = (M - L) - S;  res = ||R||_F / ||M||_F;  Y += b R;  stop at res <= tol  (pcp_adm.py:124-135)
//   b = min(rho b, b_max)
// Reductions are fixed-order trees (deterministic).  The warm start makes X nearly orthogonal
// in the directions that persist between iterations, so most iterations need few sweeps.
#include "common.cuh"

#include <cmath>

namespace l1f {
namespace seedsm {

constexpr int NT = 1024;           // threads of the persistent CTA
constexpr int64_t kSmallMaxDim = 256;
constexpr int NW = NT / 32;
constexpr int kMaxSweeps = 60;

struct Status {
  int iters, rank, converged, err, sweeps_total;
  double residual, beta_final;
};

struct Shape {
  int m, n, mt, nt;  // W is m x n (row-major, ld n); T is mt x nt (tall)
  bool tr;           // T = W^T
};

__device__ __forceinline__ double t_at(const double* __restrict__ W, const Shape& sh, int i, int j) {
  return sh.tr ? W[(int64_t)j * sh.n + i] : W[(int64_t)i * sh.n + j];
}

// deterministic block sum: warp trees, then warp 0 over the NW partials in order
__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < NW ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[NW] = t;
  }
  __syncthreads();
  return red[NW];
}

// X_cm[c][i] = sum_j T[i][j] V_cm[c][j]  (j in order).  Consecutive threads take consecutive c
// for one row i, so the T element is a broadcast and V (odd column stride) is conflict-free.
__device__ void gemm_tv(const double* __restrict__ W, const Shape& sh, const double* V, int ldv, double* X,
                        int ldx) {
  const int total = sh.mt * sh.nt;
  for (int e = threadIdx.x; e < total; e += NT) {
    const int i = e / sh.nt, c = e - i * sh.nt;
    const double* v = V + (int64_t)c * ldv;
    double acc = 0.0;
    if (sh.tr) {
      for (int j = 0; j < sh.nt; ++j) acc = fma(W[(int64_t)j * sh.n + i], v[j], acc);
    } else {
      const double* w = W + (int64_t)i * sh.n;
      for (int j = 0; j < sh.nt; ++j) acc = fma(w[j], v[j], acc);
    }
    X[(int64_t)c * ldx + i] = acc;
  }
}

// One-sided Jacobi on the nt columns of X (length mt, column stride ldx), rotating V's columns
// (length nt, stride ldv).  Round-robin (circle) ordering: nt/2 disjoint pairs per round, one group
// of G lanes per pair (G = 16 when there are more pairs than warps).  X and V sit in shared memory
// whenever they fit (the dependent dot -> rotate chain of a round is latency-bound).
// Returns the number of sweeps, or -1 if not converged.
template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int G>
__device__ int jacobi_g(double* X, int ldx, double* V, int ldv, int mt, int nt, int* flag, double loose_below) {
  constexpr int NG = NT / G;
  const int gl = threadIdx.x % G, grp = threadIdx.x / G;
  const int N = nt + (nt & 1);
  const double tolj = 2.220446049250313e-16 * sqrt((double)mt);
  const double tolj2 = tolj * tolj;
  for (int sweep = 1; sweep <= kMaxSweeps; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int r = 0; r < N - 1; ++r) {
      for (int p0 = 0; p0 < N / 2; p0 += NG) {  // uniform trip count: shuffles need full warps
        const int p = p0 + grp;
        int ca = nt, cb = nt;
        if (p < N / 2) {
          const int q = N - 1 - p;
          ca = p == 0 ? 0 : ((p - 1 + r) % (N - 1)) + 1;
          cb = ((q - 1 + r) % (N - 1)) + 1;
          if (ca > cb) { const int t = ca; ca = cb; cb = t; }
        }
        const bool live = ca < nt && cb < nt;  // dummy column of an odd nt / idle group
        double* xa = X + (int64_t)(live ? ca : 0) * ldx;
        double* xb = X + (int64_t)(live ? cb : 0) * ldx;
        double a = 0.0, b = 0.0, c = 0.0;
        if (live)
          for (int i = gl; i < mt; i += G) {
            const double u = xa[i], v = xb[i];
            a = fma(u, u, a);
            b = fma(v, v, b);
            c = fma(u, v, c);
          }
        a = group_sum<G>(a);
        b = group_sum<G>(b);
        c = group_sum<G>(c);
        // |c| > tol * sqrt(a b), squared: no square roots on the test (every warp runs this math for
        // its pairs, and the round is instruction-issue bound)
        // deep-bulk pairs (both squared norms below loose_below = eta^2 / 4 in the ALM) only need
        // cosines below 1e-8: then every singular value of the deep-bulk columns stays below
        // sqrt(1/4 + nt * 1e-8) eta < eta, so the thresholded result is that of the other columns,
        // which are orthogonalised to eps * sqrt(mt) against everything (strict for the SVD itself)
        const double tol2 = (a < loose_below && b < loose_below) ? 1e-16 : tolj2;
        if (!live || !(a > 0.0) || !(b > 0.0) || !(c * c > tol2 * a * b)) continue;
        // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)) with zeta = (b - a) / 2c, multiplied through by
        // |2c|: one square root and one division; cs = 1 / sqrt(1 + t^2) by rsqrt
        const double d = b - a;
        const double c2 = 2.0 * c;
        const double t = (d >= 0.0 ? c2 : -c2) / (fabs(d) + sqrt(fma(d, d, c2 * c2)));
        const double cs = rsqrt(fma(t, t, 1.0));
        const double sn = cs * t;
        for (int i = gl; i < mt; i += G) {
          const double u = xa[i], v = xb[i];
          xa[i] = cs * u - sn * v;
          xb[i] = sn * u + cs * v;
        }
        double* va = V + (int64_t)ca * ldv;
        double* vb = V + (int64_t)cb * ldv;
        for (int i = gl; i < nt; i += G) {
          const double u = va[i], v = vb[i];
          va[i] = cs * u - sn * v;
          vb[i] = sn * u + cs * v;
        }
        if (gl == 0) *flag = 1;
      }
      __syncthreads();
    }
    if (*flag == 0) return sweep;
    __syncthreads();
  }
  return -1;
}

__device__ int jacobi(double* X, int ldx, double* V, int ldv, int mt, int nt, int* flag, double loose_below) {
  return (nt + 1) / 2 > NW ? jacobi_g<16>(X, ldx, V, ldv, mt, nt, flag, loose_below)
                           : jacobi_g<32>(X, ldx, V, ldv, mt, nt, flag, loose_below);
}

// per-column sigma = ||x_c|| (one warp per column)
__device__ void column_norms(const double* X, int ldx, int mt, int nt, double* __restrict__ sig) {
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  for (int c = warp; c < nt; c += NW) {
    const double* x = X + (int64_t)c * ldx;
    double a = 0.0;
    for (int i = lane; i < mt; i += 32) a = fma(x[i], x[i], a);
    a = warp_sum(a);
    if (lane == 0) sig[c] = sqrt(a);
  }
}

struct Work {
  double *Y, *W, *X, *V, *sig, *fac;
  int* act;
};

__global__ void __launch_bounds__(NT, 1)
alm_small_kernel(const double* __restrict__ M, int64_t ldm, int m, int n, double lam, double tol, double beta0,
                 double rho, double beta_max, int max_iter, double* __restrict__ L, double* __restrict__ S,
                 Work w, int ldx, int ldv, int use_smem, Status* st) {
  extern __shared__ double smem_xv[];
  __shared__ double red[NW + 1];
  __shared__ int flag, nact;
  Shape sh;
  sh.m = m; sh.n = n; sh.tr = m < n;
  sh.mt = sh.tr ? n : m;
  sh.nt = sh.tr ? m : n;
  const int64_t count = (int64_t)m * n;
  const int tid = threadIdx.x;
  // ||M||_F (frobenius_norm, pcp_adm.py:97)
  double acc = 0.0;
  for (int64_t e = tid; e < count; e += NT) {
    const double v = M[(e / n) * ldm + e % n];
    acc = fma(v, v, acc);
  }
  const double norm_m = sqrt(block_sum(acc, red));
  for (int64_t e = tid; e < count; e += NT) {
    L[e] = 0.0;
    S[e] = 0.0;
    w.Y[e] = 0.0;
  }
  if (tid == 0) {
    st->iters = 0; st->rank = 0; st->converged = 0; st->err = 0; st->sweeps_total = 0;
    st->residual = 1.0; st->beta_final = 0.0;
  }
  if (norm_m == 0.0) {  // pcp_adm.py:99-105
    if (tid == 0) { st->iters = 1; st->residual = 0.0; st->converged = 1; }
    return;
  }
  double beta = beta0;
  if (!(beta0 > 0.0)) {
    // spectral_norm_estimate (pcp_adm.py:69-87): 25 power steps from the all-ones vector;
    // w (m) and v (n) live in the X / fac buffers
    double* v = w.X;
    double* wv = w.X + n;
    for (int j = tid; j < n; j += NT) v[j] = 1.0 / sqrt((double)n);
    __syncthreads();
    double sigma = 0.0;
    for (int k = 0; k < 25; ++k) {
      double part = 0.0;
      for (int i = tid; i < m; i += NT) {
        double a = 0.0;
        for (int j = 0; j < n; ++j) a = fma(M[(int64_t)i * ldm + j], v[j], a);
        wv[i] = a;
        part = fma(a, a, part);
      }
      const double nw = sqrt(block_sum(part, red));
      if (nw == 0.0) { sigma = 0.0; break; }
      part = 0.0;
      for (int j = tid; j < n; j += NT) {
        double a = 0.0;
        for (int i = 0; i < m; ++i) a = fma(M[(int64_t)i * ldm + j], wv[i] / nw, a);
        v[j] = a;
        part = fma(a, a, part);
      }
      sigma = sqrt(block_sum(part, red));
      if (sigma == 0.0) break;
      for (int j = tid; j < n; j += NT) v[j] /= sigma;
      __syncthreads();
    }
    beta = 1.25 / (sigma > DBL_MIN ? sigma : DBL_MIN);
  }
  const double bmax = beta_max > 0.0 ? beta_max : 1e7 * beta;
  // X, V in shared memory (l1f_seed_small_applies admits only blocks whose working set fits):
  // pointers derived from the shared array, so the Jacobi loads and stores are LDS / STS
  (void)use_smem;
  double* X = smem_xv;
  double* V = smem_xv + (size_t)ldx * sh.nt;
  // V = I (warm start for the first iteration)
  for (int e = tid; e < sh.nt * ldv; e += NT) V[e] = (e / ldv == e % ldv) ? 1.0 : 0.0;
  __syncthreads();
  double residual = 1.0;
  int rank = 0, it = 0, converged = 0, sweeps_total = 0;
  for (it = 1; it <= max_iter; ++it) {
    const double thr = lam / beta, eta = 1.0 / beta;
    for (int64_t e = tid; e < count; e += NT) {
      const double mv = M[(e / n) * ldm + e % n];
      const double yb = w.Y[e] / beta;
      const double s = shrink((mv - L[e]) + yb, thr);
      S[e] = s;
      w.W[e] = (mv - s) + yb;
    }
    __syncthreads();
    gemm_tv(w.W, sh, V, ldv, X, ldx);
    __syncthreads();
    const int sw = jacobi(X, ldx, V, ldv, sh.mt, sh.nt, &flag, 0.25 * eta * eta);
    if (sw < 0) {
      if (tid == 0) st->err = L1F_ERR_SVD;
      return;
    }
    sweeps_total += sw;
    column_norms(X, ldx, sh.mt, sh.nt, w.sig);
    __syncthreads();
    if (tid == 0) {  // the retained columns, in column order
      int k = 0;
      for (int c = 0; c < sh.nt; ++c) {
        const double sg = w.sig[c];
        if (sg > 0.0 && sg - eta > 0.0) {
          w.act[k] = c;
          w.fac[k] = (sg - eta) / sg;
          ++k;
        }
      }
      nact = k;
    }
    __syncthreads();
    rank = nact;
    // L = sum_c x_c f_c v_c^T ; R = (M - L) - S ; Y += b R ; ||R||^2
    acc = 0.0;
    for (int64_t e = tid; e < count; e += NT) {
      const int i = (int)(e / n), j = (int)(e % n);
      const int ti = sh.tr ? j : i, tj = sh.tr ? i : j;
      double l = 0.0;
      for (int q = 0; q < rank; ++q) {
        const int c = w.act[q];
        l = fma(X[(int64_t)c * ldx + ti] * w.fac[q], V[(int64_t)c * ldv + tj], l);
      }
      L[e] = l;
      const double r = (M[(int64_t)i * ldm + j] - l) - S[e];
      acc = fma(r, r, acc);
      w.Y[e] = w.Y[e] + beta * r;
    }
    residual = sqrt(block_sum(acc, red)) / norm_m;
    if (!isfinite(residual)) {
      if (tid == 0) { st->err = L1F_ERR_DIVERGED; st->iters = it; st->beta_final = beta; }
      return;
    }
    if (residual <= tol) { converged = 1; break; }
    beta = fmin(rho * beta, bmax);
  }
  if (it > max_iter) it = max_iter;
  if (tid == 0) {
    st->iters = it; st->rank = rank; st->converged = converged; st->residual = residual;
    st->beta_final = beta; st->sweeps_total = sweeps_total;
  }
}

// Thin SVD of a small matrix (min(m, n) <= kSmallMaxDim): one-sided Jacobi from V = I, singular
// values sorted descending (ties by column), U = x_c / sigma_c (zero for sigma_c = 0).
// U (m x p), V (n x p) row-major, p = min(m, n).
__global__ void __launch_bounds__(NT, 1)
svd_small_kernel(const double* __restrict__ A, int64_t lda, int m, int n, double* __restrict__ U,
                 double* __restrict__ sig, double* __restrict__ Vout, double* Xg, double* Vg, double* s_tmp,
                 int* order, int ldx, int ldv, int use_smem, Status* st) {
  extern __shared__ double smem_xv[];
  __shared__ int flag;
  Shape sh;
  sh.m = m; sh.n = n; sh.tr = m < n;
  sh.mt = sh.tr ? n : m;
  sh.nt = sh.tr ? m : n;
  const int tid = threadIdx.x;
  (void)use_smem; (void)Xg; (void)Vg;
  double* X = smem_xv;
  double* V = smem_xv + (size_t)ldx * sh.nt;
  for (int e = tid; e < sh.nt * ldv; e += NT) V[e] = (e / ldv == e % ldv) ? 1.0 : 0.0;
  // X = T (V = I) from A with its leading dimension
  for (int e = tid; e < sh.mt * sh.nt; e += NT) {
    const int c = e / sh.mt, i = e - c * sh.mt;
    X[(int64_t)c * ldx + i] = sh.tr ? A[(int64_t)c * lda + i] : A[(int64_t)i * lda + c];
  }
  __syncthreads();
  const int sw = jacobi(X, ldx, V, ldv, sh.mt, sh.nt, &flag, 0.0);
  if (sw < 0) {
    if (tid == 0) st->err = L1F_ERR_SVD;
    return;
  }
  column_norms(X, ldx, sh.mt, sh.nt, s_tmp);
  __syncthreads();
  // rank sort, descending, ties by column index
  for (int c = tid; c < sh.nt; c += NT) {
    const double v = s_tmp[c];
    int pos = 0;
    for (int d = 0; d < sh.nt; ++d) {
      const double u = s_tmp[d];
      pos += (u > v) || (u == v && d < c);
    }
    order[pos] = c;
  }
  __syncthreads();
  const int p = sh.nt;
  for (int k = tid; k < p; k += NT) sig[k] = s_tmp[order[k]];
  // left vectors of T: x_c / sigma_c (mt x p); right vectors: V columns (nt x p)
  double* Ut = sh.tr ? Vout : U;  // T = W^T: T's left vectors are W's right vectors
  double* Vt = sh.tr ? U : Vout;
  for (int e = tid; e < sh.mt * p; e += NT) {
    const int i = e / p, k = e - i * p;
    const int c = order[k];
    const double sg = s_tmp[c];
    Ut[e] = sg > 0.0 ? X[(int64_t)c * ldx + i] / sg : 0.0;
  }
  for (int e = tid; e < sh.nt * p; e += NT) {
    const int j = e / p, k = e - j * p;
    Vt[e] = V[(int64_t)order[k] * ldv + j];
  }
  if (tid == 0) { st->err = 0; st->sweeps_total = sw; }
}

}  // namespace seedsm
}  // namespace l1f

using namespace l1f;
using namespace l1f::seedsm;

namespace {
// column strides (odd: conflict-free shared-memory access) and whether X, V fit in shared memory
struct XvLayout {
  int ldx, ldv, use_smem;
  size_t smem;
};
XvLayout xv_layout(int64_t mt, int64_t nt) {
  XvLayout L;
  L.ldx = (int)(mt | 1);
  L.ldv = (int)(nt | 1);
  const size_t bytes = sizeof(double) * ((size_t)L.ldx * nt + (size_t)L.ldv * nt);
  L.use_smem = bytes <= 200 * 1024;
  L.smem = L.use_smem ? bytes : 0;
  return L;
}
}  // namespace

// Whether the small-block path applies (l1f_pcp_f64 / l1f_svd_*_f64 / l1f_svt_f64 use it when it
// does): the Jacobi working set X (mt x nt) and V (nt x nt) must fit in shared memory — with them in
// global memory the dependent dot -> rotate chain of a round costs ~16 us (measured: a 200 x 200 seed
// took 0.68 s against 0.16 s through the Gram / syevd path), so larger blocks go there.
bool l1f_seed_small_applies(int64_t m, int64_t n) {
  const int64_t p = m < n ? m : n, q = m < n ? n : m;
  if (!(p >= 1 && p <= kSmallMaxDim && q <= (1 << 16) && p * q <= (1 << 22))) return false;
  const size_t bytes = sizeof(double) * ((size_t)(q | 1) * p + (size_t)(p | 1) * p);
  return bytes <= 200 * 1024;
}

static int g_last_sweeps = 0;  // diagnostics: Jacobi sweeps of the last small-block solve
extern "C" int l1f_diag_seed_small_sweeps(void) { return g_last_sweeps; }

int l1f_pcp_small(const double* M, int64_t ldm, int64_t m, int64_t n, double lam, double tol, double beta0,
                  double rho, double beta_max, int32_t max_iter, double* L, double* S, int32_t* iters_host,
                  double* residual_host, int32_t* rank_host, int32_t* converged_host, double* beta_final_host,
                  cudaStream_t st) {
  const int64_t count = m * n;
  const int64_t nt = m < n ? m : n, mt = m < n ? n : m;
  Work w;
  void* buf = nullptr;
  const size_t doubles = 2 * (size_t)count + (size_t)(mt + 1) * nt + m + n + (size_t)(nt + 1) * nt + 2 * (size_t)nt + 64;
  L1F_CUDA_TRY(cudaMallocAsync(&buf, doubles * sizeof(double) + (size_t)(nt + 2) * sizeof(int) + sizeof(Status), st));
  double* d = (double*)buf;
  w.Y = d; d += count;
  w.W = d; d += count;
  const XvLayout xl = xv_layout(mt, nt);
  w.X = d; d += (int64_t)xl.ldx * nt > m + n ? (int64_t)xl.ldx * nt : m + n;  // also the spectral-norm vectors
  w.V = d; d += (int64_t)xl.ldv * nt;
  w.sig = d; d += nt;
  w.fac = d; d += nt;
  d += 64;
  w.act = (int*)d;
  Status* sp = (Status*)(w.act + nt + (nt & 1));
  if (!xl.use_smem) {
    set_error("pcp (small): working set does not fit in shared memory");
    cudaFreeAsync(buf, st);
    return L1F_ERR_UNSUPPORTED;
  }
  if (xl.use_smem)
    cudaFuncSetAttribute(alm_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xl.smem);
  alm_small_kernel<<<1, NT, xl.smem, st>>>(M, ldm, (int)m, (int)n, lam, tol, beta0, rho, beta_max, max_iter, L, S, w,
                                           xl.ldx, xl.ldv, xl.use_smem, sp);
  cudaError_t e = cudaGetLastError();
  Status h{};
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, sp, sizeof(Status), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(buf, st);
  if (e != cudaSuccess) {
    set_error("pcp (small): %s", cudaGetErrorString(e));
    return L1F_ERR_CUDA;
  }
  if (h.err == L1F_ERR_SVD) {
    set_error("SVD failed on (%lld, %lld) matrix: Jacobi did not converge", (long long)m, (long long)n);
    return L1F_ERR_SVD;
  }
  if (h.err == L1F_ERR_DIVERGED) {
    set_error("non-finite residual at iteration %d (beta=%.3g)", h.iters, h.beta_final);
    return L1F_ERR_DIVERGED;
  }
  g_last_sweeps = h.sweeps_total;
  *iters_host = h.iters;
  *residual_host = h.residual;
  *rank_host = h.rank;
  *converged_host = h.converged;
  *beta_final_host = h.beta_final;
  return L1F_OK;
}

int l1f_svd_small(const double* W, int64_t m, int64_t n, int64_t ldw, double* U, double* sigma, double* V,
                  cudaStream_t st) {
  const int64_t nt = m < n ? m : n, mt = m < n ? n : m;
  void* buf = nullptr;
  const XvLayout xl = xv_layout(mt, nt);
  const size_t doubles = (size_t)xl.ldx * nt + (size_t)xl.ldv * nt + (size_t)nt + 16;
  L1F_CUDA_TRY(cudaMallocAsync(&buf, doubles * sizeof(double) + (size_t)nt * sizeof(int) + 2 * sizeof(Status), st));
  double* X = (double*)buf;
  double* Vw = X + (int64_t)xl.ldx * nt;
  double* s_tmp = Vw + (int64_t)xl.ldv * nt;
  int* order = (int*)(s_tmp + nt + 16);
  Status* sp = (Status*)(order + nt + (nt & 1) + 2);
  if (!xl.use_smem) {
    set_error("svd (small): working set does not fit in shared memory");
    cudaFreeAsync(buf, st);
    return L1F_ERR_UNSUPPORTED;
  }
  if (xl.use_smem)
    cudaFuncSetAttribute(svd_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xl.smem);
  svd_small_kernel<<<1, NT, xl.smem, st>>>(W, ldw, (int)m, (int)n, U, sigma, V, X, Vw, s_tmp, order, xl.ldx, xl.ldv,
                                           xl.use_smem, sp);
  cudaError_t e = cudaGetLastError();
  Status h{};
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, sp, sizeof(Status), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(buf, st);
  if (e != cudaSuccess) {
    set_error("svd (small): %s", cudaGetErrorString(e));
    return L1F_ERR_CUDA;
  }
  if (h.err == L1F_ERR_SVD) {
    set_error("SVD failed on (%lld, %lld) matrix: Jacobi did not converge", (long long)m, (long long)n);
    return L1F_ERR_SVD;
  }
  return L1F_OK;
}
