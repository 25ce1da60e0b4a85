// Seed PCP for small blocks, entirely on the device: one persistent CTA runs the whole inexact-ALM
// loop of solve_pcp (pcp_adm.py:90-140) with a hand-written singular value thresholding
// (matcore.py:73-105), and a second kernel factors the final seed L (recover_seed,
// l1filter.py:90-113 -> matcore.svd) by one-sided Jacobi.  No library call and no host round trip:
// the host reads one status record after the loop.  Used when the working set fits in shared memory
// (square blocks up to 113 x 113: every l1-filtering seed up to rank 11 — configs 1 and 4, the
// reference's test and golden sizes; see l1f_seed_small_applies).
//
// One ALM iteration (all in the CTA):
//   S = shrink((M - L) + Y/b, lam/b);  W = (M - S) + Y/b                  (pcp_adm.py:122-123)
//   SVT of W at eta = 1/b, two forms (L1F_OPT_SEED_SMALL_SVT):
//   * default, alm_gram_kernel: T (W or W^T, tall mt x nt) in shared memory, G = T^T T, Householder
//     tridiagonalisation of G in shared memory, the eigenvalues above eta^2 by Sturm multisection,
//     their vectors by inverse iteration + back-transformation; L = T Z diag(1 - eta/sigma) Z^T
//   * alm_small_kernel: X = T V (V warm-started from the previous iteration's right singular
//     vectors), one-sided Jacobi on the columns of X rotating V alongside, until every column pair
//     is orthogonal to eps * sqrt(mt): X = U diag(sigma), L = sum_{sigma_c > eta} x_c (1 - eta /
//     sigma_c) v_c^T  (= U (sigma - eta)_+ V^T)
//   R = (M - L) - S;  res = ||R||_F / ||M||_F;  Y += b R;  stop at res <= tol  (pcp_adm.py:124-135)
//   b = min(rho b, b_max)
// Reductions are fixed-order trees (deterministic).
#include "common.cuh"

#include <algorithm>
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

// ---------------------------------------------------------------------------------------------
// SVT through the Gram matrix, all in shared memory (default; L1F_OPT_SEED_SMALL_SVT = 1).
// Per ALM iteration the shrink pass writes T (tall orientation, column-major, stride ldt) straight
// into shared memory; G = T^T T (nt x nt, full symmetric, stride ldg) is reduced to tridiagonal form
// by Householder reflections in place (LAPACK dsytd2 'L' order, two barriers per column: every warp
// recomputes the reflector from the finished row, so no barrier is spent on it); the eigenvalues
// above eta^2 are bracketed by Sturm multisection (one warp each), their vectors found by inverse
// iteration on the tridiagonal (one thread each, factors in global scratch), re-orthogonalised by
// CGS2 inside clusters and refined to Rayleigh quotients, then back-transformed by the reflectors
// (one warp per vector, the vector in registers).  SVT: L = T Z diag(1 - eta / sigma) Z^T with
// sigma = sqrt(lambda) (matcore.py:96-105).  Squaring the spectrum costs relative accuracy only in
// singular values far below sigma_max, whose thresholded contribution is absolutely tiny.
constexpr int kGramMaxP = 128;
#ifdef L1F_SEED_PROF
#define SPROF_MARK(slot) do { __syncthreads(); if (threadIdx.x == 0) { long long _t = clock64(); prof[slot] += _t - tprev; tprev = _t; } } while (0)
#else
#define SPROF_MARK(slot) __syncthreads()
#endif  // nt <= 128: a vector of length nt is 4 registers per lane

__device__ __forceinline__ int sturm_count_below(const double* __restrict__ d, const double* __restrict__ e2, int p,
                                                 double x, double pivmin) {
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

// the same count with the division replaced by the hardware reciprocal estimate and one Newton step
// (relative error ~2^-46 per pivot: the count of a matrix perturbed far below the bisection's
// resolution); used by the multisection, the threshold count keeps the IEEE division
__device__ __forceinline__ int sturm_count_below_fast(const double* __restrict__ d, const double* __restrict__ e2,
                                                      int p, double x, double pivmin) {
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

// Householder tridiagonalisation of the symmetric G (p x p, row stride ldg) in shared memory.
// Outputs d, e (T's diagonal / off-diagonal), tau and the reflector scale: reflector i is v[i+1] = 1,
// v[c] = G[i][c] * hsc[i] for c > i + 1 (row i's tail is final once column i is reduced).
__device__ void gram_tridiag(double* G, int ldg, int p, double* d, double* e, double* tau_s, double* hsc,
                             double* sy) {
  // per column: warp 0 forms the reflector; y = tau G v with one thread per trailing row (a full
  // row dot, four accumulators: no shuffles); every warp forms K = -tau/2 y.v; the whole CTA
  // applies the rank-2 update.  Three barriers per column.
  __shared__ double scal[2];  // tau, scale
  __shared__ double dtp[kGramMaxP / 32];  // per-warp partials of y.v
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
#ifdef L1F_SEED_PROF
  long long tq[4] = {0, 0, 0, 0};
  long long tp0 = clock64();
#define TQ(k) do { if (threadIdx.x == 0) { long long _t = clock64(); tq[k] += _t - tp0; tp0 = _t; } } while (0)
#else
#define TQ(k) do {} while (0)
#endif
  for (int i = 0; i + 1 < p; ++i) {
    const int c0 = i + 1;
    const double* gi = G + (int64_t)i * ldg;
    if (warp == 0) {
      double s = 0.0;
      for (int c = c0 + 1 + lane; c < p; c += 32) s = fma(gi[c], gi[c], s);
      const double xnorm2 = warp_sum(s);
      if (lane == 0) {
        const double alpha = gi[c0];
        double tau = 0.0, beta = alpha, scale = 0.0;
        if (xnorm2 > 0.0) householder_scalars(alpha, xnorm2, beta, tau, scale);
        d[i] = G[(int64_t)i * ldg + i];
        e[i] = beta;
        tau_s[i] = tau;
        hsc[i] = scale;
        scal[0] = tau;
        scal[1] = scale;
      }
    }
    __syncthreads();
    TQ(0);
    const double tau = scal[0], scale = scal[1];
    if (tau == 0.0) continue;  // H = I (uniform)
    if (warp < kGramMaxP / 32) {  // rows live in threads 0 .. p - 1 (p <= 128: warps 0 - 3)
      const int r = threadIdx.x;
      double yv = 0.0;
      if (r >= c0 && r < p) {
        const double* gr = G + (int64_t)r * ldg;
        double a0 = gr[c0], a1 = 0.0, a2 = 0.0, a3 = 0.0;  // v[c0] = 1
        int c = c0 + 1;
        for (; c + 3 < p; c += 4) {
          a0 = fma(gr[c], gi[c] * scale, a0);
          a1 = fma(gr[c + 1], gi[c + 1] * scale, a1);
          a2 = fma(gr[c + 2], gi[c + 2] * scale, a2);
          a3 = fma(gr[c + 3], gi[c + 3] * scale, a3);
        }
        for (; c < p; ++c) a0 = fma(gr[c], gi[c] * scale, a0);
        const double y = tau * ((a0 + a1) + (a2 + a3));
        sy[r] = y;
        yv = y * (r == c0 ? 1.0 : gi[r] * scale);  // y_r v_r: this row's share of y.v
      }
      yv = warp_sum(yv);
      if (lane == 0) dtp[warp] = yv;
    }
    __syncthreads();
    TQ(1);
    // K = -tau/2 (y.v) from the four row warps' partials (fixed order)
    const double K = -0.5 * tau * ((dtp[0] + dtp[1]) + (dtp[2] + dtp[3]));
    TQ(2);
    // w = y - (tau/2)(y.v) v ; G -= v w^T + w v^T (trailing block, both triangles)
    for (int r = c0 + warp; r < p; r += NW) {
      const double vr = r == c0 ? 1.0 : gi[r] * scale;
      const double wr = fma(K, vr, sy[r]);
      double* gr = G + (int64_t)r * ldg;
      for (int c = c0 + lane; c < p; c += 32) {
        const double vc = c == c0 ? 1.0 : gi[c] * scale;
        gr[c] -= fma(vr, fma(K, vc, sy[c]), wr * vc);
      }
    }
    __syncthreads();
    TQ(3);
  }
#ifdef L1F_SEED_PROF
  if (threadIdx.x == 0 && p > 90 && blockIdx.x == 0)
    printf("  tridiag p=%d per column: reflector %lld matvec %lld dot %lld update %lld\n", p, tq[0] / (p - 1),
           tq[1] / (p - 1), tq[2] / (p - 1), tq[3] / (p - 1));
#endif
#undef TQ
  if (threadIdx.x == 0) d[p - 1] = G[(int64_t)(p - 1) * ldg + p - 1];
  __syncthreads();
}

struct GramWork {
  double* Y;    // p x p: eigenvectors of T, column j contiguous (length p)
  double* F;    // 6 p x p: inverse-iteration factors, entry i of eigenvalue j at [i * p + j]
  double* P;    // mt x p: T Z diag(fac)
};

// eigenpairs of the tridiagonal (d, e) with lambda > thr, descending: returns k (block-uniform);
// Y column j (global) holds the normalised vector, lam[j] its Rayleigh quotient
__device__ int tridiag_eig_above(const double* d, const double* e, double* e2, int p, double thr, double* lam,
                                 double* sdot, double* red, int* kbuf, double* bnd, GramWork gw, double* fs, int kcap,
                                 unsigned* swb) {
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  if (warp == 0) {  // Gershgorin bounds, pivmin, k = #(lambda > thr)
    double lo = 1e300, hi = -1e300, emax = 0.0;
    for (int j = lane; j < p; j += 32) {
      const double el = j > 0 ? fabs(e[j - 1]) : 0.0, er = j + 1 < p ? fabs(e[j]) : 0.0;
      lo = fmin(lo, d[j] - el - er);
      hi = fmax(hi, d[j] + el + er);
      if (j + 1 < p) {
        e2[j] = e[j] * e[j];
        emax = fmax(emax, e2[j]);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    }
    __syncwarp();
    if (lane == 0) {
      const double pivmin = DBL_MIN * fmax(1.0, emax);
      bnd[0] = thr;
      bnd[1] = hi;
      bnd[2] = pivmin;
      bnd[3] = fmax(fabs(hi), fabs(lo));
      *kbuf = thr >= hi ? 0 : p - sturm_count_below(d, e2, p, thr, pivmin);
    }
  }
  __syncthreads();
  const int k = *kbuf;
  if (k == 0) return 0;
  const double pivmin = bnd[2];
  // eigenvalue j (j-th largest) by multisection, one warp per eigenvalue
  for (int j = warp; j < k; j += NW) {
    const int idx = p - 1 - j;
    double lo = bnd[0], hi = bnd[1] * (1.0 + 1e-14) + fabs(bnd[1]) * 1e-14 + pivmin;
    for (int it = 0; it < 8; ++it) {
      const double x = lo + (hi - lo) * (double)(lane + 1) / 33.0;
      const int c = sturm_count_below_fast(d, e2, p, x, pivmin);
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
  __syncthreads();
  // inverse iteration on T - lam_j I (LU with partial pivoting, dgttrf / dgttrs), two solves, one
  // thread per eigenvalue.  Factors (multiplier, reciprocal pivot, two superdiagonals, right-hand
  // side) in shared memory for the first kcap eigenvalues (plane stride p * kcap, entry i of
  // eigenvalue j at [i * kcap + j]: a warp's accesses are consecutive), in global scratch beyond;
  // the row-interchange flags as bits.
  const double eps = 2.220446049250313e-16;
  const double tnorm = bnd[3] + 1.0e-300;
  const int nwd = (p + 31) / 32;
  for (int j = threadIdx.x; j < k; j += NT) {
    const double s = lam[j];
    const bool in_smem = j < kcap;
    const int ld = in_smem ? kcap : p;
    double* base = in_smem ? fs + j : gw.F + j;
    const size_t plane = (size_t)p * ld;
    double* __restrict__ dl = base;
    double* __restrict__ dinv = base + plane;
    double* __restrict__ du = base + 2 * plane;
    double* __restrict__ du2 = base + 3 * plane;
    double* __restrict__ bb = base + 4 * plane;
    unsigned* __restrict__ sb = swb + (size_t)j * nwd;
    const double clampv = eps * tnorm;
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
      const size_t o = (size_t)i * ld;
      if (fabs(di) >= fabs(sub)) {
        const double f = di != 0.0 ? sub * rcp_nr2(di) : 0.0;
        dl[o] = f; dinv[o] = inv_pivot(di); du[o] = ui; du2[o] = 0.0;
        di = dn - f * ui;
        ui = un;
      } else {
        const double f = di * rcp_nr2(sub);
        dl[o] = f; dinv[o] = inv_pivot(sub); du[o] = dn; du2[o] = un;
        bits |= 1u << (i & 31);
        di = ui - f * dn;
        ui = -f * un;
      }
      if ((i & 31) == 31) { sb[i >> 5] = bits; bits = 0; }
    }
    if (p >= 2 && ((p - 2) & 31) != 31) sb[(p - 2) >> 5] = bits;
    dinv[(size_t)(p - 1) * ld] = inv_pivot(di);
    for (int i = 0; i < p; ++i) {  // deterministic start vector in [0.75, 1.25)
      const unsigned h = ((unsigned)i * 2654435761u) ^ ((unsigned)(j + 1) * 2246822519u);
      bb[(size_t)i * ld] = 0.75 + 0.5 * (double)((h >> 8) & 0xffffu) / 65536.0;
    }
    for (int rep = 0; rep < 2; ++rep) {
      double prev = bb[0];
      for (int i = 0; i + 1 < p; ++i) {  // forward: L with the interchanges
        const size_t o = (size_t)i * ld;
        const double nx = bb[o + ld];
        const double f = dl[o];
        if (!((sb[i >> 5] >> (i & 31)) & 1u)) {
          bb[o] = prev;
          prev = fma(-f, prev, nx);
        } else {
          bb[o] = nx;
          prev = fma(-f, nx, prev);
        }
      }
      bb[(size_t)(p - 1) * ld] = prev;
      double x1 = prev * dinv[(size_t)(p - 1) * ld];  // back substitution with U
      double nrm = x1 * x1;
      bb[(size_t)(p - 1) * ld] = x1;
      double x2 = 0.0;
      if (p > 1) {
        const size_t o = (size_t)(p - 2) * ld;
        x2 = x1;
        x1 = (bb[o] - du[o] * x2) * dinv[o];
        bb[o] = x1;
        nrm = fma(x1, x1, nrm);
      }
      for (int i = p - 3; i >= 0; --i) {
        const size_t o = (size_t)i * ld;
        const double x0 = (bb[o] - du[o] * x1 - du2[o] * x2) * dinv[o];
        bb[o] = x0;
        nrm = fma(x0, x0, nrm);
        x2 = x1;
        x1 = x0;
      }
      const double inv = nrm > 0.0 ? 1.0 / sqrt(nrm) : 0.0;
      if (rep == 0) {
        for (int i = 0; i < p; ++i) bb[(size_t)i * ld] *= inv;
      } else {
        double* y = gw.Y + (size_t)j * p;
        for (int i = 0; i < p; ++i) y[i] = bb[(size_t)i * ld] * inv;
      }
    }
  }
  __syncthreads();
  // CGS2 inside clusters (consecutive eigenvalues closer than 1e-4 ||T||), normalisation and the
  // Rayleigh quotient lam_j = y_j^T T y_j
  const double gap_tol = 1e-4 * bnd[3];
  int cstart = 0;
  for (int j = 0; j < k; ++j) {
    if (j > 0 && !(fabs(lam[j - 1] - lam[j]) < gap_tol)) cstart = j;
    double* yj = gw.Y + (size_t)j * p;
    for (int pass = 0; pass < 2 && cstart < j; ++pass) {
      for (int i = cstart + warp; i < j; i += NW) {
        const double* yi = gw.Y + (size_t)i * p;
        double s = 0.0;
        for (int r = lane; r < p; r += 32) s = fma(yi[r], yj[r], s);
        s = warp_sum(s);
        if (lane == 0) sdot[i] = s;
      }
      __syncthreads();
      for (int r = threadIdx.x; r < p; r += NT) {
        double v = yj[r];
        for (int i = cstart; i < j; ++i) v = fma(-sdot[i], gw.Y[(size_t)i * p + r], v);
        yj[r] = v;
      }
      __syncthreads();
    }
  }
  // normalisation and Rayleigh quotients, one warp per vector
  for (int j = warp; j < k; j += NW) {
    double* yj = gw.Y + (size_t)j * p;
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
  __syncthreads();
  return k;
}

__global__ void __launch_bounds__(NT, 1)
alm_gram_kernel(const double* __restrict__ M, int64_t ldm, int m, int n, double lam, double tol, double beta0,
                double rho, double beta_max, int max_iter, double* __restrict__ L, double* __restrict__ S,
                Work w, GramWork gw, int ldt, int ldg, int kcap, Status* st) {
  extern __shared__ double smem_g[];
  __shared__ double red[NW + 1];
  __shared__ double bnd[4];
  __shared__ int kbuf, nact;
  Shape sh;
  sh.m = m; sh.n = n; sh.tr = m < n;
  sh.mt = sh.tr ? n : m;
  sh.nt = sh.tr ? m : n;
  const int p = sh.nt, mt = sh.mt;
  double* T = smem_g;                       // column-major mt x p, stride ldt
  double* G = T + (size_t)ldt * p;          // p x p, stride ldg (then Z: row q = vector q)
  double* d = G + (size_t)ldg * p;
  double* e = d + p;
  double* e2 = e + p;
  double* tau_s = e2 + p;
  double* hsc = tau_s + p;
  double* sy = hsc + p;
  double* lamv = sy + p;
  double* fac = lamv + p;
  double* sdot = fac + p;
  double* fs = sdot + p;                    // inverse-iteration factors of kcap eigenvalues (5 p each)
  unsigned* swb = (unsigned*)(fs + 5 * (size_t)p * kcap);  // interchange bits, p x ceil(p / 32)
  const int64_t count = (int64_t)m * n;
  const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
  double acc = 0.0;
  for (int64_t e0 = tid; e0 < count; e0 += NT) {
    const double v = M[(e0 / n) * ldm + e0 % n];
    acc = fma(v, v, acc);
  }
  const double norm_m = sqrt(block_sum(acc, red));
  for (int64_t e0 = tid; e0 < count; e0 += NT) {
    L[e0] = 0.0;
    S[e0] = 0.0;
    w.Y[e0] = 0.0;
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
  if (!(beta0 > 0.0)) {  // spectral_norm_estimate (pcp_adm.py:69-87), vectors in w.X
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
  double residual = 1.0;
  int rank = 0, it = 0, converged = 0;
#ifdef L1F_SEED_PROF
  long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tprev = clock64();
#endif
  for (it = 1; it <= max_iter; ++it) {
    const double thr = lam / beta, eta = 1.0 / beta;
    // S = shrink((M - L) + Y/b, lam/b); T <- W = (M - S) + Y/b in the tall orientation
    for (int64_t e0 = tid; e0 < count; e0 += NT) {
      const int i = (int)(e0 / n), j = (int)(e0 - (int64_t)i * n);
      const double mv = M[(int64_t)i * ldm + j];
      const double yb = w.Y[e0] / beta;
      const double s = shrink((mv - L[e0]) + yb, thr);
      S[e0] = s;
      const int ti = sh.tr ? j : i, tj = sh.tr ? i : j;
      T[(int64_t)tj * ldt + ti] = (mv - s) + yb;
    }
    __syncthreads();
    // G = T^T T (lower triangle computed, mirrored)
    for (int x = tid; x < p * p; x += NT) {
      const int a = x / p, b = x - a * p;
      if (b > a) continue;
      const double* ta = T + (int64_t)a * ldt;
      const double* tb = T + (int64_t)b * ldt;
      double g = 0.0;
      for (int i = 0; i < mt; ++i) g = fma(ta[i], tb[i], g);
      G[(int64_t)a * ldg + b] = g;
      G[(int64_t)b * ldg + a] = g;
    }
    SPROF_MARK(0);
    gram_tridiag(G, ldg, p, d, e, tau_s, hsc, sy);
    SPROF_MARK(1);
    const int kk = tridiag_eig_above(d, e, e2, p, eta * eta, lamv, sdot, red, &kbuf, bnd, gw, fs, kcap, swb);
    SPROF_MARK(2);
    // retained: the leading run with sigma - eta > 0 (lam descending)
    if (tid == 0) {
      int k = 0;
      for (int j = 0; j < kk; ++j) {
        const double sg = lamv[j] > 0.0 ? sqrt(lamv[j]) : 0.0;
        if (!(sg > 0.0) || !(sg - eta > 0.0)) break;
        fac[k++] = 1.0 - eta / sg;
      }
      nact = k;
    }
    __syncthreads();
    rank = nact;
    // back-transformation z_j = H_0 ... H_{p-2} y_j, one warp per vector in registers
    for (int j = warp; j < rank; j += NW) {
      double* yj = gw.Y + (size_t)j * p;
      double yv[kGramMaxP / 32];
#pragma unroll
      for (int u = 0; u < kGramMaxP / 32; ++u) {
        const int c = lane + 32 * u;
        yv[u] = c < p ? yj[c] : 0.0;
      }
      for (int i = p - 2; i >= 0; --i) {
        const double t = tau_s[i];
        if (t == 0.0) continue;
        const double sc = hsc[i];
        const double* gi = G + (int64_t)i * ldg;
        double s = 0.0;
#pragma unroll
        for (int u = 0; u < kGramMaxP / 32; ++u) {
          const int c = lane + 32 * u;
          if (c > i && c < p) s = fma(c == i + 1 ? 1.0 : gi[c] * sc, yv[u], s);
        }
        s = warp_sum(s) * t;
#pragma unroll
        for (int u = 0; u < kGramMaxP / 32; ++u) {
          const int c = lane + 32 * u;
          if (c > i && c < p) yv[u] = fma(-s, c == i + 1 ? 1.0 : gi[c] * sc, yv[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < kGramMaxP / 32; ++u) {
        const int c = lane + 32 * u;
        if (c < p) yj[c] = yv[u];
      }
    }
    SPROF_MARK(3);
    // Z into G's space (row q = vector q); P = T Z diag(fac) (mt x rank, global)
    for (int x = tid; x < rank * p; x += NT) {
      const int q = x / p, a = x - q * p;
      G[(int64_t)q * ldg + a] = gw.Y[(size_t)q * p + a];
    }
    __syncthreads();
    for (int x = tid; x < mt * rank; x += NT) {
      const int q = x / mt, i = x - q * mt;
      const double* zq = G + (int64_t)q * ldg;
      double a = 0.0;
      for (int c = 0; c < p; ++c) a = fma(T[(int64_t)c * ldt + i], zq[c], a);
      gw.P[(size_t)i * p + q] = a * fac[q];
    }
    SPROF_MARK(4);
    // L = P Z^T ; R = (M - L) - S ; Y += b R ; ||R||^2
    acc = 0.0;
    for (int64_t e0 = tid; e0 < count; e0 += NT) {
      const int i = (int)(e0 / n), j = (int)(e0 - (int64_t)i * n);
      const int ti = sh.tr ? j : i, tj = sh.tr ? i : j;
      const double* pr = gw.P + (size_t)ti * p;
      double l = 0.0;
      for (int q = 0; q < rank; ++q) l = fma(pr[q], G[(int64_t)q * ldg + tj], l);
      L[e0] = l;
      const double r = (M[(int64_t)i * ldm + j] - l) - S[e0];
      acc = fma(r, r, acc);
      w.Y[e0] = w.Y[e0] + beta * r;
    }
    residual = sqrt(block_sum(acc, red)) / norm_m;
    SPROF_MARK(5);
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
    st->beta_final = beta; st->sweeps_total = 0;
#ifdef L1F_SEED_PROF
    printf("gram-alm %dx%d it %d: shrink+gram %lld tridiag %lld eig %lld back %lld P %lld Lpass %lld (cycles/iter)\n", m, n, it,
           prof[0] / it, prof[1] / it, prof[2] / it, prof[3] / it, prof[4] / it, prof[5] / it);
#endif
  }
  (void)lane;
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
  void* gbuf = nullptr;
  if (option(L1F_OPT_SEED_SMALL_SVT) != 0 && nt <= kGramMaxP) {
    // Gram / tridiagonal SVT: T (mt x nt) and G (nt x nt) in shared memory plus 9 nt-vectors
    const int ldt = (int)(mt | 1), ldg = (int)(nt | 1);
    const size_t base = sizeof(double) * ((size_t)ldt * nt + (size_t)ldg * nt + 9 * (size_t)nt) +
                        sizeof(unsigned) * (size_t)nt * ((nt + 31) / 32) + 16;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const size_t avail = (size_t)optin > base + 2048 ? (size_t)optin - base - 2048 : 0;
    const int kcap = (int)std::min<size_t>((size_t)nt, avail / (sizeof(double) * 5 * (size_t)nt));
    const size_t smem = base + sizeof(double) * 5 * (size_t)nt * kcap;
    GramWork gw;
    cudaError_t ea = cudaMallocAsync(&gbuf, sizeof(double) * ((size_t)nt * nt * 7 + (size_t)mt * nt + 16), st);
    if (ea != cudaSuccess) {
      cudaFreeAsync(buf, st);
      set_error("pcp (small): %s", cudaGetErrorString(ea));
      return L1F_ERR_CUDA;
    }
    gw.Y = (double*)gbuf;
    gw.F = gw.Y + (size_t)nt * nt;
    gw.P = gw.F + 6 * (size_t)nt * nt;
    cudaFuncSetAttribute(alm_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    alm_gram_kernel<<<1, NT, smem, st>>>(M, ldm, (int)m, (int)n, lam, tol, beta0, rho, beta_max, max_iter, L, S, w,
                                         gw, ldt, ldg, kcap, sp);
  } else {
    cudaFuncSetAttribute(alm_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xl.smem);
    alm_small_kernel<<<1, NT, xl.smem, st>>>(M, ldm, (int)m, (int)n, lam, tol, beta0, rho, beta_max, max_iter, L, S,
                                             w, xl.ldx, xl.ldv, xl.use_smem, sp);
  }
  cudaError_t e = cudaGetLastError();
  Status h{};
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, sp, sizeof(Status), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(buf, st);
  if (gbuf) cudaFreeAsync(gbuf, st);
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
