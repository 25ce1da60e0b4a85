// FP64 seed stage of l1 filtering: the small PCP of recover_seed (l1filter.py:90-113).
//
//   solve_pcp          pcp_adm.py:90-140   (inexact ALM: shrink, SVT, residual, dual/penalty)
//   spectral_norm_est. pcp_adm.py:69-87    (25-step power iteration from the all-ones vector)
//   svd / svt_with_rank matcore.py:73-105  (thin SVD; singular value thresholding)
//
// Blocks whose working set fits in shared memory (square up to 113 x 113: every seed up to rank 11,
// configs 1 and 4, the reference's test sizes) never reach this file's library path:
// l1f_pcp_f64 / l1f_svd_*_f64 / l1f_svt_f64 hand them to the one-CTA kernels of seed_small.cu (no
// library call, no host round trip).  Larger blocks (the rank-50 to rank-200 seeds of configs 2, 3
// and 5, ranks 12-25, the full-matrix ADM) run the ALM loop here: the SVT through the Gram matrix
// (cuBLAS dsyrk / dgemm for the products) and its eigenpairs above the threshold from the
// hand-written solver of eig_sym.cu (default wherever its shared-memory-resident tridiagonalisation
// applies, p <= 2000; cuSOLVER syevd beyond, or on request through L1F_OPT_SEED_EIG); the fused
// shrink / residual / dual kernels and the deterministic reductions are ours.  gesvd serves only the
// public full SVD of large matrices (l1f_svd_f64).  The seed runs in FP64: its factors
// must pass the reference's orthonormality check (l1reg.py:48-56, 1e-8) before they are cast to
// FP32 for the filter.
#include "common.cuh"

#include <cublas_v2.h>
#include <cusolverDn.h>

#include <cmath>
#include <cstdlib>
#include <vector>

bool l1f_seed_small_applies(int64_t m, int64_t n);
int l1f_pcp_small(const double* M, int64_t ldm, int64_t m, int64_t n, double lam, double tol, double beta0,
                  double rho, double beta_max, int32_t max_iter, double* L, double* S, int32_t* iters_host,
                  double* residual_host, int32_t* rank_host, int32_t* converged_host, double* beta_final_host,
                  cudaStream_t st);
int l1f_svd_small(const double* W, int64_t m, int64_t n, int64_t ldw, double* U, double* sigma, double* V,
                  cudaStream_t st);
int l1f_eig_sym_above(double* G, int p, double thr_abs, double thr_rel, double* lam, double* Z, int* k_host,
                      cudaStream_t st);
bool l1f_eig_dsm_applies(int p);

namespace l1f {
namespace seed {

struct Handles {
  cusolverDnHandle_t sol = nullptr;
  cublasHandle_t blas = nullptr;
};

// cuBLAS on every call; the cuSOLVER handle only when a cuSOLVER routine runs (its creation loads
// the library's modules, ~0.1 s, which the default seed path never needs)
static int handles(cudaStream_t st, Handles*& out) {
  // one set per device (a cuBLAS / cuSOLVER handle belongs to the device current at its creation)
  static thread_local Handles hs[64];
  int dev = 0;
  L1F_CUDA_TRY(cudaGetDevice(&dev));
  Handles& h = hs[dev & 63];
  if (!h.blas) {
    if (cublasCreate(&h.blas) != CUBLAS_STATUS_SUCCESS) {
      set_error("cublasCreate failed");
      return L1F_ERR_CUDA;
    }
  }
  cublasSetStream(h.blas, st);
  if (h.sol) cusolverDnSetStream(h.sol, st);
  out = &h;
  return L1F_OK;
}

static cusolverDnHandle_t solver(Handles* h, cudaStream_t st) {
  if (!h->sol && cusolverDnCreate(&h->sol) != CUSOLVER_STATUS_SUCCESS) {
    h->sol = nullptr;
    set_error("cusolverDnCreate failed");
    return nullptr;
  }
  cusolverDnSetStream(h->sol, st);
  return h->sol;
}
#define L1F_SOLVER(h, st)                                  \
  cusolverDnHandle_t sol_ = solver((h), (st));             \
  if (!sol_) return L1F_ERR_CUDA

struct Buf {
  void* p = nullptr;
  cudaStream_t s;
  explicit Buf(cudaStream_t st) : s(st) {}
  cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, bytes ? bytes : 16, s); }
  double* d() const { return (double*)p; }
  ~Buf() { if (p) cudaFreeAsync(p, s); }
};

// S = shrink((M - L) + Y/b, lam/b) ; W = (M - S) + Y/b        (pcp_adm.py:122-123)
__global__ void pcp_shrink_kernel(const double* __restrict__ M, const double* __restrict__ L,
                                  const double* __restrict__ Y, double* __restrict__ S, double* __restrict__ W,
                                  int64_t count, double beta, double thr) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    const double yb = Y[e] / beta;
    const double s = shrink((M[e] - L[e]) + yb, thr);
    S[e] = s;
    W[e] = (M[e] - s) + yb;
  }
}

// R = (M - L) - S ; partial sum R^2 ; Y += b R                 (pcp_adm.py:124-130)
__global__ void pcp_residual_kernel(const double* __restrict__ M, const double* __restrict__ L,
                                    const double* __restrict__ S, double* __restrict__ Y, int64_t count,
                                    double beta, double* __restrict__ part) {
  double acc = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    const double r = (M[e] - L[e]) - S[e];
    acc += r * r;
    Y[e] = Y[e] + beta * r;
  }
  __shared__ double red[32];
  acc = warp_sum(acc);
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x / 32); ++i) t += red[i];
    part[blockIdx.x] = t;
  }
}

__global__ void sum_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += part[i];
    *out = t;
  }
}

// sum of squares, deterministic
__global__ void sumsq_partial_kernel(const double* __restrict__ X, int64_t count, double* __restrict__ part) {
  double acc = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
    acc += X[e] * X[e];
  __shared__ double red[32];
  acc = warp_sum(acc);
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x / 32); ++i) t += red[i];
    part[blockIdx.x] = t;
  }
}

// U[:, t] *= w[t] for t < k (row-major m x ld)
__global__ void scale_cols_kernel(double* __restrict__ U, int64_t m, int64_t ld, int k, const double* __restrict__ w) {
  const int64_t total = m * (int64_t)k;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / k;
    const int t = (int)(e - i * k);
    U[i * ld + t] *= w[t];
  }
}

static int reduce_blocks() { return num_sms() * 2; }

static int sumsq(const double* X, int64_t count, double* part, double* out_dev, double* out_host, cudaStream_t st) {
  const int g = reduce_blocks();
  sumsq_partial_kernel<<<g, 256, 0, st>>>(X, count, part);
  L1F_CHECK_LAUNCH();
  sum_kernel<<<1, 32, 0, st>>>(part, g, out_dev);
  L1F_CHECK_LAUNCH();
  L1F_CUDA_TRY(cudaMemcpyAsync(out_host, out_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
  L1F_CUDA_TRY(cudaStreamSynchronize(st));
  return L1F_OK;
}

// Thin SVD of a row-major m x n matrix.  Row-major W is column-major W^T; cuSOLVER's gesvd
// needs rows >= cols, so the n >= m case factors W^T in place and the n < m case factors
// an explicit column-major copy of W.
static int svd_rowmajor(Handles* h, const double* W, int64_t m, int64_t n, int64_t ldw, double* U, double* sig,
                        double* V, cudaStream_t st) {
  const int64_t p = m < n ? m : n;
  const bool wide = n >= m;  // factor A = W^T (n x m, col-major)
  const int R = (int)(wide ? n : m), C = (int)(wide ? m : n);
  Buf a(st), ucm(st), vtcm(st), work(st), info(st);
  L1F_CUDA_TRY(a.alloc(sizeof(double) * (size_t)R * C));
  // column-major copy for gesvd via our gather kernel (row-major W is col-major W^T)
  int rc = wide ? l1f_gather(L1F_F64, W, ldw, nullptr, m, nullptr, n, L1F_F64, a.d(), n, 0, st)
                : l1f_gather(L1F_F64, W, ldw, nullptr, m, nullptr, n, L1F_F64, a.d(), m, 1, st);
  if (rc) return rc;
  L1F_CUDA_TRY(ucm.alloc(sizeof(double) * (size_t)R * p));
  L1F_CUDA_TRY(vtcm.alloc(sizeof(double) * (size_t)p * C));
  int lwork = 0;
  L1F_SOLVER(h, st);
  if (cusolverDnDgesvd_bufferSize(sol_, R, C, &lwork) != CUSOLVER_STATUS_SUCCESS) {
    set_error("gesvd_bufferSize failed");
    return L1F_ERR_CUDA;
  }
  L1F_CUDA_TRY(work.alloc(sizeof(double) * (size_t)(lwork > 0 ? lwork : 1)));
  L1F_CUDA_TRY(info.alloc(sizeof(int)));
  cusolverStatus_t cs = cusolverDnDgesvd(sol_, 'S', 'S', R, C, a.d(), R, sig, ucm.d(), R, vtcm.d(), (int)p,
                                         work.d(), lwork, nullptr, (int*)info.p);
  if (cs != CUSOLVER_STATUS_SUCCESS) {
    set_error("cusolverDnDgesvd failed with status %d", (int)cs);
    return L1F_ERR_SVD;
  }
  int info_h = 0;
  L1F_CUDA_TRY(cudaMemcpyAsync(&info_h, info.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  L1F_CUDA_TRY(cudaStreamSynchronize(st));
  if (info_h != 0) {
    set_error("SVD failed on (%lld, %lld) matrix: gesvd info %d", (long long)m, (long long)n, info_h);
    return L1F_ERR_SVD;
  }
  if (wide) {
    // left vectors of W^T are V (n x p col-major == p x n row-major); VT (p x m col-major)
    // is U as an m x p row-major matrix
    L1F_CUDA_TRY(cudaMemcpyAsync(U, vtcm.p, sizeof(double) * (size_t)p * C, cudaMemcpyDeviceToDevice, st));
    rc = l1f_gather(L1F_F64, ucm.d(), R, nullptr, p, nullptr, R, L1F_F64, V, p, 1, st);
  } else {
    rc = l1f_gather(L1F_F64, ucm.d(), R, nullptr, p, nullptr, R, L1F_F64, U, p, 1, st);
    if (rc) return rc;
    L1F_CUDA_TRY(cudaMemcpyAsync(V, vtcm.p, sizeof(double) * (size_t)p * C, cudaMemcpyDeviceToDevice, st));
  }
  if (rc) return rc;
  L1F_CHECK_LAUNCH();
  return L1F_OK;
}

// out = U diag(max(sig - eta, 0)) V^T for the leading k with sig > eta  (matcore.py:96-105)
static int svt_into(Handles* h, const double* W, int64_t m, int64_t n, double eta, double* out, int* rank,
                    cudaStream_t st) {
  const int64_t p = m < n ? m : n;
  Buf u(st), v(st), sg(st);
  L1F_CUDA_TRY(u.alloc(sizeof(double) * (size_t)m * p));
  L1F_CUDA_TRY(v.alloc(sizeof(double) * (size_t)n * p));
  L1F_CUDA_TRY(sg.alloc(sizeof(double) * (size_t)p));
  int rc = l1f_seed_small_applies(m, n) ? l1f_svd_small(W, m, n, n, u.d(), sg.d(), v.d(), st)
                                       : svd_rowmajor(h, W, m, n, n, u.d(), sg.d(), v.d(), st);
  if (rc) return rc;
  std::vector<double> sh((size_t)p);
  L1F_CUDA_TRY(cudaMemcpyAsync(sh.data(), sg.p, sizeof(double) * (size_t)p, cudaMemcpyDeviceToHost, st));
  L1F_CUDA_TRY(cudaStreamSynchronize(st));
  // svd(w, rank_tol=0) keeps sigma > 0; then s = sigma - eta, k = #(s > 0)
  int k = 0;
  for (int64_t t = 0; t < p; ++t) {
    if (!(sh[(size_t)t] > 0.0)) break;
    const double sv = sh[(size_t)t] - eta;
    if (sv > 0.0) { sh[(size_t)t] = sv; ++k; } else break;
  }
  *rank = k;
  if (k == 0) {
    L1F_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double) * (size_t)m * n, st));
    return L1F_OK;
  }
  L1F_CUDA_TRY(cudaMemcpyAsync(sg.p, sh.data(), sizeof(double) * (size_t)k, cudaMemcpyHostToDevice, st));
  scale_cols_kernel<<<num_sms() * 4, 256, 0, st>>>(u.d(), m, p, k, sg.d());
  L1F_CHECK_LAUNCH();
  rc = l1f_gemm_nt(L1F_F64, m, n, k, 1.0, u.p, p, v.p, p, 0.0, out, n, st);
  if (rc) return rc;
  // keep the host vector alive until the H2D copy has been consumed
  L1F_CUDA_TRY(cudaStreamSynchronize(st));
  return L1F_OK;
}

// SVT through the eigendecomposition of the smaller Gram matrix (used inside the ALM loop):
// W^T W = V diag(sigma^2) V^T (or W W^T = U diag(sigma^2) U^T when m < n), then
// out = W V_k diag(1 - eta/sigma_k) V_k^T.  Squaring the spectrum costs relative accuracy only in
// singular values far below sigma_max, whose SVT contribution (sigma - eta) is absolutely tiny, so
// the thresholded matrix matches the SVD form to ~eps * sigma_max per entry.  The seed's final
// rank-revealing factorisation (engine.recover_seed_device) takes the Gram route too (svd_gram) when
// its rank cut is >= 1e-6 of sigma_max, which every kept triplet clears by orders of magnitude; a
// smaller rank_tol takes the SVD (svd_rowmajor).
__global__ void scale_rows_cm_kernel(double* __restrict__ T, int64_t rows, int64_t cols, int64_t ld,
                                     const double* __restrict__ c) {
  // column-major T (rows x cols): row j scaled by c[j]
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = e / rows, j = e - col * rows;
    T[col * ld + j] *= c[j];
  }
}
__global__ void scale_cols_cm_kernel(double* __restrict__ T, int64_t rows, int64_t cols, int64_t ld,
                                     const double* __restrict__ c) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = e / rows, i = e - col * rows;
    T[col * ld + i] *= c[col];
  }
}

// the Gram eigensolver: hand-written (eig_sym.cu) or cuSOLVER syevd (L1F_OPT_SEED_EIG: 2 auto =
// hand-written wherever its shared-memory-resident tridiagonalisation applies, p <= 2000)
static bool hand_eig(int p) {
  const int64_t mode = option(L1F_OPT_SEED_EIG);
  return mode == 0 || (mode == 2 && l1f_eig_dsm_applies(p));
}

static int svt_gram(Handles* h, const double* W, int64_t m, int64_t n, double eta, double* out, int* rank,
                    cudaStream_t st, bool force_lib = false) {
  const bool right = n <= m;         // Gram of the smaller side
  const int p = (int)(right ? n : m), q = (int)(right ? m : n);
  // row-major W (m x n) == column-major X = W^T (n x m, ld n)
  Buf g(st), ev(st), work(st), info(st), t(st), cbuf(st);
  L1F_CUDA_TRY(g.alloc(sizeof(double) * (size_t)p * p));
  L1F_CUDA_TRY(ev.alloc(sizeof(double) * (size_t)p));
  const double one = 1.0, zero = 0.0;
  cublasSetPointerMode(h->blas, CUBLAS_POINTER_MODE_HOST);
  if (right)  // W^T W = X X^T
    cublasDsyrk(h->blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, p, q, &one, W, (int)n, &zero, g.d(), p);
  else        // W W^T = X^T X
    cublasDsyrk(h->blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, p, q, &one, W, (int)n, &zero, g.d(), p);
  if (!force_lib && hand_eig(p)) {
    // hand-written eigensolver (eig_sym.cu): only the eigenpairs with lambda > eta^2, descending
    Buf z(st);
    L1F_CUDA_TRY(z.alloc(sizeof(double) * (size_t)p * p));
    int kk = 0;
    int rc = l1f_eig_sym_above(g.d(), p, eta * eta, 0.0, ev.d(), z.d(), &kk, st);
    if (rc == L1F_ERR_UNSUPPORTED) return svt_gram(h, W, m, n, eta, out, rank, st, true);
    if (rc) return rc;
    std::vector<double> lam((size_t)(kk > 0 ? kk : 1));
    if (kk > 0) L1F_CUDA_TRY(cudaMemcpyAsync(lam.data(), ev.p, sizeof(double) * (size_t)kk, cudaMemcpyDeviceToHost, st));
    L1F_CUDA_TRY(cudaStreamSynchronize(st));
    int k = 0;
    std::vector<double> c;
    for (int j = 0; j < kk; ++j) {
      const double sg = lam[(size_t)j] > 0.0 ? std::sqrt(lam[(size_t)j]) : 0.0;
      if (!(sg > 0.0) || !(sg - eta > 0.0)) break;
      c.push_back(1.0 - eta / sg);
      ++k;
    }
    *rank = k;
    if (k == 0) {
      L1F_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double) * (size_t)m * n, st));
      return L1F_OK;
    }
    L1F_CUDA_TRY(cbuf.alloc(sizeof(double) * (size_t)k));
    L1F_CUDA_TRY(cudaMemcpyAsync(cbuf.p, c.data(), sizeof(double) * (size_t)k, cudaMemcpyHostToDevice, st));
    L1F_CUDA_TRY(t.alloc(sizeof(double) * (size_t)k * q));
    const double* Vk = z.d();  // column-major p x k, descending
    if (right) {
      cublasDgemm(h->blas, CUBLAS_OP_T, CUBLAS_OP_N, k, (int)m, (int)n, &one, Vk, p, W, (int)n, &zero, t.d(), k);
      scale_rows_cm_kernel<<<num_sms() * 4, 256, 0, st>>>(t.d(), k, m, k, cbuf.d());
      cublasDgemm(h->blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)n, (int)m, k, &one, Vk, p, t.d(), k, &zero, out, (int)n);
    } else {
      cublasDgemm(h->blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)n, k, (int)m, &one, W, (int)n, Vk, p, &zero, t.d(), (int)n);
      scale_cols_cm_kernel<<<num_sms() * 4, 256, 0, st>>>(t.d(), n, k, n, cbuf.d());
      cublasDgemm(h->blas, CUBLAS_OP_N, CUBLAS_OP_T, (int)n, (int)m, k, &one, t.d(), (int)n, Vk, p, &zero, out, (int)n);
    }
    L1F_CHECK_LAUNCH();
    L1F_CUDA_TRY(cudaStreamSynchronize(st));  // keep the host vector alive until consumed
    return L1F_OK;
  }
  int lwork = 0;
  L1F_SOLVER(h, st);
  if (cusolverDnDsyevd_bufferSize(sol_, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, p, g.d(), p, ev.d(),
                                  &lwork) != CUSOLVER_STATUS_SUCCESS) {
    set_error("syevd_bufferSize failed");
    return L1F_ERR_CUDA;
  }
  L1F_CUDA_TRY(work.alloc(sizeof(double) * (size_t)(lwork > 0 ? lwork : 1)));
  L1F_CUDA_TRY(info.alloc(sizeof(int)));
  if (cusolverDnDsyevd(sol_, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, p, g.d(), p, ev.d(), work.d(), lwork,
                       (int*)info.p) != CUSOLVER_STATUS_SUCCESS) {
    set_error("cusolverDnDsyevd failed");
    return L1F_ERR_SVD;
  }
  std::vector<double> lam((size_t)p);
  int info_h = 0;
  L1F_CUDA_TRY(cudaMemcpyAsync(lam.data(), ev.p, sizeof(double) * (size_t)p, cudaMemcpyDeviceToHost, st));
  L1F_CUDA_TRY(cudaMemcpyAsync(&info_h, info.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  L1F_CUDA_TRY(cudaStreamSynchronize(st));
  if (info_h != 0) {
    set_error("eigendecomposition failed on (%lld, %lld) matrix: syevd info %d", (long long)m, (long long)n, info_h);
    return L1F_ERR_SVD;
  }
  // eigenvalues ascending: the k largest with sigma > eta occupy the last k columns
  int k = 0;
  std::vector<double> c;
  for (int j = p - 1; j >= 0; --j) {
    const double sg = lam[(size_t)j] > 0.0 ? std::sqrt(lam[(size_t)j]) : 0.0;
    if (!(sg > 0.0) || !(sg - eta > 0.0)) break;
    ++k;
  }
  *rank = k;
  if (k == 0) {
    L1F_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double) * (size_t)m * n, st));
    return L1F_OK;
  }
  c.resize((size_t)k);
  for (int i = 0; i < k; ++i) {  // columns p-k .. p-1 in ascending order
    const double sg = std::sqrt(lam[(size_t)(p - k + i)]);
    c[(size_t)i] = 1.0 - eta / sg;
  }
  L1F_CUDA_TRY(cbuf.alloc(sizeof(double) * (size_t)k));
  L1F_CUDA_TRY(cudaMemcpyAsync(cbuf.p, c.data(), sizeof(double) * (size_t)k, cudaMemcpyHostToDevice, st));
  const double* Vk = g.d() + (size_t)(p - k) * p;  // column-major p x k block of eigenvectors
  L1F_CUDA_TRY(t.alloc(sizeof(double) * (size_t)k * q));
  if (right) {
    // Tt (k x m) = Vk^T X ; scale row j by c_j ; out^T (n x m) = Vk Tt
    cublasDgemm(h->blas, CUBLAS_OP_T, CUBLAS_OP_N, k, (int)m, (int)n, &one, Vk, p, W, (int)n, &zero, t.d(), k);
    scale_rows_cm_kernel<<<num_sms() * 4, 256, 0, st>>>(t.d(), k, m, k, cbuf.d());
    cublasDgemm(h->blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)n, (int)m, k, &one, Vk, p, t.d(), k, &zero, out, (int)n);
  } else {
    // T (n x k) = X Uk ; scale column j by c_j ; out^T (n x m) = T Uk^T
    cublasDgemm(h->blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)n, k, (int)m, &one, W, (int)n, Vk, p, &zero, t.d(), (int)n);
    scale_cols_cm_kernel<<<num_sms() * 4, 256, 0, st>>>(t.d(), n, k, n, cbuf.d());
    cublasDgemm(h->blas, CUBLAS_OP_N, CUBLAS_OP_T, (int)n, (int)m, k, &one, t.d(), (int)n, Vk, p, &zero, out, (int)n);
  }
  L1F_CHECK_LAUNCH();
  L1F_CUDA_TRY(cudaStreamSynchronize(st));  // keep the host vector alive until consumed
  return L1F_OK;
}

// ALM-loop SVT for blocks beyond the small-block kernel (seed_small.cu): Gram/eigen form
static int svt_loop(Handles* h, const double* W, int64_t m, int64_t n, double eta, double* out, int* rank,
                    cudaStream_t st) {
  return svt_gram(h, W, m, n, eta, out, rank, st);
}

static int spectral_norm(Handles* h, const double* M, int64_t m, int64_t n, int iters, double* out, cudaStream_t st) {
  // row-major M (m x n) == column-major A = M^T (n x m, ld n)
  Buf v(st), w(st);
  L1F_CUDA_TRY(v.alloc(sizeof(double) * (size_t)n));
  L1F_CUDA_TRY(w.alloc(sizeof(double) * (size_t)m));
  std::vector<double> ones((size_t)n, 1.0 / std::sqrt((double)n));
  L1F_CUDA_TRY(cudaMemcpyAsync(v.p, ones.data(), sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, st));
  cublasSetPointerMode(h->blas, CUBLAS_POINTER_MODE_HOST);
  const double one = 1.0, zero = 0.0;
  double sigma = 0.0;
  for (int i = 0; i < iters; ++i) {
    double nw = 0.0;
    cublasDgemv(h->blas, CUBLAS_OP_T, (int)n, (int)m, &one, M, (int)n, v.d(), 1, &zero, w.d(), 1);  // w = M v
    cublasDnrm2(h->blas, (int)m, w.d(), 1, &nw);
    if (nw == 0.0) { *out = 0.0; return L1F_OK; }
    const double inv = 1.0 / nw;
    cublasDscal(h->blas, (int)m, &inv, w.d(), 1);
    cublasDgemv(h->blas, CUBLAS_OP_N, (int)n, (int)m, &one, M, (int)n, w.d(), 1, &zero, v.d(), 1);  // v = M^T w
    cublasDnrm2(h->blas, (int)n, v.d(), 1, &sigma);
    if (sigma == 0.0) { *out = 0.0; return L1F_OK; }
    const double is = 1.0 / sigma;
    cublasDscal(h->blas, (int)n, &is, v.d(), 1);
  }
  L1F_CUDA_TRY(cudaStreamSynchronize(st));
  *out = sigma;
  return L1F_OK;
}

}  // namespace seed
}  // namespace l1f

using namespace l1f;
using namespace l1f::seed;

extern "C" int l1f_svd_f64(const double* W, int64_t m, int64_t n, int64_t ldw, double* U, double* sigma, double* V,
                           void* stream) {
  L1F_REQUIRE(m >= 1 && n >= 1 && ldw >= n, L1F_ERR_ARG, "svd: bad shape");
  L1F_REQUIRE(m < INT32_MAX && n < INT32_MAX, L1F_ERR_UNSUPPORTED, "svd: matrix too large");
  cudaStream_t st = (cudaStream_t)stream;
  if (l1f_seed_small_applies(m, n)) return l1f_svd_small(W, m, n, ldw, U, sigma, V, st);
  Handles* h;
  int rc = handles(st, h);
  if (rc) return rc;
  return svd_rowmajor(h, W, m, n, ldw, U, sigma, V, st);
}

extern "C" int l1f_spectral_norm_f64(const double* M, int64_t m, int64_t n, int32_t iters, double* out_host,
                                     void* stream) {
  L1F_REQUIRE(m >= 1 && n >= 1 && iters >= 0, L1F_ERR_ARG, "spectral_norm: bad shape");
  Handles* h;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = handles(st, h);
  if (rc) return rc;
  return spectral_norm(h, M, m, n, iters, out_host, st);
}

// Thin SVD through the eigendecomposition of the smaller Gram matrix (the seed's final
// factorisation, l1filter.py:90-113 -> matcore.svd).  For a kept singular triplet (sigma_i >
// rank_tol * sigma_max) the computed U (or V) column is orthonormal to ~eps * sigma_max /
// sigma_i; sigma below ~sqrt(eps) * sigma_max are not resolved (they are cut as noise).
__global__ void eig_desc_rowmajor_kernel(const double* __restrict__ G, int p, double* __restrict__ out) {
  // out (p x p row-major)[i][j] = eigenvector j in descending order, component i
  const int64_t total = (int64_t)p * p;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / p, j = e - i * p;
    out[e] = G[(int64_t)(p - 1 - j) * p + i];
  }
}
__global__ void sigma_from_eig_kernel(const double* __restrict__ lam, int p, double* __restrict__ sig,
                                      double* __restrict__ inv) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < p; j += gridDim.x * blockDim.x) {
    const double l = lam[p - 1 - j];
    const double sg = l > 0.0 ? sqrt(l) : 0.0;
    sig[j] = sg;
    inv[j] = sg > 0.0 ? 1.0 / sg : 0.0;
  }
}

// eigenpairs from l1f_eig_sym_above (Z column-major p x k, lam descending) as a row-major p x p
// eigenvector matrix (columns >= k zero), sigma = sqrt(lam) (0 beyond k) and its reciprocal
__global__ void eig_pack_kernel(const double* __restrict__ Z, const double* __restrict__ lam, int k, int p,
                                double* __restrict__ out, double* __restrict__ sig, double* __restrict__ inv) {
  const int64_t total = (int64_t)p * p;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = x / p, j = x - i * p;
    out[x] = j < k ? Z[j * (int64_t)p + i] : 0.0;
  }
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < p; j += gridDim.x * blockDim.x) {
    const double l = j < k ? lam[j] : 0.0;
    const double sg = l > 0.0 ? sqrt(l) : 0.0;
    sig[j] = sg;
    inv[j] = sg > 0.0 ? 1.0 / sg : 0.0;
  }
}

static int svd_gram(Handles* h, const double* W, int64_t m, int64_t n, int64_t ldw, double* U, double* sig, double* V,
                    cudaStream_t st, bool force_lib = false) {
  const bool right = n <= m;
  const int p = (int)(right ? n : m), q = (int)(right ? m : n);
  Buf g(st), ev(st), work(st), info(st), inv(st);
  L1F_CUDA_TRY(g.alloc(sizeof(double) * (size_t)p * p));
  L1F_CUDA_TRY(ev.alloc(sizeof(double) * (size_t)p));
  L1F_CUDA_TRY(inv.alloc(sizeof(double) * (size_t)p));
  const double one = 1.0, zero = 0.0;
  cublasSetPointerMode(h->blas, CUBLAS_POINTER_MODE_HOST);
  // row-major W (m x n, ld ldw) == column-major X = W^T (n x m, ld ldw)
  if (right) cublasDsyrk(h->blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, p, q, &one, W, (int)ldw, &zero, g.d(), p);
  else cublasDsyrk(h->blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, p, q, &one, W, (int)ldw, &zero, g.d(), p);
  const int blocks = num_sms() * 4;
  if (!force_lib && hand_eig(p)) {
    // hand-written eigensolver: the triplets with sigma > 1e-7 sigma_max (every seed rank cut keeps
    // sigma > rank_tol * sigma_max with rank_tol >= 1e-6); the rest are returned as sigma = 0
    Buf z(st);
    L1F_CUDA_TRY(z.alloc(sizeof(double) * (size_t)p * p));
    int kk = 0;
    int rc = l1f_eig_sym_above(g.d(), p, 0.0, 1e-14, ev.d(), z.d(), &kk, st);
    if (rc == L1F_ERR_UNSUPPORTED) return svd_gram(h, W, m, n, ldw, U, sig, V, st, true);
    if (rc) return rc;
    eig_pack_kernel<<<blocks, 256, 0, st>>>(z.d(), ev.d(), kk, p, right ? V : U, sig, inv.d());
    L1F_CHECK_LAUNCH();
  } else {
  int lwork = 0;
  L1F_SOLVER(h, st);
  if (cusolverDnDsyevd_bufferSize(sol_, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, p, g.d(), p, ev.d(),
                                  &lwork) != CUSOLVER_STATUS_SUCCESS) {
    set_error("syevd_bufferSize failed");
    return L1F_ERR_CUDA;
  }
  L1F_CUDA_TRY(work.alloc(sizeof(double) * (size_t)(lwork > 0 ? lwork : 1)));
  L1F_CUDA_TRY(info.alloc(sizeof(int)));
  if (cusolverDnDsyevd(sol_, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, p, g.d(), p, ev.d(), work.d(), lwork,
                       (int*)info.p) != CUSOLVER_STATUS_SUCCESS) {
    set_error("cusolverDnDsyevd failed");
    return L1F_ERR_SVD;
  }
  int info_h = 0;
  L1F_CUDA_TRY(cudaMemcpyAsync(&info_h, info.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  L1F_CUDA_TRY(cudaStreamSynchronize(st));
  if (info_h != 0) {
    set_error("SVD (Gram) failed on (%lld, %lld) matrix: syevd info %d", (long long)m, (long long)n, info_h);
    return L1F_ERR_SVD;
  }
  sigma_from_eig_kernel<<<(p + 255) / 256, 256, 0, st>>>(ev.d(), p, sig, inv.d());
  eig_desc_rowmajor_kernel<<<blocks, 256, 0, st>>>(g.d(), p, right ? V : U);
  }
  if (right) {
    // V (n x p row-major) = eigenvectors; U (m x p row-major) = W V diag(1/sigma):
    // column-major U^T (p x m) = V^T (col-major view of V) * W^T (col-major view of W)
    cublasDgemm(h->blas, CUBLAS_OP_N, CUBLAS_OP_N, p, (int)m, (int)n, &one, V, p, W, (int)ldw, &zero, U, p);
    scale_cols_kernel<<<blocks, 256, 0, st>>>(U, m, p, p, inv.d());
  } else {
    // U (m x p row-major) = eigenvectors; V (n x p row-major) = W^T U diag(1/sigma):
    // column-major V^T (p x n) = U^T (col-major view of U) * W (transpose of the col-major view)
    cublasDgemm(h->blas, CUBLAS_OP_N, CUBLAS_OP_T, p, (int)n, (int)m, &one, U, p, W, (int)ldw, &zero, V, p);
    scale_cols_kernel<<<blocks, 256, 0, st>>>(V, n, p, p, inv.d());
  }
  L1F_CHECK_LAUNCH();
  return L1F_OK;
}

// One-time initialisation on the current device (include/l1pcp_b200.h l1f_init): the cuBLAS handle
// and its first dsyrk / dgemm (cuBLAS loads its kernels on first use), and one small run of the
// hand-written eigensolver so its kernels are loaded; idempotent per host thread
extern "C" int l1f_init(void* stream) {
  static thread_local bool done_dev[64] = {};
  int dev = 0;
  L1F_CUDA_TRY(cudaGetDevice(&dev));
  bool& done = done_dev[dev & 63];
  if (done) return L1F_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Handles* h;
  int rc = handles(st, h);
  if (rc) return rc;
  const int p = 16;
  Buf a(st), g(st), lam(st), z(st);
  L1F_CUDA_TRY(a.alloc(sizeof(double) * p * p));
  L1F_CUDA_TRY(g.alloc(sizeof(double) * p * p));
  L1F_CUDA_TRY(lam.alloc(sizeof(double) * p));
  L1F_CUDA_TRY(z.alloc(sizeof(double) * p * p));
  std::vector<double> ha((size_t)p * p);
  for (int i = 0; i < p * p; ++i) ha[(size_t)i] = (i % p == i / p) ? 2.0 + i % p : 0.25 / (1 + i % 7);
  L1F_CUDA_TRY(cudaMemcpyAsync(a.p, ha.data(), sizeof(double) * p * p, cudaMemcpyHostToDevice, st));
  const double one = 1.0, zero = 0.0;
  cublasSetPointerMode(h->blas, CUBLAS_POINTER_MODE_HOST);
  cublasDsyrk(h->blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, p, p, &one, a.d(), p, &zero, g.d(), p);
  cublasDgemm(h->blas, CUBLAS_OP_N, CUBLAS_OP_N, p, p, p, &one, a.d(), p, g.d(), p, &zero, z.d(), p);
  cublasDgemm(h->blas, CUBLAS_OP_T, CUBLAS_OP_N, p, p, p, &one, a.d(), p, g.d(), p, &zero, z.d(), p);
  int k = 0;
  rc = l1f_eig_sym_above(g.d(), p, 0.0, 0.5, lam.d(), z.d(), &k, st);
  if (rc && rc != L1F_ERR_UNSUPPORTED) return rc;  // (unsupported: the library path serves instead)
  L1F_CUDA_TRY(cudaStreamSynchronize(st));
  done = true;
  return L1F_OK;
}

extern "C" int l1f_svd_gram_f64(const double* W, int64_t m, int64_t n, int64_t ldw, double* U, double* sigma,
                                double* V, void* stream) {
  L1F_REQUIRE(m >= 1 && n >= 1 && ldw >= n, L1F_ERR_ARG, "svd_gram: bad shape");
  L1F_REQUIRE(m < INT32_MAX && n < INT32_MAX, L1F_ERR_UNSUPPORTED, "svd_gram: matrix too large");
  cudaStream_t st = (cudaStream_t)stream;
  if (l1f_seed_small_applies(m, n)) return l1f_svd_small(W, m, n, ldw, U, sigma, V, st);
  Handles* h;
  int rc = handles(st, h);
  if (rc) return rc;
  return svd_gram(h, W, m, n, ldw, U, sigma, V, st);
}

extern "C" int l1f_svt_f64(const double* W, int64_t m, int64_t n, double eta, double* out, int32_t* rank_host,
                           void* stream) {
  L1F_REQUIRE(m >= 1 && n >= 1, L1F_ERR_ARG, "svt: bad shape");
  L1F_REQUIRE(eta >= 0.0, L1F_ERR_ARG, "eta must be nonnegative");
  Handles* h;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = handles(st, h);
  if (rc) return rc;
  int k = 0;
  rc = svt_into(h, W, m, n, eta, out, &k, st);
  *rank_host = k;
  return rc;
}

extern "C" int l1f_pcp_f64(const double* M, int64_t m, int64_t n, double lam, double tol, double beta0, double rho,
                           double beta_max, int32_t max_iter, double* L, double* S, int32_t* iters_host,
                           double* residual_host, int32_t* rank_host, int32_t* converged_host,
                           double* beta_final_host, void* stream) {
  L1F_REQUIRE(m >= 1 && n >= 1, L1F_ERR_ARG, "matrix must be nonempty");
  L1F_REQUIRE(rho > 1.0 && tol > 0.0 && lam > 0.0, L1F_ERR_ARG, "pcp: need rho > 1, tol > 0, lam > 0");
  cudaStream_t st = (cudaStream_t)stream;
  if (l1f_seed_small_applies(m, n))  // one persistent CTA, hand-written Jacobi SVT (seed_small.cu)
    return l1f_pcp_small(M, n, m, n, lam, tol, beta0, rho, beta_max, max_iter, L, S, iters_host, residual_host,
                         rank_host, converged_host, beta_final_host, st);
  Handles* h;
  int rc = handles(st, h);
  if (rc) return rc;
  const int64_t count = m * n;
  const int g = reduce_blocks();
  Buf y(st), w(st), part(st), scal(st);
  L1F_CUDA_TRY(part.alloc(sizeof(double) * (size_t)g));
  L1F_CUDA_TRY(scal.alloc(sizeof(double)));
  double norm2 = 0.0;
  rc = sumsq(M, count, part.d(), scal.d(), &norm2, st);
  if (rc) return rc;
  const double norm_m = std::sqrt(norm2);
  L1F_CUDA_TRY(cudaMemsetAsync(L, 0, sizeof(double) * (size_t)count, st));
  L1F_CUDA_TRY(cudaMemsetAsync(S, 0, sizeof(double) * (size_t)count, st));
  *iters_host = 0; *residual_host = 1.0; *rank_host = 0; *converged_host = 0; *beta_final_host = 0.0;
  if (norm_m == 0.0) {  // pcp_adm.py:99-105
    *iters_host = 1; *residual_host = 0.0; *converged_host = 1;
    L1F_CUDA_TRY(cudaStreamSynchronize(st));
    return L1F_OK;
  }
  double beta = beta0;
  if (!(beta0 > 0.0)) {
    double sn = 0.0;
    rc = spectral_norm(h, M, m, n, 25, &sn, st);
    if (rc) return rc;
    beta = 1.25 / (sn > DBL_MIN ? sn : DBL_MIN);
  }
  const double bmax = beta_max > 0.0 ? beta_max : 1e7 * beta;
  L1F_CUDA_TRY(y.alloc(sizeof(double) * (size_t)count));
  L1F_CUDA_TRY(w.alloc(sizeof(double) * (size_t)count));
  L1F_CUDA_TRY(cudaMemsetAsync(y.p, 0, sizeof(double) * (size_t)count, st));
  double residual = 1.0;
  int rank = 0, it = 0, converged = 0;
  const int eg = num_sms() * 8;
  for (it = 1; it <= max_iter; ++it) {
    pcp_shrink_kernel<<<eg, 256, 0, st>>>(M, L, y.d(), S, w.d(), count, beta, lam / beta);
    L1F_CHECK_LAUNCH();
    rc = svt_loop(h, w.d(), m, n, 1.0 / beta, L, &rank, st);
    if (rc) return rc;
    pcp_residual_kernel<<<g, 256, 0, st>>>(M, L, S, y.d(), count, beta, part.d());
    L1F_CHECK_LAUNCH();
    sum_kernel<<<1, 32, 0, st>>>(part.d(), g, scal.d());
    L1F_CHECK_LAUNCH();
    double r2 = 0.0;
    L1F_CUDA_TRY(cudaMemcpyAsync(&r2, scal.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    L1F_CUDA_TRY(cudaStreamSynchronize(st));
    residual = std::sqrt(r2) / norm_m;
    if (!std::isfinite(residual)) {
      set_error("non-finite residual at iteration %d (beta=%.3g)", it, beta);
      return L1F_ERR_DIVERGED;
    }
    if (residual <= tol) { converged = 1; break; }
    beta = std::min(rho * beta, bmax);
  }
  if (it > max_iter) it = max_iter;
  *iters_host = it;
  *residual_host = residual;
  *rank_host = rank;
  *converged_host = converged;
  *beta_final_host = beta;
  L1F_CUDA_TRY(cudaStreamSynchronize(st));
  return L1F_OK;
}
