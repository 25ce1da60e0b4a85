/*
 * l1pcp_b200 — C ABI of the B200-native l1-filtering PCP hot path.
 *
 * This is the drop-in boundary for the data-parallel core of the reference package
 * `l1pcp` (/root/reference/pkg/src/l1pcp). The reference is pure Python/numpy and has no
 * FFI of its own, so each entry point below names the reference function it replaces
 * (file:line, relative to pkg/src/l1pcp/); a reference-side binding (ctypes) is shown in
 * INTEGRATION.md.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers unless the parameter name ends in `_host`.
 *  - Matrices are row-major with an explicit leading dimension (elements, not bytes).
 *  - "Unit-major" panels store one l1-regression unit (a column of the reference's X,
 *    l1reg.py:59) contiguously: x_u[i] = X[u*ldx + i].
 *  - Work is enqueued on `stream` (a cudaStream_t; NULL = legacy default stream) and is
 *    stream-ordered; entry points that return host values synchronise that stream.
 *  - Return value: L1F_OK (0) or a negative L1F_ERR_* code; l1f_last_error() gives the
 *    message for the calling thread. No exception crosses the ABI.
 *  - dtype codes: L1F_F32 (float) / L1F_F64 (double).
 */
#ifndef L1PCP_B200_H_
#define L1PCP_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define L1F_OK 0
#define L1F_ERR_ARG (-1)          /* invalid argument (reference: ValueError)              */
#define L1F_ERR_CUDA (-2)         /* CUDA runtime failure                                   */
#define L1F_ERR_SVD (-3)          /* SVD did not converge (matcore.py:9-10,82-85)           */
#define L1F_ERR_DIVERGED (-4)     /* non-finite PCP residual (pcp_adm.py:19-20,126-129)     */
#define L1F_ERR_UNSUPPORTED (-5)  /* shape outside the compiled kernel family               */

#define L1F_F32 0
#define L1F_F64 1

/* per-unit status written by l1f_filter_* (reference bookkeeping l1reg.py:107-135) */
#define L1F_UNIT_OK 0       /* res <= tol*||x||_inf                                        */
#define L1F_UNIT_STALLED 1  /* 20 iterations of relative change < 1e-12, not ok -> failed   */
#define L1F_UNIT_MAXITER 2  /* max_iter exhausted -> failed                                 */
#define L1F_UNIT_ZERO 3     /* ||x||_inf == 0: z = e = 0, iterations 0, not failed          */

/* generator kinds for l1f_generate_f32 */
#define L1F_GEN_GAUSSIAN 0  /* L0 = X Y^T, X,Y ~ N(0,1); S0 Bernoulli(rho_s) x U[-mag,mag]  */
#define L1F_GEN_VIDEO 1     /* L0 = X Y^T, X ~ U[0,1), Y ~ U[0,1)*255/r; S0 moving boxes    */

/* Library options: explicit, process-wide switches of the kernel selection (A/B comparisons and
 * tests).  The defaults are the production choices; nothing is read from the environment. */
#define L1F_OPT_FILTER_STREAMING 1  /* 1: every filter call takes the streaming SIMT kernel (default 0) */
#define L1F_OPT_FILTER_TC 2         /* 0: no tensor-core filter kernel (default 1)                      */
#define L1F_OPT_TC_GROUPS 3         /* 2: at most two slot groups per CTA; 0: automatic (default)       */
#define L1F_OPT_RECON_TC 4          /* 0: no tensor-core reconstruction (default 1)                      */
#define L1F_OPT_RECON_STREAM 5      /* 0: the overlapped row-filter + reconstruction calls decline
                                       with L1F_ERR_UNSUPPORTED (default 1)                              */
#define L1F_OPT_RECON_CONCURRENT 6  /* 0: the streamed reconstruction runs only after the filter
                                       (no concurrent launch on the idle SMs; default 1)                 */
#define L1F_OPT_GATHER_OVERLAP 7    /* 0: l1f_filter_with_gather_f32 declines (default 1)                */
#define L1F_OPT_WAIT_TIMEOUT_MS 8   /* bound of the device-side waits of the overlapped calls (default
                                       10000; 0 = give up at once, tests).  A timed-out wait leaves the
                                       call's residual NaN; the caller must then recompute the step
                                       with the separate calls (the Python layer does)               */
#define L1F_OPT_SMALL_LANES 9       /* lanes per unit of the k <= 10 filter kernel: 0 auto (8 for s <= 104),
                                       16 or 32                                                          */
#define L1F_OPT_SEED_EIG 10         /* eigensolver of the Gram matrix in the seed SVT / factorisation for
                                       blocks the small-block kernel does not take: 2 auto (default:
                                       the hand-written solver of eig_sym.cu wherever its shared-
                                       memory-resident tridiagonalisation applies, p <= 2000 on 148
                                       SMs; cuSOLVER syevd beyond), 1 syevd always, 0 hand-written
                                       always (Householder tridiagonalisation + bisection + inverse
                                       iteration + back-transformation; same results to ~5e-15)       */
#define L1F_OPT_SEED_SMALL_SVT 11   /* SVT inside the one-CTA small-block ALM kernel: 1 Gram matrix +
                                       shared-memory Householder tridiagonalisation + bisection +
                                       inverse iteration (default), 0 one-sided Jacobi on the block   */
#define L1F_OPT_SEED_EIG_DSM 12     /* tridiagonalisation of the hand-written eigensolver: 1 the matrix
                                       resident in the shared memory of all SMs, one grid-wide wait per
                                       column (default, p <= 2000); 0 the L2-resident two-barrier form */
int l1f_set_option(int key, int64_t value);
int l1f_get_option(int key, int64_t* value_host);

const char* l1f_last_error(void);
int l1f_version(void);
/* one-time initialisation on the current device (the cuBLAS handle and its first GEMMs, the
 * eigensolver's kernels); idempotent per device and host thread.  The Python layer calls it once
 * after loading the library; a caller that skips it pays the same cost inside its first seed solve. */
int l1f_init(void* stream);
/* number of SMs of the current device, written to *out_host */
int l1f_sm_count(int* out_host);

/* ------------------------------------------------------------------------------------
 * Column-separable l1 regression by ADM — replaces `_solve_block` (l1reg.py:59-137), the
 * body of `solve_l1reg` (l1reg.py:140-160) and `solve_l1reg_columnwise`
 * (l1reg.py:163-214).  Solves, independently per unit u (x_u of length s):
 *     min ||e||_1  s.t.  x_u = A z_u + e_u,   A (s x k) with orthonormal columns,
 * with the reference's per-unit penalty schedule (beta0 = 1/||x_u||_inf unless beta0>0;
 * beta_max = 1e7*beta0 unless beta_max>0), per-unit stop res <= tol*||x_u||_inf,
 * stagnation rule (20 iterations below 1e-12 relative change) and max_iter.
 *  X   unit-major panel, n_units x s, leading dimension ldx >= s
 *  A   s x k row-major (lda >= k); orthonormality is validated by the caller
 *  Z   unit-major output n_units x k (ldz >= k)            -> reference z (transposed)
 *  E   unit-major output n_units x s (lde >= s), nullable  -> reference e (transposed)
 *  iters/res/status: per-unit iteration count, final max|r|, L1F_UNIT_* code (nullable)
 *  workspace: l1f_filter_workspace_bytes() bytes, or NULL to allocate stream-ordered.
 * Results are bitwise independent of n_units, unit order and GPU count.
 * ---------------------------------------------------------------------------------- */
size_t l1f_filter_workspace_bytes(int dtype, int32_t s, int32_t k, int64_t n_units);
int l1f_filter_f32(const float* X, int64_t ldx, int32_t s, int64_t n_units,
                   const float* A, int64_t lda, int32_t k,
                   float tol, float rho, float beta0, float beta_max, int32_t max_iter,
                   float* Z, int64_t ldz, float* E, int64_t lde,
                   int32_t* iters, float* res, uint8_t* status,
                   void* workspace, size_t workspace_bytes, void* stream);
int l1f_filter_f64(const double* X, int64_t ldx, int32_t s, int64_t n_units,
                   const double* A, int64_t lda, int32_t k,
                   double tol, double rho, double beta0, double beta_max, int32_t max_iter,
                   double* Z, int64_t ldz, double* E, int64_t lde,
                   int32_t* iters, double* res, uint8_t* status,
                   void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------------------
 * Column and row filtering in one call — filter_columns + filter_rows (l1filter.py:116-134)
 * as the pipeline runs them (l1filter.py:244-245), fp32, no e output.  Unit set 1 (X1, A1)
 * and unit set 2 (X2, A2) share s and k.  With the tensor-core kernel the two sets can run in
 * one grid, the clusters split in proportion to their sizes, so the drains at the end of the
 * two sets overlap; mode 0 lets the library choose by its pass-count model, 1 forces one
 * launch, 2 two launches.  Per-unit results are bitwise those of two l1f_filter_f32 calls.
 * ---------------------------------------------------------------------------------- */
int l1f_filter_pair_f32(const float* X1, int64_t ldx1, int64_t n1, const float* A1, int64_t lda1,
                        float* Z1, int64_t ldz1, int32_t* iters1, float* res1, uint8_t* status1,
                        const float* X2, int64_t ldx2, int64_t n2, const float* A2, int64_t lda2,
                        float* Z2, int64_t ldz2, int32_t* iters2, float* res2, uint8_t* status2,
                        int32_t s, int32_t k, float tol, float rho, float beta0, float beta_max,
                        int32_t max_iter, int32_t mode, void* stream);

/* Whether l1f_filter_pair_f32 (mode 0) would run the two unit sets in one grid: *one_grid = 1
 * or 0 (0 also when the tensor-core kernel does not apply).  No device work. */
int l1f_filter_pair_plan_f32(int32_t s, int32_t k, int64_t n1, int64_t n2, int32_t* one_grid);

/* ------------------------------------------------------------------------------------
 * Index gather — replaces `m[np.ix_(rows, cols)]` (l1filter.py:87 sample_submatrix,
 * :242-243 panel extraction).  out[r][c] = M[rows[r]][cols[c]] (transpose=0) or
 * out[c][r] (transpose=1, the unit-major column panel).  rows/cols may be NULL (= arange).
 * Converts dtype_in -> dtype_out on the fly.
 * ---------------------------------------------------------------------------------- */
int l1f_gather(int dtype_in, const void* M, int64_t ldm,
               const int64_t* rows, int64_t n_rows, const int64_t* cols, int64_t n_cols,
               int dtype_out, void* out, int64_t ldo, int32_t transpose, void* stream);

/* ------------------------------------------------------------------------------------
 * Rank-k completion factors — the unified form of `nystrom_complete` (l1filter.py:137-141)
 * and the four blocks of `assemble` (l1filter.py:151-167):  L[i][j] = Af[i] . Bf[j] with
 *   Af[i] = U[p]                 (i = row_idx[p], a seed row)
 *         = Zr[i'] / sigma       (i the i'-th non-seed row; Zr = P~^T, unit-major)
 *   Bf[j] = sigma * V[q]         (j = col_idx[q], a seed column)
 *         = Zc[j']               (j the j'-th non-seed column; Zc = Q~^T, unit-major)
 * row_idx / col_idx must be sorted ascending (sample_submatrix sorts them, l1filter.py:85-86).
 * U (s_r x k), sigma (k), V (s_c x k) are the seed factors in FP64.
 * ---------------------------------------------------------------------------------- */
int l1f_build_factors(int dtype, int64_t m, int64_t n, int32_t k,
                      const int64_t* row_idx, int64_t s_r, const int64_t* col_idx, int64_t s_c,
                      const double* U, const double* sigma, const double* V,
                      const void* Zc, int64_t ldzc, const void* Zr, int64_t ldzr,
                      void* Af, void* Bf, void* stream);

/* ------------------------------------------------------------------------------------
 * Reconstruction + residual — replaces `nystrom_complete`+`assemble` (l1filter.py:137-167),
 * `s = m - l` (:253) and the residual numerator/denominator (:256-257):
 *   L = Af Bf^T (m x n, K = k),  S = M - L,  resid_sq[0] += sum((M-L)-S)^2,
 *   resid_sq[1] += sum(M^2)   (resid_sq is a device double[2], zeroed by the callee).
 * M and S may be NULL (then only L is formed, e.g. the completion block alone).
 * ---------------------------------------------------------------------------------- */
int l1f_reconstruct(int dtype, int64_t m, int64_t n, int32_t k,
                    const void* Af, int64_t ldaf, const void* Bf, int64_t ldbf,
                    const void* M, int64_t ldm, void* L, int64_t ldl, void* S, int64_t lds,
                    double* resid_sq, void* stream);

/* ------------------------------------------------------------------------------------
 * Row filtering and reconstruction, overlapped — filter_rows (l1filter.py:125-134) followed
 * by assemble + s = m - l (l1filter.py:151-167,253), for the fp32 tensor-core path.
 * Runs the row units X (the m - s_r non-seed rows of M, in order; unit_rows[u] = their row
 * index, i.e. comp_rows) against V exactly as l1f_filter_f32 (no e output), then
 *   L = Af Bf^T, S = M - L, resid_sq as l1f_reconstruct,
 * with Af built from (row_idx, U, sigma, Zr) and Bf from (col_idx, sigma, V64, Zc = the column
 * filter's z) as l1f_build_factors does.  L and S are bitwise those of l1f_filter_f32 +
 * l1f_build_factors + l1f_reconstruct.  Bf, its pieces and the reconstruction of each 128-row
 * strip run on the SMs the filter's clusters leave free, a strip as soon as its row units are
 * finished; the rest follows the filter on every SM.
 * ev_filter_done (a cudaEvent_t, nullable) is recorded on `stream` after the filter launch.
 * Returns L1F_ERR_UNSUPPORTED (nothing to undo; call the three functions instead) when the
 * tensor-core filter or reconstruction does not apply (k <= 16, k > 224, alignment).
 * ---------------------------------------------------------------------------------- */
int l1f_rowfilter_reconstruct_f32(const float* X, int64_t ldx, int32_t s, int64_t n_units,
                                  const float* V, int64_t ldv, int32_t k, float tol, float rho,
                                  float beta0, float beta_max, int32_t max_iter,
                                  float* Zr, int64_t ldz, int32_t* iters, float* res, uint8_t* status,
                                  const int64_t* unit_rows, const int64_t* row_idx, int64_t s_r,
                                  const double* U, const double* sigma, const int64_t* col_idx,
                                  int64_t s_c, const double* V64, const float* Zc, int64_t ldzc,
                                  const float* M, int64_t m, int64_t n, int64_t ldm,
                                  float* L, int64_t ldl, float* S, int64_t lds, double* resid_sq,
                                  void* ev_filter_done, void* stream);

/* The same for k <= 16 with the FP64 small-k filter (configs 1 and 4): X, V, Zr, res in FP64;
 * Zc is the column filter's z rounded to fp32 (as the pipeline's factor build reads it).  The
 * reconstruction runs beside the filter's blocks on the same SMs.  L, S bitwise those of
 * l1f_filter_f64 + l1f_build_factors + l1f_reconstruct (float). */
int l1f_rowfilter_reconstruct_small(const double* X, int64_t ldx, int32_t s, int64_t n_units,
                                    const double* V, int64_t ldv, int32_t k, double tol, double rho,
                                    double beta0, double beta_max, int32_t max_iter,
                                    double* Zr, int64_t ldz, int32_t* iters, double* res, uint8_t* status,
                                    const int64_t* unit_rows, const int64_t* row_idx, int64_t s_r,
                                    const double* U, const double* sigma, const int64_t* col_idx,
                                    int64_t s_c, const double* V64, const float* Zc, int64_t ldzc,
                                    const float* M, int64_t m, int64_t n, int64_t ldm,
                                    float* L, int64_t ldl, float* S, int64_t lds, double* resid_sq,
                                    void* ev_filter_done, void* stream);

/* ------------------------------------------------------------------------------------
 * A filter launch with an index gather beside it — filter_columns (l1filter.py:116-122) while
 * the row panel m[np.ix_(comp_rows, col_idx)] (l1filter.py:243) is extracted: the filter as
 * l1f_filter_f32 (no e output) and out = l1f_gather(dtype_in, M, ..., L1F_F32, out, ...), the
 * gather on the SMs the filter's clusters leave free once they are all resident.  Both are
 * complete when the stream reaches the next operation.  L1F_ERR_UNSUPPORTED (nothing launched)
 * when the tensor-core filter does not apply; then call the two functions.
 * ---------------------------------------------------------------------------------- */
int l1f_filter_with_gather_f32(const float* X, int64_t ldx, int32_t s, int64_t n_units,
                               const float* A, int64_t lda, int32_t k, float tol, float rho,
                               float beta0, float beta_max, int32_t max_iter,
                               float* Z, int64_t ldz, int32_t* iters, float* res, uint8_t* status,
                               int32_t dtype_in, const void* M, int64_t ldm,
                               const int64_t* rows, int64_t n_rows, const int64_t* cols, int64_t n_cols,
                               float* out, int64_t ldo, int32_t transpose, void* stream);

/* General C = alpha * A B^T (+ beta*C), A m x k, B n x k, row-major; used for the small
 * dense products of the reference API (SkinnySvd.reconstruct matcore.py:36-38,
 * pseudo_inverse_apply matcore.py:116-123, nystrom_complete_via_pinv l1filter.py:144-148). */
int l1f_gemm_nt(int dtype, int64_t m, int64_t n, int64_t k, double alpha,
                const void* A, int64_t lda, const void* B, int64_t ldb,
                double beta, void* C, int64_t ldc, void* stream);

/* ------------------------------------------------------------------------------------
 * Synthetic inputs — replaces `synth.generate` (synth.py:43-64) for the benchmark configs
 * by a counter-based Philox4x64-10 generator (bit-identical to numpy.random.Philox with
 * counter = block index), so any row shard [row0, row0+rows) is reproducible on any rank.
 *  l1f_generate_factors_f32: X (m x r) and Y (n x r) row-major.
 *  l1f_generate_f32: rows [row0,row0+rows) of M = L0 + S0 (and of L0 when L0 != NULL),
 *     L0[i][j] = sum_t X[i][t]*Y[j][t] accumulated in t order with separately rounded
 *     multiply and add (no FMA), so the numpy oracle reproduces it bit for bit.
 * ---------------------------------------------------------------------------------- */
int l1f_generate_factors_f32(uint64_t seed, int32_t kind, int64_t m, int64_t n, int32_t r,
                             float* X, float* Y, void* stream);
int l1f_generate_f32(uint64_t seed, int32_t kind, int64_t m, int64_t n, int32_t r,
                     float rho_s, float magnitude, const float* X, const float* Y,
                     int64_t row0, int64_t rows, float* M, int64_t ldm,
                     float* L0, int64_t ldl0, void* stream);

/* Exact-count sparse part — replaces synth.generate's support and values (synth.py:56-61):
 * S (dtype L1F_F32/L1F_F64, m*n contiguous, row-major) gets exactly p nonzeros at uniformly random
 * distinct positions (a radix select of the p smallest Philox keys, on the device), each
 * U[-magnitude, magnitude).  ValueError-equivalent L1F_ERR_ARG when p > m*n. */
int l1f_generate_sparse_exact(int dtype, uint64_t seed, int64_t m, int64_t n, int64_t p, double magnitude,
                              void* S, void* stream);

/* ------------------------------------------------------------------------------------
 * Reductions — `frobenius_norm`, `l1_norm`, `linf_norm`, `l0_count` and the finiteness
 * check of `as_dense` (matcore.py:13-20,41-63).  out (device double[5]):
 *   [0] sum|x|, [1] max|x|, [2] sum x^2, [3] count(|x| > thr), [4] count(non-finite)
 * Deterministic (fixed-order two-level reduction, no float atomics).
 * l1f_diff_norms: out2 = { sum (a-b)^2, sum b^2 }  (rel_err synth.py:92-97)
 * ---------------------------------------------------------------------------------- */
int l1f_norms(int dtype, const void* X, int64_t rows, int64_t cols, int64_t ld, double thr,
              double* out5, void* stream);
int l1f_diff_norms(int dtype, const void* A, int64_t lda, const void* B, int64_t ldb,
                   int64_t rows, int64_t cols, double* out2, void* stream);
/* Y = sign(X) * max(|X| - eta, 0) elementwise (matcore.py:66-70); X, Y may alias. */
int l1f_soft_threshold(int dtype, const void* X, void* Y, int64_t count, double eta,
                       void* stream);

/* ------------------------------------------------------------------------------------
 * Seed-stage dense kernels (FP64) — the small PCP of `recover_seed` (l1filter.py:90-113).
 *  l1f_svd_f64: thin SVD W = U diag(sigma) V^T, p = min(m,n), sigma descending
 *     (matcore.py:73-88 before the rank cut).  U m x p, V n x p, row-major.
 *  l1f_svd_gram_f64: the same outputs through the eigendecomposition of the smaller Gram
 *     matrix (the seed's final factorisation, l1filter.py:90-113): columns with sigma_i above
 *     ~sqrt(eps) * sigma_max are accurate to ~eps * sigma_max / sigma_i; smaller ones are noise
 *     (below the seed's rank cut of 1e-6 * sigma_max).
 *  l1f_spectral_norm_f64: 25-step power iteration from the all-ones vector
 *     (pcp_adm.py:69-87); result to *out_host.
 *  l1f_svt_f64: out = U max(sigma - eta, 0) V^T and *rank_host = #(sigma > eta)
 *     (matcore.py:96-105).
 *  l1f_pcp_f64: inexact-ALM PCP (pcp_adm.py:90-140) with lam, beta0 (<=0: 1.25/||M||_2),
 *     beta_max (<=0: 1e7*beta0), rho, tol, max_iter.  Host outputs: iterations, final
 *     residual, rank of L, converged flag, final beta.
 * ---------------------------------------------------------------------------------- */
int l1f_svd_f64(const double* W, int64_t m, int64_t n, int64_t ldw,
                double* U, double* sigma, double* V, void* stream);
int l1f_svd_gram_f64(const double* W, int64_t m, int64_t n, int64_t ldw,
                     double* U, double* sigma, double* V, void* stream);
int l1f_spectral_norm_f64(const double* M, int64_t m, int64_t n, int32_t iters,
                          double* out_host, void* stream);
int l1f_svt_f64(const double* W, int64_t m, int64_t n, double eta, double* out,
                int32_t* rank_host, void* stream);
int l1f_pcp_f64(const double* M, int64_t m, int64_t n, double lam, double tol,
                double beta0, double rho, double beta_max, int32_t max_iter,
                double* L, double* S, int32_t* iters_host, double* residual_host,
                int32_t* rank_host, int32_t* converged_host, double* beta_final_host,
                void* stream);

/* FP32 FMA-throughput microbenchmark (roofline denominator for the filter kernel):
 * runs `iters` dependent-chain FMA loops on every SM; *flops_host = FLOPs executed. */
int l1f_fma_peak_probe(int32_t iters, float* sink, double* flops_host, void* stream);
/* the same for FP64 FMAs (sink: 8 x SMs doubles): the roofline of the FP64 small-k filter */
int l1f_fma_peak_probe_f64(int32_t iters, double* sink, double* flops_host, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* L1PCP_B200_H_ */
