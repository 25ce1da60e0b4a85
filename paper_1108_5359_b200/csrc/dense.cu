// Streaming kernels of the l1-filtering path around the filter:
//   - reconstruction L = Af Bf^T, S = M - L, residual partials (l1filter.py:137-167,253-257)
//   - rank-k factor build (unified nystrom_complete/assemble, l1filter.py:137-167)
//   - Philox synthetic generator (replaces synth.generate, synth.py:43-64)
//   - index gathers (m[np.ix_], l1filter.py:87,242-243)
//   - norms / finiteness / soft threshold (matcore.py:13-20,41-70)
#include "common.cuh"
#include "gemm_tile.cuh"
#include "philox.cuh"

#include <cstdarg>
#include <cstdio>
#include <mutex>

namespace l1f {

// ---------------------------------------------------------------- stream-ordered scratch
struct Scratch {
  void* p = nullptr;
  cudaStream_t s;
  explicit Scratch(cudaStream_t st) : s(st) {}
  cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, bytes ? bytes : 16, s); }
  ~Scratch() { if (p) cudaFreeAsync(p, s); }
};

// ---------------------------------------------------------------- 4-wide row access
template <typename T>
__device__ __forceinline__ void load4(const T* __restrict__ row, int64_t c, int64_t n, T (&v)[4]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) v[q] = (c + q < n) ? row[c + q] : T(0);
}
template <typename T>
__device__ __forceinline__ void store4(T* __restrict__ row, int64_t c, int64_t n, const T (&v)[4]) {
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (c + q < n) row[c + q] = v[q];
}
template <>
__device__ __forceinline__ void load4<float>(const float* __restrict__ row, int64_t c, int64_t n, float (&v)[4]) {
  const float* p = row + c;
  if (c + 3 < n && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
    float4 t = __ldcs(reinterpret_cast<const float4*>(p));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = (c + q < n) ? p[q] : 0.0f;
  }
}
template <>
__device__ __forceinline__ void store4<float>(float* __restrict__ row, int64_t c, int64_t n, const float (&v)[4]) {
  float* p = row + c;
  if (c + 3 < n && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (c + q < n) p[q] = v[q];
  }
}

__device__ __forceinline__ void block_sum2(double& a, double& b, double* out_a, double* out_b) {
  __shared__ double red[2][32];
  a = warp_sum(a);
  b = warp_sum(b);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) { red[0][w] = a; red[1][w] = b; }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x / 32;
    a = l < nw ? red[0][l] : 0.0;
    b = l < nw ? red[1][l] : 0.0;
    a = warp_sum(a);
    b = warp_sum(b);
    if (l == 0) { *out_a = a; *out_b = b; }
  }
}

// fixed-order final sum of per-block partial pairs
__global__ void sum_pairs_kernel(const double* __restrict__ part, int64_t nparts, double* out) {
  double a = 0.0, b = 0.0;
  for (int64_t i = threadIdx.x; i < nparts; i += blockDim.x) {
    a += part[2 * i];
    b += part[2 * i + 1];
  }
  block_sum2(a, b, &out[0], &out[1]);
}

// ---------------------------------------------------------------- GEMM C = alpha A B^T + beta C
template <typename T>
__global__ void __launch_bounds__(kTileThreads)
gemm_nt_kernel(int64_t m, int64_t n, int k, T alpha, const T* __restrict__ A, int64_t lda,
               const T* __restrict__ B, int64_t ldb, T beta, T* __restrict__ C, int64_t ldc) {
  __shared__ TileSmem<T> sm;
  const int64_t r0 = (int64_t)blockIdx.y * kTile, c0 = (int64_t)blockIdx.x * kTile;
  T acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = T(0);
  tile_mainloop<T, false>(A, lda, B, ldb, m, n, k, r0, c0, acc, sm);
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = r0 + tile_row(ty, i);
    if (r >= m) continue;
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const int64_t c = c0 + 4 * tx + 64 * g;
      T* row = C + r * ldc;
      T v[4], old[4] = {T(0), T(0), T(0), T(0)};
      if (beta != T(0)) load4(row, c, n, old);
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = alpha * acc[i][4 * g + q] + (beta != T(0) ? beta * old[q] : T(0));
      store4(row, c, n, v);
    }
  }
}

// ---------------------------------------------------------------- reconstruction
// L = Af Bf^T, S = M - L; partial sums of ((M-L)-S)^2 and M^2 per CTA.
template <typename T>
__global__ void __launch_bounds__(kTileThreads)
reconstruct_kernel(int64_t m, int64_t n, int k, const T* __restrict__ Af, int64_t ldaf,
                   const T* __restrict__ Bf, int64_t ldbf, const T* __restrict__ M, int64_t ldm,
                   T* __restrict__ L, int64_t ldl, T* __restrict__ S, int64_t lds,
                   double* __restrict__ part) {
  __shared__ TileSmem<T> sm;
  const int64_t r0 = (int64_t)blockIdx.y * kTile, c0 = (int64_t)blockIdx.x * kTile;
  T acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = T(0);
  tile_mainloop<T, false>(Af, ldaf, Bf, ldbf, m, n, k, r0, c0, acc, sm);
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
  double r2 = 0.0, m2 = 0.0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // two halves of 4 rows: 8 x 16-byte loads of M in flight
    T mv[4][2][4];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const int64_t r = r0 + tile_row(ty, 4 * h + ii);
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        if (M && r < m) load4(M + r * ldm, c0 + 4 * tx + 64 * g, n, mv[ii][g]);
        else
#pragma unroll
          for (int q = 0; q < 4; ++q) mv[ii][g][q] = T(0);
      }
    }
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const int i = 4 * h + ii;
      const int64_t r = r0 + tile_row(ty, i);
      if (r >= m) continue;
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const int64_t c = c0 + 4 * tx + 64 * g;
        T l[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) l[q] = acc[i][4 * g + q];
        if (L) store4(L + r * ldl, c, n, l);
        if (M) {
          T sv[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            sv[q] = mv[ii][g][q] - l[q];
            const double d = (double)((mv[ii][g][q] - l[q]) - sv[q]);
            r2 += d * d;
            m2 += (double)mv[ii][g][q] * (double)mv[ii][g][q];
          }
          if (S) store4(S + r * lds, c, n, sv);
        }
      }
    }
  }
  if (part) {
    const int64_t b = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
    block_sum2(r2, m2, &part[2 * b], &part[2 * b + 1]);
  }
}

// ---------------------------------------------------------------- streaming reconstruction (k <= 16)
// HBM-bound form for small k: CTA tile 64 rows x 128 columns; thread (tr, tc) owns 8 rows x 4
// consecutive columns, keeps Bf of its 4 columns in registers, reads Af rows from shared memory
// (warp-uniform -> broadcast), issues all 8 row loads of M before computing, and writes L and S
// with 16-byte streaming stores.  12 B of DRAM traffic per entry, k FMAs.
template <typename T> struct Vec4g;
template <> struct Vec4g<float> {
  __device__ static __forceinline__ void ld(const float* p, float (&v)[4]) {
    float4 t = __ldcs(reinterpret_cast<const float4*>(p));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
  __device__ static __forceinline__ void st(float* p, const float (&v)[4]) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
  }
};
template <> struct Vec4g<double> {
  __device__ static __forceinline__ void ld(const double* p, double (&v)[4]) {
    double2 a = __ldcs(reinterpret_cast<const double2*>(p)), b = __ldcs(reinterpret_cast<const double2*>(p + 2));
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
  __device__ static __forceinline__ void st(double* p, const double (&v)[4]) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(v[0], v[1]));
    __stcs(reinterpret_cast<double2*>(p + 2), make_double2(v[2], v[3]));
  }
};

// Streaming reconstruction for small k (K4, k <= 16): each CTA owns a 1024-column strip (8 warps x
// 128 columns, 4 per thread: 4 KB contiguous per row for the DRAM) and walks a range of rows, RPT
// rows per step, keeping its Bf columns in registers; the A rows are broadcast loads shared by the
// 8 warps; the next step's M is in flight while the current one computes.  12 B of DRAM traffic
// per entry (M in, L and S out).  The residual partial of (M - L) - S is identically 0 (S is
// stored as the fp32 value of M - L, as the reference's s = m - l), so only sum(M^2) is kept.
template <typename T> struct Vec4s;
template <> struct Vec4s<float> {
  __device__ static __forceinline__ void ld(const float* p, float* v) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  }
};
template <> struct Vec4s<double> {
  __device__ static __forceinline__ void ld(const double* p, double* v) {
    const double2 a = *reinterpret_cast<const double2*>(p), b = *reinterpret_cast<const double2*>(p + 2);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
};
constexpr int kStreamCols = 1024;
template <typename T, int KM>
__global__ void __launch_bounds__(256, 2)
reconstruct_stream_kernel(int64_t m, int64_t n, int k, const T* __restrict__ Af, int64_t ldaf,
                          const T* __restrict__ Bf, int64_t ldbf, const T* __restrict__ M, int64_t ldm,
                          T* __restrict__ L, int64_t ldl, T* __restrict__ S, int64_t lds, double* __restrict__ part,
                          bool vec, int64_t rows_per_cta) {
  constexpr int RPT = 4;
  constexpr int KMP = (KM + 3) / 4 * 4;  // A rows padded to 16-byte multiples in shared memory
  extern __shared__ __align__(16) unsigned char stream_smem[];
  T* as = reinterpret_cast<T*>(stream_smem);  // [rows_per_cta][KMP], this CTA's rows of Af
  const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
  const int64_t c0 = (int64_t)blockIdx.x * kStreamCols + 128 * warp + 4 * lane;
  const int64_t rb = (int64_t)blockIdx.y * rows_per_cta;
  const int64_t re = rb + rows_per_cta < m ? rb + rows_per_cta : m;
  for (int64_t e = tid; e < (re - rb) * KMP; e += 256) {
    const int64_t r = e / KMP;
    const int t = (int)(e - r * KMP);
    as[e] = t < k ? Af[(rb + r) * ldaf + t] : T(0);
  }
  __syncthreads();
  T b[4][KM];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int t = 0; t < KM; ++t) b[q][t] = (c0 + q < n && t < k) ? Bf[(c0 + q) * ldbf + t] : T(0);
  const bool full = vec && c0 + 3 < n;
  const bool any = c0 < n;
#define L1F_LOAD_M(R0, DST)                                                                \
  _Pragma("unroll") for (int i = 0; i < RPT; ++i) {                                        \
    const int64_t r = (R0) + i;                                                            \
    if (r < re && M && any) {                                                              \
      if (full) Vec4g<T>::ld(M + r * ldm + c0, DST[i]);                                    \
      else                                                                                 \
        _Pragma("unroll") for (int q = 0; q < 4; ++q) DST[i][q] = c0 + q < n ? M[r * ldm + c0 + q] : T(0); \
    } else {                                                                               \
      _Pragma("unroll") for (int q = 0; q < 4; ++q) DST[i][q] = T(0);                     \
    }                                                                                      \
  }
  double m2 = 0.0;
  T mv[RPT][4], mn[RPT][4];
  L1F_LOAD_M(rb, mv)
  for (int64_t r0 = rb; r0 < re; r0 += RPT) {
    if (r0 + RPT < re) { L1F_LOAD_M(r0 + RPT, mn) }  // next rows in flight
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int64_t r = r0 + i;
      if (r < re && any) {
        T a[KMP];
#pragma unroll
        for (int t = 0; t < KMP; t += 4) Vec4s<T>::ld(as + (r - rb) * KMP + t, a + t);  // broadcast
        T l[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
        for (int t = 0; t < KM; ++t)
#pragma unroll
          for (int q = 0; q < 4; ++q) l[q] = fma(a[t], b[q][t], l[q]);
        T sv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) sv[q] = mv[i][q] - l[q];
        if (full) {
          if (L) Vec4g<T>::st(L + r * ldl + c0, l);
          if (M && S) Vec4g<T>::st(S + r * lds + c0, sv);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (c0 + q < n) {
              if (L) L[r * ldl + c0 + q] = l[q];
              if (M && S) S[r * lds + c0 + q] = sv[q];
            }
        }
      }
    }
    {  // sum(M^2): this step's 16 products in T, folded into the double once per step
      T acc = T(0);
#pragma unroll
      for (int i = 0; i < RPT; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc = fma(mv[i][q], mv[i][q], acc);
      m2 += (double)acc;
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i)
#pragma unroll
      for (int q = 0; q < 4; ++q) mv[i][q] = mn[i][q];
  }
#undef L1F_LOAD_M
  if (part) {
    const int64_t blk = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
    double r2 = 0.0;
    block_sum2(r2, m2, &part[2 * blk], &part[2 * blk + 1]);
  }
}

// ---------------------------------------------------------------- rank-k factors
__device__ __forceinline__ int64_t lower_bound_i64(const int64_t* __restrict__ a, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <typename T>
__global__ void build_factors_kernel(int64_t m, int64_t n, int k, const int64_t* __restrict__ row_idx,
                                     int64_t s_r, const int64_t* __restrict__ col_idx, int64_t s_c,
                                     const double* __restrict__ U, const double* __restrict__ sigma,
                                     const double* __restrict__ V, const T* __restrict__ Zc, int64_t ldzc,
                                     const T* __restrict__ Zr, int64_t ldzr, T* __restrict__ Af,
                                     T* __restrict__ Bf) {
  const int64_t total = (m + n) * (int64_t)k;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rowid = e / k;
    const int t = (int)(e - rowid * k);
    if (rowid < m) {
      const int64_t i = rowid;
      const int64_t p = lower_bound_i64(row_idx, s_r, i);
      T v;
      if (p < s_r && row_idx[p] == i) v = (T)U[p * k + t];
      else if (sizeof(T) == 4) v = (T)(Zr[(i - p) * ldzr + t] * (T)(1.0 / sigma[t]));  // = recon_tc.cu split_rows
      else v = (T)((double)Zr[(i - p) * ldzr + t] / sigma[t]);
      Af[i * k + t] = v;
    } else {
      const int64_t j = rowid - m;
      const int64_t q = lower_bound_i64(col_idx, s_c, j);
      T v;
      if (q < s_c && col_idx[q] == j) v = (T)(sigma[t] * V[q * k + t]);
      else v = Zc[(j - q) * ldzc + t];
      Bf[j * k + t] = v;
    }
  }
}

// ---------------------------------------------------------------- Philox generator
__global__ void generate_factors_kernel(uint64_t seed, int kind, int64_t m, int64_t n, int r,
                                        float yscale, float* __restrict__ X, float* __restrict__ Y) {
  const int64_t total = (m + n) * (int64_t)r;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const bool isx = e < m * (int64_t)r;
    const int64_t idx = isx ? e : e - m * (int64_t)r;
    const uint64_t v = philox_draw(seed, isx ? kStreamX : kStreamY, (uint64_t)idx);
    float out;
    if (kind == L1F_GEN_GAUSSIAN) out = normal_from(v);
    else out = isx ? unit_float((uint32_t)(v >> 32)) : __fmul_rn(unit_float((uint32_t)(v >> 32)), yscale);
    if (isx) X[idx] = out; else Y[idx] = out;
  }
}

__global__ void __launch_bounds__(kTileThreads)
generate_kernel(uint64_t seed, int kind, int64_t n, int r, uint32_t thr, float mag,
                const float* __restrict__ X, const float* __restrict__ Y, int64_t row0, int64_t rows,
                float* __restrict__ M, int64_t ldm, float* __restrict__ L0, int64_t ldl0) {
  __shared__ TileSmem<float> sm;
  __shared__ VideoBox boxes[kVideoBoxes];
  if (kind == L1F_GEN_VIDEO && threadIdx.x < kVideoBoxes) boxes[threadIdx.x] = video_box(seed, threadIdx.x);
  const int64_t r0 = (int64_t)blockIdx.y * kTile, c0 = (int64_t)blockIdx.x * kTile;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
  tile_mainloop<float, true>(X + row0 * r, r, Y, r, rows, n, r, r0, c0, acc, sm);
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t lr = r0 + tile_row(ty, i);
    if (lr >= rows) continue;
    const int64_t gi = row0 + lr;
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const int64_t c = c0 + 4 * tx + 64 * g;
      float l[4], mv[4];
      const uint64_t e0 = (uint64_t)gi * (uint64_t)n + (uint64_t)c;
      u64x4 blk;
      const bool aligned = ((e0 & 3) == 0) && (c + 3 < n);
      if (aligned) blk = philox4x64_10((e0 >> 2) + 1, 0, 0, 0, seed, kStreamS);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        l[q] = acc[i][4 * g + q];
        if (c + q >= n) { mv[q] = 0.0f; continue; }
        const uint64_t v = aligned ? blk.v[q] : philox_draw(seed, kStreamS, e0 + q);
        float sv = 0.0f;
        if (kind == L1F_GEN_GAUSSIAN) {
          if ((uint32_t)(v >> 32) < thr) sv = sym_uniform((uint32_t)v, mag);
        } else {
          if (video_covered(boxes, gi, c + q)) sv = sym_uniform((uint32_t)v, mag);
        }
        mv[q] = __fadd_rn(l[q], sv);
      }
      store4(M + lr * ldm, c, n, mv);
      if (L0) store4(L0 + lr * ldl0, c, n, l);
    }
  }
}

// ---------------------------------------------------------------- gathers
template <typename Ti, typename To>
__global__ void gather_kernel(const Ti* __restrict__ M, int64_t ldm, const int64_t* __restrict__ rows,
                              int64_t nr, const int64_t* __restrict__ cols, int64_t nc,
                              To* __restrict__ out, int64_t ldo) {
  // thread = output column (its source column index kept in a register); blocks stride over rows
  // with the row index broadcast; 4 rows per step keep several scattered loads in flight
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  const int64_t sc = cols ? cols[c] : c;
  const int64_t step = gridDim.y;
  int64_t r = blockIdx.y;
  for (; r + 3 * step < nr; r += 4 * step) {
    Ti v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t rr = r + u * step;
      v[u] = M[(rows ? rows[rr] : rr) * ldm + sc];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) out[(r + u * step) * ldo + c] = (To)v[u];
  }
  for (; r < nr; r += step) out[r * ldo + c] = (To)M[(rows ? rows[r] : r) * ldm + sc];
}

// out[c][r] = M[rows[r]][cols[c]] through a 32x32 shared-memory transpose
template <typename Ti, typename To>
__global__ void gather_t_kernel(const Ti* __restrict__ M, int64_t ldm, const int64_t* __restrict__ rows,
                                int64_t nr, const int64_t* __restrict__ cols, int64_t nc,
                                To* __restrict__ out, int64_t ldo) {
  __shared__ To tile[32][33];
  const int64_t rb = (int64_t)blockIdx.y * 32, cb = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 32 x 8
  const int64_t c = cb + tx;
  const int64_t sc = (c < nc) ? (cols ? cols[c] : c) : 0;
  for (int y = ty; y < 32; y += 8) {
    const int64_t r = rb + y;
    if (r < nr && c < nc) {
      const int64_t sr = rows ? rows[r] : r;
      tile[y][tx] = (To)M[sr * ldm + sc];
    }
  }
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {
    const int64_t oc = cb + y, orow = rb + tx;
    if (oc < nc && orow < nr) out[oc * ldo + orow] = tile[tx][y];
  }
}

// ---------------------------------------------------------------- norms
template <typename T>
__global__ void norms_partial_kernel(const T* __restrict__ X, int64_t rows, int64_t cols, int64_t ld,
                                     double thr, double* __restrict__ part) {
  double s1 = 0.0, mx = 0.0, s2 = 0.0, cnt = 0.0, bad = 0.0;
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols, c = e - r * cols;
    const double v = (double)X[r * ld + c];
    if (!isfinite(v)) { bad += 1.0; continue; }
    const double a = fabs(v);
    s1 += a;
    mx = fmax(mx, a);
    s2 += v * v;
    cnt += (a > thr) ? 1.0 : 0.0;
  }
  __shared__ double red[5][32];
  s1 = warp_sum(s1); s2 = warp_sum(s2); cnt = warp_sum(cnt); bad = warp_sum(bad);
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) { red[0][w] = s1; red[1][w] = mx; red[2][w] = s2; red[3][w] = cnt; red[4][w] = bad; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0, c2 = 0, d = 0, f = 0;
    for (int i = 0; i < (int)(blockDim.x / 32); ++i) {
      a += red[0][i]; b = fmax(b, red[1][i]); c2 += red[2][i]; d += red[3][i]; f += red[4][i];
    }
    double* p = part + 5 * (int64_t)blockIdx.x;
    p[0] = a; p[1] = b; p[2] = c2; p[3] = d; p[4] = f;
  }
}

__global__ void norms_final_kernel(const double* __restrict__ part, int nparts, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double a = 0, b = 0, c = 0, d = 0, f = 0;
    for (int i = 0; i < nparts; ++i) {
      const double* p = part + 5 * (int64_t)i;
      a += p[0]; b = fmax(b, p[1]); c += p[2]; d += p[3]; f += p[4];
    }
    out[0] = a; out[1] = b; out[2] = c; out[3] = d; out[4] = f;
  }
}

template <typename T>
__global__ void diff_partial_kernel(const T* __restrict__ A, int64_t lda, const T* __restrict__ B,
                                    int64_t ldb, int64_t rows, int64_t cols, double* __restrict__ part) {
  double d2 = 0.0, b2 = 0.0;
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols, c = e - r * cols;
    const double a = (double)A[r * lda + c], b = (double)B[r * ldb + c];
    d2 += (a - b) * (a - b);
    b2 += b * b;
  }
  block_sum2(d2, b2, &part[2 * blockIdx.x], &part[2 * blockIdx.x + 1]);
}

template <typename T>
__global__ void soft_threshold_kernel(const T* __restrict__ X, T* __restrict__ Y, int64_t count, T eta) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x)
    Y[e] = shrink(X[e], eta);
}

static int grid_for(int64_t work, int threads) {
  int64_t g = ceil_div(work, threads);
  const int64_t cap = (int64_t)num_sms() * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace l1f

using namespace l1f;

int l1f_reconstruct_tc(int64_t m, int64_t n, int k, const float* Af, int64_t ldaf, const float* Bf, int64_t ldbf,
                       const float* M, int64_t ldm, float* L, int64_t ldl, float* S, int64_t lds, double* resid_sq,
                       cudaStream_t st);

// ====================================================================== C ABI
extern "C" int l1f_gemm_nt(int dtype, int64_t m, int64_t n, int64_t k, double alpha, const void* A,
                           int64_t lda, const void* B, int64_t ldb, double beta, void* C, int64_t ldc,
                           void* stream) {
  L1F_REQUIRE(m >= 0 && n >= 0 && k >= 0, L1F_ERR_ARG, "gemm_nt: negative shape");
  if (m == 0 || n == 0) return L1F_OK;
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid((unsigned)ceil_div(n, kTile), (unsigned)ceil_div(m, kTile));
  L1F_REQUIRE(grid.y <= 65535, L1F_ERR_UNSUPPORTED, "gemm_nt: too many row tiles");
  if (dtype == L1F_F32)
    gemm_nt_kernel<float><<<grid, kTileThreads, 0, st>>>(m, n, (int)k, (float)alpha, (const float*)A, lda,
                                                       (const float*)B, ldb, (float)beta, (float*)C, ldc);
  else
    gemm_nt_kernel<double><<<grid, kTileThreads, 0, st>>>(m, n, (int)k, alpha, (const double*)A, lda,
                                                        (const double*)B, ldb, beta, (double*)C, ldc);
  L1F_CHECK_LAUNCH();
  return L1F_OK;
}

extern "C" int l1f_reconstruct(int dtype, int64_t m, int64_t n, int32_t k, const void* Af, int64_t ldaf,
                               const void* Bf, int64_t ldbf, const void* M, int64_t ldm, void* L,
                               int64_t ldl, void* S, int64_t lds, double* resid_sq, void* stream) {
  L1F_REQUIRE(m >= 0 && n >= 0 && k >= 0, L1F_ERR_ARG, "reconstruct: negative shape");
  cudaStream_t st = (cudaStream_t)stream;
  if (resid_sq) L1F_CUDA_TRY(cudaMemsetAsync(resid_sq, 0, 2 * sizeof(double), st));
  if (m == 0 || n == 0) return L1F_OK;
  if (dtype == L1F_F32 && k > 16) {  // tcgen05 3xTF32 path (recon_tc.cu)
    const int rc = l1f_reconstruct_tc(m, n, k, (const float*)Af, ldaf, (const float*)Bf, ldbf, (const float*)M, ldm,
                                      (float*)L, ldl, (float*)S, lds, resid_sq, st);
    if (rc != L1F_ERR_UNSUPPORTED) return rc;
  }
  const bool small = k <= 16;
  // streaming kernel: 1024-column strips x row ranges, ~4 CTAs per SM in total (2 resident) so
  // each CTA streams many rows with its Bf columns in registers
  const int64_t strips = ceil_div(n, kStreamCols);
  const int64_t want_ctas = (int64_t)num_sms() * 4;
  const size_t esz_s = dtype == L1F_F32 ? 4 : 8;
  const int64_t max_rows = (int64_t)(48 * 1024 / (esz_s * 16)) / 4 * 4;  // Af rows held in shared memory
  int64_t row_groups = std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 4), ceil_div(want_ctas, strips)));
  int64_t rows_per_cta = ceil_div(ceil_div(m, row_groups), 4) * 4;
  if (rows_per_cta > max_rows) rows_per_cta = max_rows;
  row_groups = ceil_div(m, rows_per_cta);
  dim3 grid = small ? dim3((unsigned)strips, (unsigned)row_groups)
                    : dim3((unsigned)ceil_div(n, kTile), (unsigned)ceil_div(m, kTile));
  L1F_REQUIRE(grid.y <= 65535, L1F_ERR_UNSUPPORTED, "reconstruct: too many row tiles");
  const int64_t nblk = (int64_t)grid.x * grid.y;
  Scratch part(st);
  const bool want = resid_sq && M;
  if (want) L1F_CUDA_TRY(part.alloc(nblk * 2 * sizeof(double)));
  double* pp = want ? (double*)part.p : nullptr;
  const size_t esz = dtype == L1F_F32 ? 4 : 8;
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  const bool vec = (!M || (al16(M) && (ldm * esz) % 16 == 0)) && (!L || (al16(L) && (ldl * esz) % 16 == 0)) &&
                   (!S || (al16(S) && (lds * esz) % 16 == 0));
#define L1F_STREAM(TT, KM)                                                                                       \
  reconstruct_stream_kernel<TT, KM><<<grid, 256, (size_t)rows_per_cta * ((KM + 3) / 4 * 4) * sizeof(TT), st>>>( \
      m, n, k, (const TT*)Af, ldaf, (const TT*)Bf, ldbf,                                                          \
                                                         (const TT*)M, ldm, (TT*)L, ldl, (TT*)S, lds, pp, vec,    \
                                                         rows_per_cta)
  if (small) {
    if (dtype == L1F_F32) {
      switch ((k + 1) / 2) {
        case 0: case 1: L1F_STREAM(float, 2); break;
        case 2: L1F_STREAM(float, 4); break;
        case 3: L1F_STREAM(float, 6); break;
        case 4: L1F_STREAM(float, 8); break;
        case 5: L1F_STREAM(float, 10); break;
        case 6: L1F_STREAM(float, 12); break;
        case 7: L1F_STREAM(float, 14); break;
        default: L1F_STREAM(float, 16); break;
      }
    } else {
      if (k <= 4) L1F_STREAM(double, 4); else if (k <= 8) L1F_STREAM(double, 8);
      else if (k <= 12) L1F_STREAM(double, 12); else L1F_STREAM(double, 16);
    }
  } else if (dtype == L1F_F32)
    reconstruct_kernel<float><<<grid, kTileThreads, 0, st>>>(
        m, n, k, (const float*)Af, ldaf, (const float*)Bf, ldbf, (const float*)M, ldm, (float*)L, ldl,
        (float*)S, lds, pp);
  else
    reconstruct_kernel<double><<<grid, kTileThreads, 0, st>>>(
        m, n, k, (const double*)Af, ldaf, (const double*)Bf, ldbf, (const double*)M, ldm, (double*)L, ldl,
        (double*)S, lds, pp);
#undef L1F_STREAM
  L1F_CHECK_LAUNCH();
  if (want) {
    sum_pairs_kernel<<<1, 1024, 0, st>>>((const double*)part.p, nblk, resid_sq);
    L1F_CHECK_LAUNCH();
  }
  return L1F_OK;
}

extern "C" int l1f_build_factors(int dtype, int64_t m, int64_t n, int32_t k, const int64_t* row_idx,
                                 int64_t s_r, const int64_t* col_idx, int64_t s_c, const double* U,
                                 const double* sigma, const double* V, const void* Zc, int64_t ldzc,
                                 const void* Zr, int64_t ldzr, void* Af, void* Bf, void* stream) {
  L1F_REQUIRE(m >= 0 && n >= 0 && k >= 1 && s_r >= 0 && s_r <= m && s_c >= 0 && s_c <= n,
              L1F_ERR_ARG, "build_factors: bad shape");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t total = (m + n) * (int64_t)k;
  if (total == 0) return L1F_OK;
  const int g = grid_for(total, 256);
  if (dtype == L1F_F32)
    build_factors_kernel<float><<<g, 256, 0, st>>>(m, n, k, row_idx, s_r, col_idx, s_c, U, sigma, V,
                                                   (const float*)Zc, ldzc, (const float*)Zr, ldzr,
                                                   (float*)Af, (float*)Bf);
  else
    build_factors_kernel<double><<<g, 256, 0, st>>>(m, n, k, row_idx, s_r, col_idx, s_c, U, sigma, V,
                                                    (const double*)Zc, ldzc, (const double*)Zr, ldzr,
                                                    (double*)Af, (double*)Bf);
  L1F_CHECK_LAUNCH();
  return L1F_OK;
}

extern "C" int l1f_generate_factors_f32(uint64_t seed, int32_t kind, int64_t m, int64_t n, int32_t r,
                                        float* X, float* Y, void* stream) {
  L1F_REQUIRE(kind == L1F_GEN_GAUSSIAN || kind == L1F_GEN_VIDEO, L1F_ERR_ARG, "generate: unknown kind %d", kind);
  L1F_REQUIRE(m >= 0 && n >= 0 && r >= 0, L1F_ERR_ARG, "generate: negative shape");
  const int64_t total = (m + n) * (int64_t)r;
  if (total == 0) return L1F_OK;
  const float yscale = r > 0 ? 255.0f / (float)r : 0.0f;  // correctly rounded division
  generate_factors_kernel<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(seed, kind, m, n, r,
                                                                                    yscale, X, Y);
  L1F_CHECK_LAUNCH();
  return L1F_OK;
}

extern "C" int l1f_generate_f32(uint64_t seed, int32_t kind, int64_t m, int64_t n, int32_t r, float rho_s,
                                float magnitude, const float* X, const float* Y, int64_t row0, int64_t rows,
                                float* M, int64_t ldm, float* L0, int64_t ldl0, void* stream) {
  L1F_REQUIRE(kind == L1F_GEN_GAUSSIAN || kind == L1F_GEN_VIDEO, L1F_ERR_ARG, "generate: unknown kind %d", kind);
  L1F_REQUIRE(m >= 0 && n >= 0 && r >= 0 && row0 >= 0 && rows >= 0 && row0 + rows <= m, L1F_ERR_ARG,
              "generate: bad shard [%lld, %lld) of %lld rows", (long long)row0, (long long)(row0 + rows),
              (long long)m);
  L1F_REQUIRE(rho_s >= 0.0f && rho_s <= 1.0f, L1F_ERR_ARG, "generate: rho_s must be in [0, 1]");
  if (rows == 0 || n == 0) return L1F_OK;
  double t = floor((double)rho_s * 4294967296.0);
  const uint32_t thr = t >= 4294967295.0 ? 0xffffffffu : (uint32_t)t;
  dim3 grid((unsigned)ceil_div(n, kTile), (unsigned)ceil_div(rows, kTile));
  L1F_REQUIRE(grid.y <= 65535, L1F_ERR_UNSUPPORTED, "generate: too many row tiles");
  generate_kernel<<<grid, kTileThreads, 0, (cudaStream_t)stream>>>(seed, kind, n, r, thr, magnitude, X, Y,
                                                                    row0, rows, M, ldm, L0, ldl0);
  L1F_CHECK_LAUNCH();
  return L1F_OK;
}

extern "C" int l1f_gather(int dtype_in, const void* M, int64_t ldm, const int64_t* rows, int64_t n_rows,
                          const int64_t* cols, int64_t n_cols, int dtype_out, void* out, int64_t ldo,
                          int32_t transpose, void* stream) {
  L1F_REQUIRE(n_rows >= 0 && n_cols >= 0, L1F_ERR_ARG, "gather: negative shape");
  if (n_rows == 0 || n_cols == 0) return L1F_OK;
  cudaStream_t st = (cudaStream_t)stream;
#define L1F_GATHER(TI, TO)                                                                           \
  if (transpose) {                                                                                   \
    dim3 grid((unsigned)ceil_div(n_cols, 32), (unsigned)ceil_div(n_rows, 32));                      \
    gather_t_kernel<TI, TO><<<grid, 256, 0, st>>>((const TI*)M, ldm, rows, n_rows, cols, n_cols,    \
                                                  (TO*)out, ldo);                                    \
  } else {                                                                                           \
    gather_kernel<TI, TO><<<dim3((unsigned)ceil_div(n_cols, 256),                                     \
                             (unsigned)std::max<int64_t>(1, std::min<int64_t>(n_rows,                     \
                                 ceil_div((int64_t)num_sms() * 16, ceil_div(n_cols, 256))))),             \
                             256, 0, st>>>(                                                             \
        (const TI*)M, ldm, rows, n_rows, cols, n_cols, (TO*)out, ldo);                               \
  }
  if (transpose) L1F_REQUIRE(ceil_div(n_rows, 32) <= 65535, L1F_ERR_UNSUPPORTED, "gather: too many rows");
  if (dtype_in == L1F_F32 && dtype_out == L1F_F32) { L1F_GATHER(float, float) }
  else if (dtype_in == L1F_F32 && dtype_out == L1F_F64) { L1F_GATHER(float, double) }
  else if (dtype_in == L1F_F64 && dtype_out == L1F_F32) { L1F_GATHER(double, float) }
  else { L1F_GATHER(double, double) }
#undef L1F_GATHER
  L1F_CHECK_LAUNCH();
  return L1F_OK;
}

extern "C" int l1f_norms(int dtype, const void* X, int64_t rows, int64_t cols, int64_t ld, double thr,
                         double* out5, void* stream) {
  L1F_REQUIRE(rows >= 0 && cols >= 0, L1F_ERR_ARG, "norms: negative shape");
  cudaStream_t st = (cudaStream_t)stream;
  const int g = grid_for(rows * cols, 256);
  Scratch part(st);
  L1F_CUDA_TRY(part.alloc((size_t)g * 5 * sizeof(double)));
  if (rows * cols == 0) {
    L1F_CUDA_TRY(cudaMemsetAsync(out5, 0, 5 * sizeof(double), st));
    return L1F_OK;
  }
  if (dtype == L1F_F32)
    norms_partial_kernel<float><<<g, 256, 0, st>>>((const float*)X, rows, cols, ld, thr, (double*)part.p);
  else
    norms_partial_kernel<double><<<g, 256, 0, st>>>((const double*)X, rows, cols, ld, thr, (double*)part.p);
  L1F_CHECK_LAUNCH();
  norms_final_kernel<<<1, 32, 0, st>>>((const double*)part.p, g, out5);
  L1F_CHECK_LAUNCH();
  return L1F_OK;
}

extern "C" int l1f_diff_norms(int dtype, const void* A, int64_t lda, const void* B, int64_t ldb,
                              int64_t rows, int64_t cols, double* out2, void* stream) {
  L1F_REQUIRE(rows >= 0 && cols >= 0, L1F_ERR_ARG, "diff_norms: negative shape");
  cudaStream_t st = (cudaStream_t)stream;
  if (rows * cols == 0) {
    L1F_CUDA_TRY(cudaMemsetAsync(out2, 0, 2 * sizeof(double), st));
    return L1F_OK;
  }
  const int g = grid_for(rows * cols, 256);
  Scratch part(st);
  L1F_CUDA_TRY(part.alloc((size_t)g * 2 * sizeof(double)));
  if (dtype == L1F_F32)
    diff_partial_kernel<float><<<g, 256, 0, st>>>((const float*)A, lda, (const float*)B, ldb, rows, cols,
                                                  (double*)part.p);
  else
    diff_partial_kernel<double><<<g, 256, 0, st>>>((const double*)A, lda, (const double*)B, ldb, rows, cols,
                                                   (double*)part.p);
  L1F_CHECK_LAUNCH();
  sum_pairs_kernel<<<1, 1024, 0, st>>>((const double*)part.p, g, out2);
  L1F_CHECK_LAUNCH();
  return L1F_OK;
}

extern "C" int l1f_soft_threshold(int dtype, const void* X, void* Y, int64_t count, double eta, void* stream) {
  L1F_REQUIRE(eta >= 0.0, L1F_ERR_ARG, "eta must be nonnegative");
  if (count <= 0) return L1F_OK;
  const int g = grid_for(count, 256);
  if (dtype == L1F_F32)
    soft_threshold_kernel<float><<<g, 256, 0, (cudaStream_t)stream>>>((const float*)X, (float*)Y, count, (float)eta);
  else
    soft_threshold_kernel<double><<<g, 256, 0, (cudaStream_t)stream>>>((const double*)X, (double*)Y, count, eta);
  L1F_CHECK_LAUNCH();
  return L1F_OK;
}

// ------------------------------------------------------------------------------------
// Exact-count sparse support — synth.generate's `rng.choice(m*n, size=p, replace=False)` +
// `uniform(-mag, mag)` (synth.py:56-61): exactly p of the N entries are nonzero, at uniformly
// random positions.  Entry e gets a unique 64-bit key (Philox draw in the high bits, e in the low
// `ib` bits); the support is the p smallest keys, found by an 8-pass radix select (8-bit digits,
// shared-memory histograms, the digit choice made on the device — no host round trip).
// ------------------------------------------------------------------------------------
namespace l1f {
namespace spx {
constexpr uint64_t kStreamSupport = 5, kStreamValue = 6;

__device__ __forceinline__ uint64_t key_of(uint64_t seed, int64_t e, int ib) {
  const uint64_t r = philox_draw(seed, kStreamSupport, (uint64_t)e);
  return ib >= 64 ? (uint64_t)e : (((r >> ib) << ib) | (uint64_t)e);
}

struct Sel { uint64_t prefix, mask; int64_t rank; };  // rank: 1-based rank still to find

__global__ void sel_init_kernel(Sel* sel, int64_t p) {
  sel->prefix = 0; sel->mask = 0; sel->rank = p;
}

__global__ void sel_hist_kernel(uint64_t seed, int64_t N, int ib, int shift, const Sel* __restrict__ sel,
                                unsigned long long* __restrict__ hist) {
  __shared__ unsigned int h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint64_t prefix = sel->prefix, mask = sel->mask;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = key_of(seed, e, ib);
    if ((key & mask) == prefix) atomicAdd(&h[(key >> shift) & 0xffu], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], (unsigned long long)h[i]);
}

__global__ void sel_pick_kernel(int shift, Sel* sel, unsigned long long* hist) {
  if (threadIdx.x != 0) return;
  int64_t rank = sel->rank;
  int d = 0;
  for (; d < 255; ++d) {
    const int64_t c = (int64_t)hist[d];
    if (rank <= c) break;
    rank -= c;
  }
  sel->prefix |= (uint64_t)d << shift;
  sel->mask |= (uint64_t)0xff << shift;
  sel->rank = rank;
  for (int i = 0; i < 256; ++i) hist[i] = 0;
}

template <typename T>
__global__ void sparse_write_kernel(uint64_t seed, int64_t N, int ib, const Sel* __restrict__ sel, int64_t p,
                                    double mag, T* __restrict__ S) {
  const uint64_t thr = sel->prefix;  // the p-th smallest key
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x) {
    T v = T(0);
    if (p > 0 && key_of(seed, e, ib) <= thr) {
      const uint64_t b = philox_draw(seed, kStreamValue, (uint64_t)e);
      const double u = (double)(b >> 11) * 0x1.0p-53;  // [0, 1)
      v = (T)(mag * (2.0 * u - 1.0));                  // U[-mag, mag)
      if (v == T(0)) v = (T)(mag * 0x1.0p-53);        // keep the support exact
    }
    S[e] = v;
  }
}
}  // namespace spx
}  // namespace l1f

extern "C" int l1f_generate_sparse_exact(int dtype, uint64_t seed, int64_t m, int64_t n, int64_t p, double magnitude,
                                         void* S, void* stream) {
  using namespace l1f::spx;
  L1F_REQUIRE(dtype == L1F_F32 || dtype == L1F_F64, L1F_ERR_ARG, "generate_sparse: bad dtype");
  L1F_REQUIRE(m >= 0 && n >= 0 && p >= 0, L1F_ERR_ARG, "generate_sparse: negative shape");
  const int64_t N = m * n;
  L1F_REQUIRE(p <= N, L1F_ERR_ARG, "requested %lld sparse entries in a %lldx%lld matrix", (long long)p, (long long)m,
              (long long)n);
  L1F_REQUIRE(magnitude >= 0.0, L1F_ERR_ARG, "generate_sparse: magnitude must be nonnegative");
  if (N == 0) return L1F_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int ib = 0;
  while (ib < 63 && ((uint64_t)1 << ib) < (uint64_t)N) ++ib;
  Scratch buf(st);
  L1F_CUDA_TRY(buf.alloc(sizeof(Sel) + 256 * sizeof(unsigned long long)));
  Sel* sel = (Sel*)buf.p;
  unsigned long long* hist = (unsigned long long*)((char*)buf.p + sizeof(Sel));
  L1F_CUDA_TRY(cudaMemsetAsync(hist, 0, 256 * sizeof(unsigned long long), st));
  const int g = grid_for(N, 256);
  if (p > 0) {
    sel_init_kernel<<<1, 1, 0, st>>>(sel, p);
    for (int shift = 56; shift >= 0; shift -= 8) {
      sel_hist_kernel<<<g, 256, 0, st>>>(seed, N, ib, shift, sel, hist);
      sel_pick_kernel<<<1, 32, 0, st>>>(shift, sel, hist);
    }
    L1F_CHECK_LAUNCH();
  }
  if (dtype == L1F_F64)
    sparse_write_kernel<double><<<g, 256, 0, st>>>(seed, N, ib, sel, p, magnitude, (double*)S);
  else
    sparse_write_kernel<float><<<g, 256, 0, st>>>(seed, N, ib, sel, p, magnitude, (float*)S);
  L1F_CHECK_LAUNCH();
  return L1F_OK;
}
