// 128x128 CTA tile, 8x8-per-thread register tile SIMT GEMM mainloop for the rank-k
// products of the path (C = A B^T with K = k <= a few hundred).  Used by the
// reconstruction L = Af Bf^T (l1filter.py:137-167 unified), the generator's L0 = X Y^T
// (synth.py:54) and the small dense products of the reference API.
//
// Thread (ty, tx) = (tid/16, tid%16) owns rows {4ty..4ty+3, 64+4ty..64+4ty+3} and columns
// {4tx..4tx+3, 64+4tx..64+4tx+3} of the tile.  Each k-step loads two float4 of A and two
// of B from shared memory for 64 FMAs.  With EXACT, every product and sum is separately
// rounded (no FMA contraction) in k order so the numpy oracle reproduces L0 bit for bit.
#pragma once
#include "common.cuh"

namespace l1f {

constexpr int kTile = 128;
constexpr int kTileK = 8;
constexpr int kTilePad = 4;
constexpr int kTileThreads = 256;

template <typename T>
struct TileSmem {
  T a[kTileK][kTile + kTilePad];
  T b[kTileK][kTile + kTilePad];
};

template <typename T> __device__ __forceinline__ T mul_rn(T a, T b);
template <> __device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
template <typename T> __device__ __forceinline__ T add_rn(T a, T b);
template <> __device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

__device__ __forceinline__ int tile_row(int ty, int i) { return (i < 4) ? 4 * ty + i : 64 + 4 * ty + (i - 4); }

// acc[i][j] += sum_t A[r0+row(i)][t] * B[c0+col(j)][t]
template <typename T, bool EXACT>
__device__ __forceinline__ void tile_mainloop(const T* __restrict__ A, int64_t lda,
                                              const T* __restrict__ B, int64_t ldb,
                                              int64_t m, int64_t n, int k, int64_t r0,
                                              int64_t c0, T (&acc)[8][8], TileSmem<T>& sm) {
  const int tid = threadIdx.x;
  const int ty = tid / 16, tx = tid % 16;
  // loader mapping: row lr = tid/2 (0..127), k offset lk = (tid%2)*4
  const int lr = tid >> 1, lk = (tid & 1) * 4;
  for (int k0 = 0; k0 < k; k0 += kTileK) {
    {
      const int64_t ar = r0 + lr, bc = c0 + lr;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int kk = k0 + lk + q;
        T av = T(0), bv = T(0);
        if (kk < k) {
          if (ar < m) av = A[ar * lda + kk];
          if (bc < n) bv = B[bc * ldb + kk];
        }
        sm.a[lk + q][lr] = av;
        sm.b[lk + q][lr] = bv;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kTileK; ++kk) {
      T a[8], b[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = sm.a[kk][4 * ty + q];
        a[4 + q] = sm.a[kk][64 + 4 * ty + q];
        b[q] = sm.b[kk][4 * tx + q];
        b[4 + q] = sm.b[kk][64 + 4 * tx + q];
      }
      if (EXACT) {
        // padded k-steps must not touch the accumulator: x + 0*0 could flip -0.0
        if (k0 + kk < k) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = add_rn(acc[i][j], mul_rn(a[i], b[j]));
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      }
    }
    __syncthreads();
  }
}

}  // namespace l1f
