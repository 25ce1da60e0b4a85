// Counter-based Philox4x64-10 and the float transforms of the synthetic-input generator.
//
// Replaces the PCG64 draws of synth.generate (pkg/src/l1pcp/synth.py:43-64).  Block b of
// stream (seed, stream_id) is philox(counter = {b+1, 0, 0, 0}, key = {seed, stream_id}),
// which is exactly what numpy.random.Philox(key=[seed, stream_id], counter=[b,0,0,0])
// emits first (numpy pre-increments its counter); the oracle uses that bit generator.
// Every float transform below uses only separately rounded IEEE operations
// (__fadd_rn/__fmul_rn/__fdiv_rn/__fsqrt_rn, never a contracted FMA), so a numpy float32
// restatement of the same operation sequence reproduces each value bit for bit.
#pragma once
#include <stdint.h>

namespace l1f {

enum : uint64_t { kStreamX = 1, kStreamY = 2, kStreamS = 3, kStreamBox = 4 };
constexpr int kVideoW = 320, kVideoH = 240, kVideoBoxes = 6;

struct u64x4 { uint64_t v[4]; };

__host__ __device__ __forceinline__ void mulhilo64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
#ifdef __CUDA_ARCH__
  lo = a * b;
  hi = __umul64hi(a, b);
#else
  unsigned __int128 p = (unsigned __int128)a * b;
  lo = (uint64_t)p;
  hi = (uint64_t)(p >> 64);
#endif
}

__host__ __device__ __forceinline__ u64x4 philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2,
                                                        uint64_t c3, uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += W0; k1 += W1; }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(M0, c0, hi0, lo0);
    mulhilo64(M1, c2, hi1, lo1);
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  u64x4 o; o.v[0] = c0; o.v[1] = c1; o.v[2] = c2; o.v[3] = c3;
  return o;
}

// raw 64-bit draw number e of a stream
__device__ __forceinline__ uint64_t philox_draw(uint64_t seed, uint64_t stream, uint64_t e) {
  u64x4 o = philox4x64_10((e >> 2) + 1, 0, 0, 0, seed, stream);
  return o.v[e & 3];
}

// [0,1) with 24 random bits
__device__ __forceinline__ float unit_float(uint32_t b) {
  return __fmul_rn((float)(b >> 8), 5.9604644775390625e-08f);
}
// U[-mag, mag)
__device__ __forceinline__ float sym_uniform(uint32_t b, float mag) {
  return __fmul_rn(mag, __fsub_rn(__fmul_rn(2.0f, unit_float(b)), 1.0f));
}

// natural log of u in (0, 1] via the atanh series on [sqrt(1/2), sqrt(2))
__device__ __forceinline__ float exact_log(float u) {
  uint32_t bits = __float_as_uint(u);
  int e = (int)((bits >> 23) & 0xffu) - 127;
  float f = __uint_as_float((bits & 0x7fffffu) | 0x3f800000u);
  if (f > 1.41421353816986083984375f) { f = __fmul_rn(f, 0.5f); e += 1; }
  float s = __fdiv_rn(__fsub_rn(f, 1.0f), __fadd_rn(f, 1.0f));
  float s2 = __fmul_rn(s, s);
  float p = 0.0909090936183929443359375f;                       // 1/11
  p = __fadd_rn(__fmul_rn(p, s2), 0.111111111938953399658203125f);  // 1/9
  p = __fadd_rn(__fmul_rn(p, s2), 0.14285714924335479736328125f);   // 1/7
  p = __fadd_rn(__fmul_rn(p, s2), 0.20000000298023223876953125f);   // 1/5
  p = __fadd_rn(__fmul_rn(p, s2), 0.3333333432674407958984375f);    // 1/3
  p = __fadd_rn(__fmul_rn(p, s2), 1.0f);
  float lnf = __fmul_rn(__fmul_rn(2.0f, s), p);
  return __fadd_rn(__fmul_rn((float)e, 0.693147182464599609375f), lnf);
}

// cos(2*pi*t) for t in [0,1): quadrant split, Taylor polynomials on [0, pi/2)
__device__ __forceinline__ float exact_cos2pi(float t) {
  float t4 = __fmul_rn(t, 4.0f);
  float qf = floorf(t4);
  int q = (int)qf;
  float th = __fmul_rn(__fsub_rn(t4, qf), 1.57079637050628662109375f);
  float x = __fmul_rn(th, th);
  float c = 2.08767570e-09f;                                  // 1/12!
  c = __fadd_rn(__fmul_rn(c, x), -2.75573188e-07f);           // -1/10!
  c = __fadd_rn(__fmul_rn(c, x), 2.48015876e-05f);            // 1/8!
  c = __fadd_rn(__fmul_rn(c, x), -1.38888892e-03f);           // -1/6!
  c = __fadd_rn(__fmul_rn(c, x), 4.16666679e-02f);            // 1/4!
  c = __fadd_rn(__fmul_rn(c, x), -0.5f);
  c = __fadd_rn(__fmul_rn(c, x), 1.0f);
  float sn = 1.60590444e-10f;                                 // 1/13!
  sn = __fadd_rn(__fmul_rn(sn, x), -2.50521079e-08f);         // -1/11!
  sn = __fadd_rn(__fmul_rn(sn, x), 2.75573188e-06f);          // 1/9!
  sn = __fadd_rn(__fmul_rn(sn, x), -1.98412701e-04f);         // -1/7!
  sn = __fadd_rn(__fmul_rn(sn, x), 8.33333377e-03f);          // 1/5!
  sn = __fadd_rn(__fmul_rn(sn, x), -0.166666672f);            // -1/3!
  sn = __fadd_rn(__fmul_rn(sn, x), 1.0f);
  sn = __fmul_rn(th, sn);
  return q == 0 ? c : (q == 1 ? -sn : (q == 2 ? -c : sn));
}

// one N(0,1) draw from one 64-bit word (Box-Muller, cosine branch)
__device__ __forceinline__ float normal_from(uint64_t v) {
  uint32_t hi = (uint32_t)(v >> 32), lo = (uint32_t)v;
  float u1 = __fmul_rn((float)((hi >> 8) + 1u), 5.9604644775390625e-08f);
  float u2 = unit_float(lo);
  float rad = __fsqrt_rn(__fmul_rn(-2.0f, exact_log(u1)));
  return __fmul_rn(rad, exact_cos2pi(u2));
}

struct VideoBox { int w, h, x0, y0, vx, vy; };

__host__ __device__ __forceinline__ VideoBox video_box(uint64_t seed, int b) {
  u64x4 o = philox4x64_10((uint64_t)b + 1, 0, 0, 0, seed, kStreamBox);
  VideoBox B;
  B.w = 10 + (int)((o.v[0] >> 32) % 31u);
  B.h = 10 + (int)((o.v[0] & 0xffffffffu) % 31u);
  B.x0 = (int)((o.v[1] >> 32) % (uint64_t)kVideoW);
  B.y0 = (int)((o.v[1] & 0xffffffffu) % (uint64_t)kVideoH);
  B.vx = (int)((o.v[2] >> 32) % 7u) - 3;
  B.vy = (int)((o.v[2] & 0xffffffffu) % 7u) - 3;
  return B;
}

__host__ __device__ __forceinline__ int pos_mod(int64_t a, int m) {
  int64_t r = a % m;
  return (int)(r < 0 ? r + m : r);
}

// is pixel i (row-major 240x320 frame) of frame f covered by a moving box?
__device__ __forceinline__ bool video_covered(const VideoBox* boxes, int64_t i, int64_t f) {
  int px = (int)(i % kVideoW), py = (int)(i / kVideoW);
  bool hit = false;
#pragma unroll
  for (int b = 0; b < kVideoBoxes; ++b) {
    const VideoBox& B = boxes[b];
    int bx = pos_mod((int64_t)B.x0 + (int64_t)B.vx * f, kVideoW);
    int by = pos_mod((int64_t)B.y0 + (int64_t)B.vy * f, kVideoH);
    hit |= (pos_mod(px - bx, kVideoW) < B.w) && (pos_mod(py - by, kVideoH) < B.h);
  }
  return hit;
}

}  // namespace l1f
