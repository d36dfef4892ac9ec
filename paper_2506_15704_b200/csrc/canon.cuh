// canon.cuh -- the canonical device arithmetic.
//
// Every helper here is a fixed IEEE-754 op sequence with explicit _rn
// intrinsics (never contracted into FMA), restated op for op by
// oracle/devmath.py so that index sets, table entries and scalars computed
// on the GPU can be checked bit for bit.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace lfps {

__device__ __forceinline__ double cadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double csub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double cmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double cdiv(double a, double b) { return __ddiv_rn(a, b); }

// a / n for a count n > 0: when n is a power of two the quotient is the
// exact product a * 2^-k (same correctly rounded value as the division, far
// cheaper than the division sequence); otherwise a true IEEE division.
__device__ __forceinline__ double cdiv_count(double a, double n) {
  const long long b = __double_as_longlong(n);
  if ((b & 0x000FFFFFFFFFFFFFll) == 0) return __dmul_rn(a, __longlong_as_double(0x7FE0000000000000ll - b));
  return __ddiv_rn(a, n);
}

// Constants as exact bit patterns (equal to the Python doubles in
// oracle/devmath.py: LN2_HI/LN2_LO fdlibm split, 1/ln2, 1.0/math.factorial(i)).
__device__ __forceinline__ double dbits(unsigned long long b) { return __longlong_as_double((long long)b); }

// exp(x) from +,-,*,rint and an exact power-of-two scale; 0 below -708.
// devmath.cexp: k = rint(x / ln2), r = (x - k LN2_HI) - k LN2_LO, Horner
// Taylor of degree 13, times 2^k.
__device__ __forceinline__ double cexp(double x) {
  if (x < -708.0) return 0.0;
  const double k = rint(cmul(x, dbits(0x3ff71547652b82feull)));
  const double r = csub(csub(x, cmul(k, dbits(0x3fe62e42fee00000ull))),
                        cmul(k, dbits(0x3dea39ef35793c76ull)));
  double p = dbits(0x3de6124613a86d09ull);               // 1/13!
  p = cadd(cmul(p, r), dbits(0x3e21eed8eff8d898ull));    // 1/12!
  p = cadd(cmul(p, r), dbits(0x3e5ae64567f544e4ull));    // 1/11!
  p = cadd(cmul(p, r), dbits(0x3e927e4fb7789f5cull));    // 1/10!
  p = cadd(cmul(p, r), dbits(0x3ec71de3a556c734ull));    // 1/9!
  p = cadd(cmul(p, r), dbits(0x3efa01a01a01a01aull));    // 1/8!
  p = cadd(cmul(p, r), dbits(0x3f2a01a01a01a01aull));    // 1/7!
  p = cadd(cmul(p, r), dbits(0x3f56c16c16c16c17ull));    // 1/6!
  p = cadd(cmul(p, r), dbits(0x3f81111111111111ull));    // 1/5!
  p = cadd(cmul(p, r), dbits(0x3fa5555555555555ull));    // 1/4!
  p = cadd(cmul(p, r), dbits(0x3fc5555555555555ull));    // 1/3!
  p = cadd(cmul(p, r), 0.5);
  p = cadd(cmul(p, r), 1.0);
  p = cadd(cmul(p, r), 1.0);
  const long long e = (long long)k + 1023;
  return cmul(p, __longlong_as_double(e << 52));
}

// Butterfly fold over a full warp: v[i] + v[i ^ h], h = 16..1.
__device__ __forceinline__ double warp_fold(double v) {
#pragma unroll
  for (int h = 16; h >= 1; h >>= 1) v = cadd(v, __shfl_xor_sync(0xffffffffu, v, h));
  return v;
}

// Adjacent-pair tree over 16 lane-resident values (devmath.table_sum):
// ((v0+v1)+(v2+v3)) + ... ; depth 4 instead of a 16-long dependent chain.
__device__ __forceinline__ double lane_tree16(double* v) {
#pragma unroll
  for (int h = 1; h < 16; h <<= 1) {
#pragma unroll
    for (int k = 0; k < 16; k += 2 * h) v[k] = cadd(v[k], v[k + h]);
  }
  return v[0];
}

// Fold within 16-lane halves: h = 8..1 (fp32, score dots).
__device__ __forceinline__ float half_fold(float v) {
#pragma unroll
  for (int h = 8; h >= 1; h >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, h));
  return v;
}

// In-place adjacent-pair tree over buf[0, n2) (n2 a power of two, >= 1)
// executed by one warp; returns buf[0].  devmath._pairwise_tree.
__device__ __forceinline__ double warp_pairwise_tree(double* buf, int n2, int lane) {
  for (int len = n2; len > 1; len >>= 1) {
    const int half = len >> 1;
    for (int i0 = 0; i0 < half; i0 += 32) {
      const int i = i0 + lane;
      double a = 0.0, b = 0.0;
      if (i < half) { a = buf[2 * i]; b = buf[2 * i + 1]; }
      __syncwarp();
      if (i < half) buf[i] = cadd(a, b);
      __syncwarp();
    }
  }
  return buf[0];
}

// Canonical 256-thread block sum (devmath.block_sum) of per-thread partial
// accumulators; `red` is a 9-entry shared scratch.  All threads get it.
__device__ __forceinline__ double block_fold256(double acc, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  acc = warp_fold(acc);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  double v = (lane < 8) ? red[lane] : 0.0;
  if (warp == 0) {
    // fold 4, 2, 1 over the 8 warp sums
#pragma unroll
    for (int h = 4; h >= 1; h >>= 1) v = cadd(v, __shfl_xor_sync(0xffffffffu, v, h));
    if (lane == 0) red[8] = v;
  }
  __syncthreads();
  const double out = red[8];
  __syncthreads();
  return out;
}

// bf16 helpers
__device__ __forceinline__ float bf2f(uint16_t b) {
  return __uint_as_float(((uint32_t)b) << 16);
}

// Order-preserving map of an fp32 score to uint32 (larger float -> larger
// key); -0.0 is canonicalised to +0.0 so they tie (attention.py:40-45).
__device__ __forceinline__ uint32_t score_key(float f) {
  uint32_t u = __float_as_uint(f);
  if (u == 0x80000000u) u = 0u;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

}  // namespace lfps
