// arith_probe.cu -- one-off B200 checks behind two score-path rewrites
// (results recorded in profiles/r01_arith_probe.txt):
//   1. fma.rn.f32.bf16 (FHFMA.BF16) == fma.rn.f32 of the exactly widened
//      operands, over random and edge bit patterns (incl. subnormals);
//   2. v / c == q1 for q0 = v * r, e = fma(-q0, c, v), q1 = fma(e, r, q0),
//      r = RN(1 / c), over ALL 2^32 v, c = fp32(sqrt d), d = 32, 64, 128, 256;
//   3. issue throughput of FHFMA.BF16 vs FFMA2 vs FFMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o arith_probe arith_probe.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ float fmab_lo(uint32_t a, uint32_t b, float c) {
  float d; unsigned short al, ah, bl, bh;
  asm("mov.b32 {%0,%1}, %2;" : "=h"(al), "=h"(ah) : "r"(a));
  asm("mov.b32 {%0,%1}, %2;" : "=h"(bl), "=h"(bh) : "r"(b));
  asm("fma.rn.f32.bf16 %0, %1, %2, %3;" : "=f"(d) : "h"(al), "h"(bl), "f"(c));
  return d;
}
__device__ __forceinline__ uint32_t hash(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return (uint32_t)x;
}
__global__ void k_fhfma(uint64_t n, unsigned long long* bad) {
  unsigned long long loc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t a = hash(3 * i) & 0xffff, b = hash(3 * i + 1) & 0xffff, cbits = hash(3 * i + 2);
    if (i & 1) { a &= 0x80ff; a |= (hash(i) & 0x7) << 7; }      // tiny / subnormal bf16
    if (i & 2) cbits &= 0x807fffffu;                               // subnormal accumulator
    const float c = __uint_as_float(cbits);
    if (isnan(c)) continue;
    const float x = __uint_as_float(a << 16), y = __uint_as_float(b << 16);
    if (isnan(x) || isnan(y)) continue;
    const float r0 = __fmaf_rn(x, y, c);
    const float r1 = fmab_lo(a, b, c);
    if (__float_as_uint(r0) != __float_as_uint(r1) && !(isnan(r0) && isnan(r1))) ++loc;
  }
  if (loc) atomicAdd(bad, loc);
}
__global__ void k_div(float c, float r, unsigned long long* bad, unsigned long long* first) {
  unsigned long long loc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (1ull << 32); i += (uint64_t)gridDim.x * blockDim.x) {
    const float v = __uint_as_float((uint32_t)i);
    if (isnan(v)) continue;
    const float q0 = __fmul_rn(v, r);
    const float e = __fmaf_rn(-q0, c, v);
    const float q1 = (e == e) ? __fmaf_rn(e, r, q0) : q0;
    const float ref = __fdiv_rn(v, c);
    if (__float_as_uint(q1) != __float_as_uint(ref)) { ++loc; atomicMin(first, i); }
  }
  if (loc) atomicAdd(bad, loc);
}
template <int MODE>
__global__ void k_tput(float* out, int iters) {
  uint32_t w[8]; float acc[8]; float2 a2[4];
  for (int j = 0; j < 8; ++j) { w[j] = 0x3f803f80u + threadIdx.x + j; acc[j] = 0.f; }
  for (int j = 0; j < 4; ++j) a2[j] = make_float2(0.f, 0.f);
  const float2 k2 = make_float2(1.0001f, 0.9999f), q2 = make_float2(0.5f, 0.25f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) acc[j] = fmab_lo(w[j], w[(j + 1) & 7], acc[j]);
      else if (MODE == 1) acc[j] = __fmaf_rn(acc[j], 1.0001f, 0.5f);
    }
    if (MODE == 2) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        unsigned long long r, aa, bb, cc;
        asm("mov.b64 %0, {%1,%2};" : "=l"(aa) : "f"(k2.x), "f"(k2.y));
        asm("mov.b64 %0, {%1,%2};" : "=l"(bb) : "f"(q2.x), "f"(q2.y));
        asm("mov.b64 %0, {%1,%2};" : "=l"(cc) : "f"(a2[j].x), "f"(a2[j].y));
        asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(aa), "l"(bb), "l"(cc));
        asm("mov.b64 {%0,%1}, %2;" : "=f"(a2[j].x), "=f"(a2[j].y) : "l"(r));
      }
    }
  }
  float s = 0.f;
  for (int j = 0; j < 8; ++j) s += acc[j];
  for (int j = 0; j < 4; ++j) s += a2[j].x + a2[j].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  unsigned long long *bad, *first;
  cudaMalloc(&bad, 8); cudaMalloc(&first, 8);
  cudaMemset(bad, 0, 8);
  k_fhfma<<<148 * 8, 256>>>(1ull << 30, bad);
  unsigned long long h = 0, f = 0;
  cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
  printf("fhfma_vs_ffma samples=%llu mismatches=%llu\n", 1ull << 30, h);
  for (int d : {32, 64, 128, 256}) {
    const float c = (float)std::sqrt((double)d);
    const float r = (float)(1.0 / (double)c);   // checked below against the exact RN(1/c)
    const double rr = 1.0 / (double)c;
    const float rlo = nextafterf(r, 0.f), rhi = nextafterf(r, 1.f);
    const bool rn = std::fabs((double)r - rr) <= std::fabs((double)rlo - rr) && std::fabs((double)r - rr) <= std::fabs((double)rhi - rr);
    cudaMemset(bad, 0, 8); cudaMemset(first, 0xff, 8);
    k_div<<<148 * 16, 256>>>(c, r, bad, first);
    cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&f, first, 8, cudaMemcpyDeviceToHost);
    printf("div d=%d c=%.9g r=%.9g r_is_RN=%d mismatches_of_2^32=%llu first=0x%08llx\n", d, c, r, rn, h, h ? f : 0ull);
  }
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[3] = {"FHFMA.BF16", "FFMA", "FFMA2"};
  for (int mode = 0; mode < 3; ++mode) {
    const int iters = 20000;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k_tput<0><<<148 * 8, 256>>>(out, iters);
      if (mode == 1) k_tput<1><<<148 * 8, 256>>>(out, iters);
      if (mode == 2) k_tput<2><<<148 * 8, 256>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)148 * 8 * 256 * iters * (mode == 2 ? 4 : 8);   // instructions (thread level)
    printf("tput %-11s %.1f G thread-instr/s  (%.1f per SM per clk at 1.965 GHz)\n", names[mode], ops / ms / 1e6,
           ops / (ms * 1e-3) / 148 / 1.965e9);
  }
  return 0;
}
