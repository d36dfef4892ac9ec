// k_attend.cu -- fused gather-softmax-PV over sinks and the selection (K5).
//
// Restates the output stage of decode_step (engine.py:173-181) and
// attention_output (attention.py:66-85): one joint max-shifted softmax over
// [sink logits, selected logits] and out = sum_j w_j V[j] over
// [0, S) u C2.  Sink logits use the same canonical fp32 dot as the probe
// scores; the selected logits are the stored Top-k scores.  fp32 math,
// fp32 output; checked against the fp64 oracle to 1e-5 relative L2.
// One CTA per session; a half-warp gathers one V row (16 B per lane).
#include "common.cuh"
#include "canon.cuh"

namespace lfps {

namespace {

constexpr int kThreads = 256;
constexpr int kHalves = kThreads / 16;

template <int PER>
__device__ __forceinline__ void load_frag(const __nv_bfloat16* row, int hl, float* out) {
  const uint16_t* r = reinterpret_cast<const uint16_t*>(row) + hl * PER;
  if constexpr (PER % 8 == 0) {
#pragma unroll
    for (int k = 0; k < PER / 8; ++k) {
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(r) + k);
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        out[k * 8 + 2 * t] = __uint_as_float(w[t] << 16);
        out[k * 8 + 2 * t + 1] = __uint_as_float(w[t] & 0xffff0000u);
      }
    }
  } else if constexpr (PER == 4) {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(r));
    out[0] = __uint_as_float(u.x << 16);
    out[1] = __uint_as_float(u.x & 0xffff0000u);
    out[2] = __uint_as_float(u.y << 16);
    out[3] = __uint_as_float(u.y & 0xffff0000u);
  } else {
    const uint32_t u = __ldg(reinterpret_cast<const uint32_t*>(r));
    out[0] = __uint_as_float(u << 16);
    out[1] = __uint_as_float(u & 0xffff0000u);
  }
}

template <int PER>
__global__ void __launch_bounds__(kThreads) lfps_attend_kernel(Ctx c, const __nv_bfloat16* q,
                                                          int exact_mode) {
  __shared__ float sink_z[32];
  __shared__ float red_max[kThreads / 32];
  __shared__ float part[kHalves][PER * 16];
  __shared__ float wsum[kHalves];
  const int s = blockIdx.x, tid = threadIdx.x;
  if (!exact_mode && c.bypass[s]) return;        // gate already wrote the output
  const int half = tid >> 4, hl = tid & 15;
  const int b = s / c.Hq, h = (s % c.Hq) / c.G;
  const int S = c.S;
  const int n2 = c.counts[(size_t)s * CNT_N + CNT_C2];
  const int* idx = c.c2_idx + (size_t)s * c.list_cap;
  const float* zc = c.c2_score + (size_t)s * c.list_cap;

  float qf[PER];
  load_frag<PER>(q + (size_t)s * c.d, hl, qf);
  // sink logits (canonical fp32 dot, same as probe scores)
  for (int i = half; i < S; i += kHalves) {
    float kf[PER];
    load_frag<PER>(krow(c, b, h, i), hl, kf);
    float acc = 0.0f;
#pragma unroll
    for (int e = 0; e < PER; ++e) acc = __fmaf_rn(kf[e], qf[e], acc);
    acc = half_fold(acc);
    if (hl == 0) sink_z[i] = __fdiv_rn(acc, c.sqrt_d_f32);
  }
  __syncthreads();
  // joint max
  float mx = -INFINITY;
  for (int j = tid; j < S + n2; j += kThreads) mx = fmaxf(mx, j < S ? sink_z[j] : zc[j - S]);
  for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(LFPS_FULL, mx, o));
  if ((tid & 31) == 0) red_max[tid >> 5] = mx;
  __syncthreads();
  mx = red_max[0];
#pragma unroll
  for (int w = 1; w < kThreads / 32; ++w) mx = fmaxf(mx, red_max[w]);

  // weighted V gather: two rows in flight per half-warp
  float acc[PER];
#pragma unroll
  for (int e = 0; e < PER; ++e) acc[e] = 0.0f;
  float ws = 0.0f;
  const int tot = S + n2;
  int j = half;
  for (; j + kHalves < tot; j += 2 * kHalves) {
    const int j1 = j + kHalves;
    const int r0 = j < S ? j : __ldg(idx + j - S);
    const int r1 = j1 < S ? j1 : __ldg(idx + j1 - S);
    const float w0 = expf((j < S ? sink_z[j] : __ldg(zc + j - S)) - mx);
    const float w1 = expf((j1 < S ? sink_z[j1] : __ldg(zc + j1 - S)) - mx);
    float v0[PER], v1[PER];
    load_frag<PER>(vrow(c, b, h, r0), hl, v0);
    load_frag<PER>(vrow(c, b, h, r1), hl, v1);
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[e] = fmaf(w1, v1[e], fmaf(w0, v0[e], acc[e]));
    ws += w0 + w1;
  }
  if (j < tot) {
    const int r0 = j < S ? j : __ldg(idx + j - S);
    const float w0 = expf((j < S ? sink_z[j] : __ldg(zc + j - S)) - mx);
    float v0[PER];
    load_frag<PER>(vrow(c, b, h, r0), hl, v0);
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[e] = fmaf(w0, v0[e], acc[e]);
    ws += w0;
  }
#pragma unroll
  for (int e = 0; e < PER; ++e) part[half][hl * PER + e] = acc[e];
  if (hl == 0) wsum[half] = ws;
  __syncthreads();
  float total = 0.0f;
#pragma unroll
  for (int k = 0; k < kHalves; ++k) total += wsum[k];
  float* out = c.out + (size_t)s * c.d;
  for (int t = tid; t < c.d; t += kThreads) {
    float o = 0.0f;
#pragma unroll
    for (int k = 0; k < kHalves; ++k) o += part[k][t];
    out[t] = o / total;
  }
}

template <int PER>
cudaError_t launch_attend_d(const Ctx& c, const __nv_bfloat16* q, int exact_mode, cudaStream_t st) {
  lfps_attend_kernel<PER><<<c.NS, kThreads, 0, st>>>(c, q, exact_mode);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attend(const Ctx& c, const __nv_bfloat16* q, int exact_mode, cudaStream_t st) {
  switch (c.d) {
    case 32: return launch_attend_d<2>(c, q, exact_mode, st);
    case 64: return launch_attend_d<4>(c, q, exact_mode, st);
    case 128: return launch_attend_d<8>(c, q, exact_mode, st);
    case 256: return launch_attend_d<16>(c, q, exact_mode, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lfps
