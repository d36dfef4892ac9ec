// k_score.cu -- candidate-only q.K scoring (K3) and the exact full scan (KX).
//
// fp32 score z = (K[j] . q) / fp32(sqrt d) in the canonical order of
// devmath.sdot32: a half-warp owns one bf16 key row (16 lanes x d/16
// contiguous elements, one 16-byte load per 8 elements), each lane
// accumulates its products in order (bf16 x bf16 products are exact in fp32,
// so the FMA equals multiply-then-add), the half folds 8, 4, 2, 1, then an
// IEEE division.  Restates engine.py:168-170 / numerics.py:33-49 with fp32
// accumulation (Top-k identical given fp32 scores).
//
// lfps_score_kernel: gathers the rows of each session's probe list.
// lfps_exact_score_kernel: streams every non-sink row of a (request, KV-head)
// once and scores it against all G query heads of the unit (GQA GEMV).
#include "common.cuh"
#include "canon.cuh"

namespace lfps {

namespace {

constexpr int kThreads = 256;
constexpr int kHalves = kThreads / 16;

template <int PER>
struct RowFrag {
  float v[PER];
};

// Load lane `hl`'s PER contiguous bf16 elements of a row as fp32.
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
    static_assert(PER == 2, "d must be 32, 64, 128 or 256");
    const uint32_t u = __ldg(reinterpret_cast<const uint32_t*>(r));
    out[0] = __uint_as_float(u << 16);
    out[1] = __uint_as_float(u & 0xffff0000u);
  }
}

template <int PER>
__device__ __forceinline__ float frag_dot(const float* k, const float* q) {
  float acc = 0.0f;
#pragma unroll
  for (int e = 0; e < PER; ++e) acc = __fmaf_rn(k[e], q[e], acc);
  return acc;
}

template <int PER>
__global__ void __launch_bounds__(kThreads) lfps_score_kernel(Ctx c, const __nv_bfloat16* q) {
  const int s = blockIdx.y;
  const int p = c.counts[(size_t)s * CNT_N + CNT_PROBE];
  const int half = threadIdx.x >> 4, hl = threadIdx.x & 15;
  const int first = blockIdx.x * kHalves + half;
  if (blockIdx.x * kHalves >= p) return;
  const int b = s / c.Hq, h = (s % c.Hq) / c.G;
  float qf[PER];
  load_frag<PER>(q + (size_t)s * c.d, hl, qf);
  const int* idx = c.probe_idx + (size_t)s * c.list_cap;
  float* out = c.probe_score + (size_t)s * c.list_cap;
  const int stride = gridDim.x * kHalves;
  const __nv_bfloat16* kbase = krow(c, b, h, 0);
  // two rows in flight per half-warp
  int j = first;
  for (; j + stride < p; j += 2 * stride) {
    float k0[PER], k1[PER];
    load_frag<PER>(kbase + (size_t)__ldg(idx + j) * c.d, hl, k0);
    load_frag<PER>(kbase + (size_t)__ldg(idx + j + stride) * c.d, hl, k1);
    const float z0 = half_fold(frag_dot<PER>(k0, qf));
    const float z1 = half_fold(frag_dot<PER>(k1, qf));
    if (hl == 0) {
      out[j] = __fdiv_rn(z0, c.sqrt_d_f32);
      out[j + stride] = __fdiv_rn(z1, c.sqrt_d_f32);
    }
  }
  if (j < p) {
    float k0[PER];
    load_frag<PER>(kbase + (size_t)__ldg(idx + j) * c.d, hl, k0);
    const float z0 = half_fold(frag_dot<PER>(k0, qf));
    if (hl == 0) out[j] = __fdiv_rn(z0, c.sqrt_d_f32);
  }
}

// Exact path: all rows [S, n) of unit u scored for its G sessions.
// Scores land in probe_score[s][row - S] (implicit index list).
template <int PER, int G>
__global__ void __launch_bounds__(kThreads) lfps_exact_score_kernel(Ctx c, const __nv_bfloat16* q) {
  const int u = blockIdx.y;
  const int b = u / c.Hkv, h = u % c.Hkv;
  const int n = c.n_ctx[b];
  const int S = c.S;
  const int m = n - S;
  const int half = threadIdx.x >> 4, hl = threadIdx.x & 15;
  const int s0 = b * c.Hq + h * G;
  float qf[G][PER];
#pragma unroll
  for (int g = 0; g < G; ++g) load_frag<PER>(q + (size_t)(s0 + g) * c.d, hl, qf[g]);
  const __nv_bfloat16* kbase = krow(c, b, h, S);
  const int stride = gridDim.x * kHalves;
  for (int j = blockIdx.x * kHalves + half; j < m; j += stride) {
    float kk[PER];
    load_frag<PER>(kbase + (size_t)j * c.d, hl, kk);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float z = half_fold(frag_dot<PER>(kk, qf[g]));
      if (hl == g) c.probe_score[(size_t)(s0 + g) * c.list_cap + j] = __fdiv_rn(z, c.sqrt_d_f32);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < G) {
    c.counts[(size_t)(s0 + threadIdx.x) * CNT_N + CNT_PROBE] = m;
  }
}

template <int PER>
cudaError_t launch_score_d(const Ctx& c, const __nv_bfloat16* q, int max_list, cudaStream_t st) {
  // enough CTAs to fill the machine (148 SMs x 8 resident CTAs), at least 2
  // per session; the probe count itself lives on the device (grid-stride).
  int per_session = (148 * 8 + c.NS - 1) / c.NS;
  const int cap = (max_list + kHalves - 1) / kHalves;
  if (per_session > cap) per_session = cap;
  if (per_session > 64) per_session = 64;
  if (per_session < 2) per_session = 2;
  lfps_score_kernel<PER><<<dim3(per_session, c.NS), kThreads, 0, st>>>(c, q);
  return cudaGetLastError();
}

template <int PER>
cudaError_t launch_exact_d(const Ctx& c, const __nv_bfloat16* q, int m_max, cudaStream_t st) {
  const int units = c.B * c.Hkv;
  // ~4 waves of 148 SMs x 8 CTAs over all units
  int per_unit = (148 * 8 * 4 + units - 1) / units;
  const int rows_cap = (m_max + kHalves - 1) / kHalves;
  if (per_unit > rows_cap) per_unit = rows_cap;
  if (per_unit < 1) per_unit = 1;
  const dim3 grid(per_unit, units);
  switch (c.G) {
    case 1: lfps_exact_score_kernel<PER, 1><<<grid, kThreads, 0, st>>>(c, q); break;
    case 2: lfps_exact_score_kernel<PER, 2><<<grid, kThreads, 0, st>>>(c, q); break;
    case 4: lfps_exact_score_kernel<PER, 4><<<grid, kThreads, 0, st>>>(c, q); break;
    case 8: lfps_exact_score_kernel<PER, 8><<<grid, kThreads, 0, st>>>(c, q); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_score(const Ctx& c, const __nv_bfloat16* q, int max_list, cudaStream_t st) {
  switch (c.d) {
    case 32: return launch_score_d<2>(c, q, max_list, st);
    case 64: return launch_score_d<4>(c, q, max_list, st);
    case 128: return launch_score_d<8>(c, q, max_list, st);
    case 256: return launch_score_d<16>(c, q, max_list, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_exact_score(const Ctx& c, const __nv_bfloat16* q, int m_max, cudaStream_t st) {
  switch (c.d) {
    case 32: return launch_exact_d<2>(c, q, m_max, st);
    case 64: return launch_exact_d<4>(c, q, m_max, st);
    case 128: return launch_exact_d<8>(c, q, m_max, st);
    case 256: return launch_exact_d<16>(c, q, m_max, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lfps
