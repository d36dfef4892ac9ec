// frag.cuh -- half-warp bf16 row fragments: lane hl of a 16-lane half owns
// the PER = d/16 contiguous elements [hl*PER, hl*PER + PER) of a row.
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

namespace lfps {

template <int PER>
struct RawFrag {
  static constexpr int kWords = PER / 2;   // packed bf16 pairs
  uint32_t w[kWords];
};

// raw (still packed) load: 16 B / 8 B / 4 B per lane, read-only path
template <int PER>
__device__ __forceinline__ RawFrag<PER> ld_frag(const __nv_bfloat16* row, int hl) {
  RawFrag<PER> f;
  const uint16_t* r = reinterpret_cast<const uint16_t*>(row) + hl * PER;
  if constexpr (PER % 8 == 0) {
#pragma unroll
    for (int k = 0; k < PER / 8; ++k) {
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(r) + k);
      f.w[4 * k] = u.x; f.w[4 * k + 1] = u.y; f.w[4 * k + 2] = u.z; f.w[4 * k + 3] = u.w;
    }
  } else if constexpr (PER == 4) {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(r));
    f.w[0] = u.x; f.w[1] = u.y;
  } else {
    static_assert(PER == 2, "d must be 32, 64, 128 or 256");
    f.w[0] = __ldg(reinterpret_cast<const uint32_t*>(r));
  }
  return f;
}

template <int PER>
__device__ __forceinline__ void unpack(const RawFrag<PER>& f, float* out) {
#pragma unroll
  for (int t = 0; t < PER / 2; ++t) {
    out[2 * t] = __uint_as_float(f.w[t] << 16);
    out[2 * t + 1] = __uint_as_float(f.w[t] & 0xffff0000u);
  }
}

// canonical fp32 lane dot (devmath.sdot32): sequential in element order;
// bf16*bf16 products are exact in fp32, so the fused form rounds identically
template <int PER>
__device__ __forceinline__ float frag_dot(const RawFrag<PER>& k, const float* q) {
  float acc = 0.0f;
#pragma unroll
  for (int t = 0; t < PER / 2; ++t) {
    acc = __fmaf_rn(__uint_as_float(k.w[t] << 16), q[2 * t], acc);
    acc = __fmaf_rn(__uint_as_float(k.w[t] & 0xffff0000u), q[2 * t + 1], acc);
  }
  return acc;
}

}  // namespace lfps
