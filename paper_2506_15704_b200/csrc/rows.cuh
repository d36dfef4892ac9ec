// rows.cuh -- shared machinery of the row-gather kernels (k_finish.cu,
// k_attend.cu, k_score.cu): canonical fp32 row scores in 8-lane groups with
// packed FFMA2, the online-softmax attention state, and the cp.async-staged
// row pipeline.  256-thread CTAs.
#pragma once

#include "common.cuh"
#include "canon.cuh"
#include "ptx.cuh"

namespace lfps {
namespace rows {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kGroups8 = kThreads / 8;   // 8-lane row groups
constexpr int kTile = 32;                // rows per stage (one per row group)
constexpr int kStages = 3;
constexpr int kCanon = 256;              // canonical block-sum width (devmath.BLOCK_THREADS)
constexpr int kMaxE = 8;                 // exponentials cached per thread (|C2| <= 2048)

enum Mode { kFused = 0, kScore = 1, kAttend = 2 };

// ---- packed fp32x2 arithmetic (FFMA2 / FMUL2: each half rounds like FFMA / FMUL) ----
__device__ __forceinline__ unsigned long long pk2(float2 v) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y));
  return r;
}
__device__ __forceinline__ float2 up2(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)), "l"(pk2(c)));
  return up2(r);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
  return up2(r);
}
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// PQ = d / 16 elements per canonical partial; a lane holds partials a = l8
// and b = l8 + 8 of a row, PQ / 2 packed bf16 words each
template <int PQ>
struct Part {
  uint32_t a[PQ / 2], b[PQ / 2];
};

template <int PQ>
__device__ __forceinline__ Part<PQ> ld_part(const __nv_bfloat16* row, int l8) {
  Part<PQ> r;
  const uint32_t* p = reinterpret_cast<const uint32_t*>(row);
  if constexpr (PQ % 8 == 0) {            // 16-byte vector loads
#pragma unroll
    for (int t = 0; t < PQ / 2; t += 4) {
      const uint4 x = *reinterpret_cast<const uint4*>(p + l8 * (PQ / 2) + t);
      const uint4 y = *reinterpret_cast<const uint4*>(p + (l8 + 8) * (PQ / 2) + t);
      r.a[t] = x.x; r.a[t + 1] = x.y; r.a[t + 2] = x.z; r.a[t + 3] = x.w;
      r.b[t] = y.x; r.b[t + 1] = y.y; r.b[t + 2] = y.z; r.b[t + 3] = y.w;
    }
  } else {
#pragma unroll
    for (int t = 0; t < PQ / 2; ++t) {
      r.a[t] = p[l8 * (PQ / 2) + t];
      r.b[t] = p[(l8 + 8) * (PQ / 2) + t];
    }
  }
  return r;
}

// canonical fp32 dot of one row with q (devmath.sdot32) -> z, all 8 lanes
template <int PQ>
__device__ __forceinline__ float row_score(const Part<PQ>& k, const float2* q2, float sqrt_d) {
  float2 p = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int t = 0; t < PQ / 2; ++t) {
    p = ffma2(make_float2(bf_lo(k.a[t]), bf_lo(k.b[t])), q2[2 * t], p);
    p = ffma2(make_float2(bf_hi(k.a[t]), bf_hi(k.b[t])), q2[2 * t + 1], p);
  }
  float v = __fadd_rn(p.x, p.y);                        // fold 8 (in-lane)
  // only this 8-lane group takes part: groups of a warp may hold no row
  const unsigned gm = 0xffu << (threadIdx.x & 24);
#pragma unroll
  for (int h = 4; h >= 1; h >>= 1) v = __fadd_rn(v, __shfl_xor_sync(gm, v, h));
  return __fdiv_rn(v, sqrt_d);
}


// exclusive block scan over the 256 threads
__device__ __forceinline__ int scan256(int v, int* warp_sums, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(LFPS_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  int before = 0, all = 0;
#pragma unroll
  for (int k = 0; k < kWarps; ++k) {
    const int w = warp_sums[k];
    before += k < warp ? w : 0;
    all += w;
  }
  __syncthreads();
  *total = all;
  return before + x - v;
}

// canonical 256-wide block sum (devmath.block_sum); all threads get it
__device__ __forceinline__ double canon_sum(double acc, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  acc = warp_fold(acc);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (warp == 0) {
    double v = lane < 8 ? red[lane] : 0.0;
#pragma unroll
    for (int h = 4; h >= 1; h >>= 1) v = cadd(v, __shfl_xor_sync(LFPS_FULL, v, h));
    if (lane == 0) red[8] = v;
  }
  __syncthreads();
  const double out = red[8];
  __syncthreads();
  return out;
}

// Online-softmax state of one 8-lane row group (all 8 lanes hold m, s).
template <int PQ>
struct Attn {
  float m, s;
  float2 acc[PQ];     // dims (a * PQ + e, b * PQ + e)
  __device__ __forceinline__ void init() {
    m = -INFINITY;
    s = 0.0f;
#pragma unroll
    for (int e = 0; e < PQ; ++e) acc[e] = make_float2(0.0f, 0.0f);
  }
  __device__ __forceinline__ void absorb(float z, const Part<PQ>& v) {
    if (z > m) {
      const float r = __expf(m - z);
      s *= r;
#pragma unroll
      for (int e = 0; e < PQ; ++e) acc[e] = fmul2(acc[e], make_float2(r, r));
      m = z;
    }
    const float w = __expf(z - m);
    s += w;
    const float2 w2 = make_float2(w, w);
#pragma unroll
    for (int t = 0; t < PQ / 2; ++t) {
      acc[2 * t] = ffma2(make_float2(bf_lo(v.a[t]), bf_lo(v.b[t])), w2, acc[2 * t]);
      acc[2 * t + 1] = ffma2(make_float2(bf_hi(v.a[t]), bf_hi(v.b[t])), w2, acc[2 * t + 1]);
    }
  }
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Stream rows [0, nrows) through shared memory, kStages tiles of kTile rows
// deep: every thread copies 16-byte chunks of one row (cp.async, L2 only),
// 8 threads per row; row_of(rid) gives the cache row of list entry rid, and
// visit(rid, k_row, v_row) consumes a staged row (8-lane group `grp` owns
// tile row `grp`).  Each thread fetches its row index one tile before it
// issues the copies, so the index load is off the critical path.
template <int MODE, int PQ, typename RowOf, typename Visit>
__device__ __forceinline__ void stream_rows(const Ctx& c, uint8_t* stages,
                                            const __nv_bfloat16* kb, const __nv_bfloat16* vb,
                                            int nrows, RowOf row_of, Visit visit) {
  constexpr bool kK = MODE != kAttend, kV = MODE != kScore;
  constexpr int D = PQ * 16;
  constexpr int kRowB = D * 2;                        // bytes per row
  constexpr int kChunks = kRowB / 16;                 // 16-byte chunks per row
  constexpr int kStageB = kTile * kRowB * 2;          // K block then V block
  const int grp = threadIdx.x >> 3, l8 = threadIdx.x & 7;
  const int ntiles = (nrows + kTile - 1) / kTile;
  auto fetch = [&](int tile) {
    const int rid = tile * kTile + grp;
    return (tile < ntiles && rid < nrows) ? row_of(rid) : -1;
  };
  auto issue = [&](int tile, int row) {
    if (tile < ntiles && row >= 0) {
      uint8_t* st = stages + (size_t)(tile % kStages) * kStageB + grp * kRowB;
#pragma unroll
      for (int ch = l8; ch < kChunks; ch += 8) {
        if (kK) cp_async16(st + ch * 16, reinterpret_cast<const uint8_t*>(kb + (size_t)row * D) + ch * 16);
        if (kV) cp_async16(st + kTile * kRowB + ch * 16,
                           reinterpret_cast<const uint8_t*>(vb + (size_t)row * D) + ch * 16);
      }
    }
    cp_async_commit();                                // one group per tile, even if empty
  };
#pragma unroll 1
  for (int t = 0; t < kStages - 1; ++t) issue(t, fetch(t));
  int ahead = fetch(kStages - 1);
#pragma unroll 1
  for (int tile = 0; tile < ntiles; ++tile) {
    cp_async_wait<kStages - 2>();                     // this thread's copies of `tile` landed
    __syncthreads();                                  // everyone's; stage (tile - 1) is free
    issue(tile + kStages - 1, ahead);
    ahead = fetch(tile + kStages);
    const uint8_t* st = stages + (size_t)(tile % kStages) * kStageB;
    const int rid = tile * kTile + grp;
    if (rid < nrows)
      visit(rid, reinterpret_cast<const __nv_bfloat16*>(st + grp * kRowB),
            reinterpret_cast<const __nv_bfloat16*>(st + (kTile + grp) * kRowB));
  }
  cp_async_wait<0>();
  __syncthreads();
}

}  // namespace rows
}  // namespace lfps
