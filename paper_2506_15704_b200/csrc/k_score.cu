// k_score.cu -- exact full-scan scoring (KX): every non-sink row of a
// (request, KV-head) unit scored against all G query heads of the unit.
//
// Restates the scoring half of exact_topk_step (bench.py:73-80): z_j =
// (K[j] . q) / fp32(sqrt d) for j in [S, n), in the canonical fp32 order of
// devmath.sdot32 (the same order as the decode path's probe scores, so the
// exact and the LFPS selections compare like for like).  The K stream is the
// HBM-bound part of the exact path: each row is read ONCE for the G heads
// (the GQA GEMV); 8 lanes own a row (lane l: canonical partials l and l + 8,
// two chains in one packed FFMA2 per element; the bf16 widening is shared
// by the G heads).  K rows stream through shared memory with cp.async, 4
// tiles of 64 rows in flight per CTA, each group staging its own rows.
// Scores land in probe_score[s][j - S] (implicit index list).
#include "rows.cuh"

namespace lfps {

namespace {

using namespace rows;

constexpr int kR = 2;                       // rows per 8-lane group per tile
#ifndef LFPS_SCORE_CTAS
#define LFPS_SCORE_CTAS 2
#endif
// tiles in flight (cp.async stages): 64 KiB of K per CTA
__host__ __device__ constexpr int score_stages(int pq) { return pq >= 16 ? 2 : 4; }

template <int PQ>
__device__ __forceinline__ Part<PQ> ldg_part(const __nv_bfloat16* row, int l8) {
  Part<PQ> r;
  const uint32_t* p = reinterpret_cast<const uint32_t*>(row);
  if constexpr (PQ % 8 == 0) {
#pragma unroll
    for (int t = 0; t < PQ / 2; t += 4) {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(p + l8 * (PQ / 2) + t));
      const uint4 y = __ldg(reinterpret_cast<const uint4*>(p + (l8 + 8) * (PQ / 2) + t));
      r.a[t] = x.x; r.a[t + 1] = x.y; r.a[t + 2] = x.z; r.a[t + 3] = x.w;
      r.b[t] = y.x; r.b[t + 1] = y.y; r.b[t + 2] = y.z; r.b[t + 3] = y.w;
    }
  } else {
#pragma unroll
    for (int t = 0; t < PQ / 2; ++t) {
      r.a[t] = __ldg(p + l8 * (PQ / 2) + t);
      r.b[t] = __ldg(p + (l8 + 8) * (PQ / 2) + t);
    }
  }
  return r;
}

// The canonical folds at lane distances LVL .. 1 of N values per lane (one
// per head) as a reduce-scatter: at each level the lanes whose LVL bit is
// set keep the upper half of the values, the others the lower half, so that
// the lane ends with the full sum of value (l8 / (8 / N)) and each level
// costs N / 2 shuffles.  Every add is x_l + x_(l^LVL) of devmath.sdot32's
// tree (IEEE addition commutes), bit-identical to N butterflies.
template <int N, int LVL>
struct FoldScatter {
  static __device__ __forceinline__ float run(const float (&v)[N], int l8) {
    if constexpr (N == 1) {
      float x = v[0];
#pragma unroll
      for (int o = LVL; o >= 1; o >>= 1) x = __fadd_rn(x, __shfl_xor_sync(LFPS_FULL, x, o));
      return x;
    } else {
      const bool hi = (l8 & LVL) != 0;
      float keep[N / 2];
#pragma unroll
      for (int i = 0; i < N / 2; ++i) {
        const float send = hi ? v[i] : v[i + N / 2];
        keep[i] = __fadd_rn(hi ? v[i + N / 2] : v[i], __shfl_xor_sync(LFPS_FULL, send, LVL));
      }
      return FoldScatter<N / 2, LVL / 2>::run(keep, l8);
    }
  }
};

// RM: RowMapT mode -- 0 contiguous cache (unit base, local rows), 1 block table
template <int PQ, int G, int RM>
__global__ void __launch_bounds__(kThreads, LFPS_SCORE_CTAS) lfps_exact_score_kernel(Ctx c, const __nv_bfloat16* q) {
  const int u = blockIdx.y;
  const int b = u / c.Hkv, h = u % c.Hkv;
  const int n = c.n_ctx[b];
  const int S = c.S;
  const int m = n - S;
  const int l8 = threadIdx.x & 7, grp = threadIdx.x >> 3;
  const int s0 = b * c.Hq + h * G;
  // this CTA's contiguous row chunk
  constexpr int kStep = kGroups8 * kR;
  const int per = ((m + gridDim.x - 1) / gridDim.x + kStep - 1) / kStep * kStep;
  const int r0 = blockIdx.x * per;
  const int r1 = min(m, r0 + per);
  if (blockIdx.x == 0 && threadIdx.x < G) c.counts[(size_t)(s0 + threadIdx.x) * CNT_N + CNT_PROBE] = m;
  if (r0 >= r1) return;
  float2 q2[G][PQ];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const Part<PQ> qp = ldg_part<PQ>(q + (size_t)(s0 + g) * c.d, l8);
#pragma unroll
    for (int t = 0; t < PQ / 2; ++t) {
      q2[g][2 * t] = make_float2(bf_lo(qp.a[t]), bf_lo(qp.b[t]));
      q2[g][2 * t + 1] = make_float2(bf_hi(qp.a[t]), bf_hi(qp.b[t]));
    }
  }
  // contiguous: the unit's base in registers, unit-local rows; block table:
  // the pool base, pool rows (RowMap)
  const RowMapT<RM> rmap(c, b, h);
  const __nv_bfloat16* kbase = RM ? c.K : krow(c, b, h, 0);
  auto rm = [&](int r) { return RM ? rmap(r) : r; };
  const int gs = l8 / (8 / G);                        // the head this lane divides and writes
  const bool writer = l8 % (8 / G) == 0;
  float* out = c.probe_score + (size_t)(s0 + gs) * c.list_cap;
  // K rows stream through shared memory, kScoreStages tiles of kStep rows:
  // each 8-lane group copies (cp.async) and reads only its own rows, so the
  // warps run independently with warp barriers only
  extern __shared__ __align__(128) uint8_t kst[];
  constexpr int kScoreStages = score_stages(PQ);
  constexpr int kRowB = PQ * 32;                      // bytes per K row
  constexpr int kChunks = kRowB / 16;
  constexpr int kStageB = kStep * kRowB;
  const uint32_t sb = smem_u32(kst) + grp * kRowB;
  const uint8_t* kb8 = reinterpret_cast<const uint8_t*>(kbase) + l8 * 16;
  const int ntiles = (r1 - r0 + kStep - 1) / kStep;
  auto issue = [&](int tile) {
    if (tile < ntiles) {
      const uint32_t st = sb + (tile % kScoreStages) * kStageB + l8 * 16;
#pragma unroll
      for (int i = 0; i < kR; ++i) {
        const int row = r0 + tile * kStep + grp + kGroups8 * i;
        if (row < r1) {
#pragma unroll
          for (int ch = 0; ch < kChunks; ch += 8) {
            if (kChunks % 8 != 0 && ch + l8 >= kChunks) continue;
            cp_async16_s(st + i * kGroups8 * kRowB + ch * 16,
                         kb8 + (size_t)rm(S + row) * kRowB + ch * 16);
          }
        }
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int t = 0; t < kScoreStages - 1; ++t) issue(t);
#pragma unroll 1
  for (int tile = 0; tile < ntiles; ++tile) {         // uniform trip count: full-warp shuffles
    cp_async_wait<kScoreStages - 2>();
    __syncwarp();
    issue(tile + kScoreStages - 1);
    const uint32_t st = sb + (tile % kScoreStages) * kStageB;
#pragma unroll
    for (int i = 0; i < kR; ++i) {
      const int rr = r0 + tile * kStep + grp + kGroups8 * i;
      const Part<PQ> kr = ld_part_s<PQ>(st + i * kGroups8 * kRowB, l8);
      float2 kp[PQ];
#pragma unroll
      for (int t = 0; t < PQ / 2; ++t) {
        kp[2 * t] = make_float2(bf_lo(kr.a[t]), bf_lo(kr.b[t]));
        kp[2 * t + 1] = make_float2(bf_hi(kr.a[t]), bf_hi(kr.b[t]));
      }
      float v[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float2 p = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int e = 0; e < PQ; ++e) p = ffma2(kp[e], q2[g][e], p);
        v[g] = __fadd_rn(p.x, p.y);                 // canonical fold 8 (in-lane)
      }
      // folds 4, 2, 1 as a reduce-scatter over the heads: lane l8 ends with
      // head gs's score
      const float z = __fdiv_rn(FoldScatter<G, 4>::run(v, l8), c.sqrt_d_f32);
      if (rr < r1 && writer) out[rr] = z;
    }
  }
  cp_async_wait<0>();
}

template <int PQ, int RM>
cudaError_t launch_exact_rm(const Ctx& c, const __nv_bfloat16* q, int m_max, cudaStream_t st) {
  const int units = c.B * c.Hkv;
  // ~4 waves of 148 SMs x 2 CTAs over all units, >= 1 step of rows per CTA
  int per_unit = (148 * 2 * 4 + units - 1) / units;
  const int cap = (m_max + kGroups8 * kR - 1) / (kGroups8 * kR);
  if (per_unit > cap) per_unit = cap;
  if (per_unit < 1) per_unit = 1;
  const dim3 grid(per_unit, units);
  const size_t smem = (size_t)score_stages(PQ) * kGroups8 * kR * PQ * 32;
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads, smem, st>>>(c, q);
    return cudaSuccess;
  };
  cudaError_t e;
  switch (c.G) {
    case 1: e = go(lfps_exact_score_kernel<PQ, 1, RM>); break;
    case 2: e = go(lfps_exact_score_kernel<PQ, 2, RM>); break;
    case 4: e = go(lfps_exact_score_kernel<PQ, 4, RM>); break;
    case 8: e = go(lfps_exact_score_kernel<PQ, 8, RM>); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int PQ>
cudaError_t launch_exact_d(const Ctx& c, const __nv_bfloat16* q, int m_max, cudaStream_t st) {
  return c.bt ? launch_exact_rm<PQ, 1>(c, q, m_max, st) : launch_exact_rm<PQ, 0>(c, q, m_max, st);
}

}  // namespace

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
