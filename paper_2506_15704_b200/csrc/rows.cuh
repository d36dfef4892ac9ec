// rows.cuh -- shared machinery of the row-gather kernels (k_finish.cu,
// k_attend.cu, k_score.cu): canonical fp32 row scores in 8-lane groups, the
// online-softmax attention state, and the cp.async-staged row pipeline.
// 256-thread CTAs.
#pragma once

#include "common.cuh"
#include "canon.cuh"
#include "ptx.cuh"

namespace lfps {
namespace rows {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kGroups8 = kThreads / 8;   // 8-lane row groups
constexpr int kR = 2;                    // stream_rows: max rows per 8-lane group per tile
// rows per group per tile for d = 16 PQ: two (one tile = 64 rows), one for
// d = 256 so that a stage stays at 32 KB
#ifndef LFPS_ROWS_R
#define LFPS_ROWS_R 2
#endif
__host__ __device__ constexpr int rows_per_group(int pq) { return pq >= 16 ? 1 : LFPS_ROWS_R; }
#ifndef LFPS_ROW_STAGES
#define LFPS_ROW_STAGES 2
#endif
constexpr int kStagesR = LFPS_ROW_STAGES;   // stream_rows: stages
#ifndef LFPS_ROW_CTAS
#define LFPS_ROW_CTAS (kStagesR == 2 ? 3 : 2)
#endif
constexpr int kRowCtas = LFPS_ROW_CTAS;   // resident stream_rows CTAs per SM (smem)
// dynamic shared memory of a stream_rows kernel (K block + V block per stage)
__host__ __device__ constexpr size_t rows_smem(int d) {
  return (size_t)kStagesR * kGroups8 * rows_per_group(d / 16) * d * 2 * 2;
}
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

// fma.rn.f32.bf16 (FHFMA.BF16): the exact bf16 x bf16 product added to an
// fp32 accumulator with ONE rounding -- the same IEEE operation as FFMA of the
// widened operands, without the widening (bit identity over 2^30 patterns
// incl. subnormals, and full FFMA issue rate: profiles/r01_arith_probe.txt).
// lo / hi select the bf16 halves of packed words.
__device__ __forceinline__ float fma_lo(uint32_t a, uint32_t b, float c) {
  float d;
  asm("{\n\t.reg .b16 al, ah, bl, bh;\n\t"
      "mov.b32 {al, ah}, %1;\n\tmov.b32 {bl, bh}, %2;\n\t"
      "fma.rn.f32.bf16 %0, al, bl, %3;\n\t}"
      : "=f"(d) : "r"(a), "r"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float fma_hi(uint32_t a, uint32_t b, float c) {
  float d;
  asm("{\n\t.reg .b16 al, ah, bl, bh;\n\t"
      "mov.b32 {al, ah}, %1;\n\tmov.b32 {bl, bh}, %2;\n\t"
      "fma.rn.f32.bf16 %0, ah, bh, %3;\n\t}"
      : "=f"(d) : "r"(a), "r"(b), "f"(c));
  return d;
}

// canonical partials of one row (devmath.sdot32): lane l8 accumulates partial
// l8 (pa) and partial l8 + 8 (pb), d/16 contiguous elements each in order from
// +0, then folds 8 in-lane; k and q are packed bf16
template <int PQ>
__device__ __forceinline__ float row_dot(const Part<PQ>& k, const Part<PQ>& q) {
  float pa = 0.0f, pb = 0.0f;
#pragma unroll
  for (int t = 0; t < PQ / 2; ++t) {
    pa = fma_lo(k.a[t], q.a[t], pa);
    pb = fma_lo(k.b[t], q.b[t], pb);
    pa = fma_hi(k.a[t], q.a[t], pa);
    pb = fma_hi(k.b[t], q.b[t], pb);
  }
  return __fadd_rn(pa, pb);
}

// canonical fp32 score of one row per 8-lane group -> z in all 8 lanes: fold
// 4, 2, 1 across the group, IEEE division.  Every lane of the warp must call
// it (full-warp shuffles): groups without a row pass any finite data.
template <int PQ>
__device__ __forceinline__ float row_score(const Part<PQ>& k, const Part<PQ>& q, float sqrt_d) {
  float v = row_dot<PQ>(k, q);
#pragma unroll
  for (int h = 4; h >= 1; h >>= 1) v = __fadd_rn(v, __shfl_xor_sync(LFPS_FULL, v, h));
  return __fdiv_rn(v, sqrt_d);
}

// ld_part from a 32-bit shared-window address (row start)
template <int PQ>
__device__ __forceinline__ Part<PQ> ld_part_s(uint32_t row, int l8) {
  Part<PQ> r;
  if constexpr (PQ % 8 == 0) {
#pragma unroll
    for (int t = 0; t < PQ / 2; t += 4) {
      asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(r.a[t]), "=r"(r.a[t + 1]), "=r"(r.a[t + 2]), "=r"(r.a[t + 3])
                   : "r"(row + (l8 * (PQ / 2) + t) * 4));
      asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(r.b[t]), "=r"(r.b[t + 1]), "=r"(r.b[t + 2]), "=r"(r.b[t + 3])
                   : "r"(row + ((l8 + 8) * (PQ / 2) + t) * 4));
    }
  } else if constexpr (PQ == 4) {
    asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(r.a[0]), "=r"(r.a[1]) : "r"(row + l8 * 8));
    asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(r.b[0]), "=r"(r.b[1]) : "r"(row + (l8 + 8) * 8));
  } else {
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(r.a[0]) : "r"(row + l8 * 4));
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(r.b[0]) : "r"(row + (l8 + 8) * 4));
  }
  return r;
}

// canonical scores of TWO rows per 8-lane group (a, b) -> (z_a, z_b) in all 8
// lanes.  Reduce-scatter: lanes 0-3 fold row a, lanes 4-7 row b, so one
// shuffle serves both rows at fold 4 and each lane divides once.  Every add
// is x_l + x_(l^h) of the same canonical tree as row_score (IEEE addition
// commutes), so the scores are bit-identical to devmath.sdot32.
template <int PQ>
__device__ __forceinline__ float2 row_score2(const Part<PQ>& ka, const Part<PQ>& kb,
                                             const Part<PQ>& q, float sqrt_d) {
  const float va = row_dot<PQ>(ka, q), vb = row_dot<PQ>(kb, q);
  const bool hi = (threadIdx.x & 4) != 0;
  float v = __fadd_rn(hi ? vb : va, __shfl_xor_sync(LFPS_FULL, hi ? va : vb, 4));
  v = __fadd_rn(v, __shfl_xor_sync(LFPS_FULL, v, 2));
  v = __fadd_rn(v, __shfl_xor_sync(LFPS_FULL, v, 1));
  const float z = __fdiv_rn(v, sqrt_d);
  const float zo = __shfl_xor_sync(LFPS_FULL, z, 4);
  return hi ? make_float2(zo, z) : make_float2(z, zo);
}

constexpr float kLog2e = 1.4426950408889634f;

// 2^x (MUFU.EX2, flush-to-zero): softmax weights in the base-2 domain
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
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

// Online-softmax state of one 8-lane row group (all 8 lanes hold m, s), in
// the base-2 domain: absorb() takes zl = z * log2(e), weights are
// 2^(zl - m).  fp32, checked against the fp64 oracle to a tolerance.
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
  __device__ __forceinline__ void absorb(float zl, const Part<PQ>& v) {
    if (zl > m) {
      const float r = ex2(m - zl);
      s *= r;
#pragma unroll
      for (int e = 0; e < PQ; ++e) acc[e] = fmul2(acc[e], make_float2(r, r));
      m = zl;
    }
    const float w = ex2(zl - m);
    s += w;
    const float2 w2 = make_float2(w, w);
#pragma unroll
    for (int t = 0; t < PQ / 2; ++t) {
      acc[2 * t] = ffma2(make_float2(bf_lo(v.a[t]), bf_lo(v.b[t])), w2, acc[2 * t]);
      acc[2 * t + 1] = ffma2(make_float2(bf_hi(v.a[t]), bf_hi(v.b[t])), w2, acc[2 * t + 1]);
    }
  }
  // two rows at once (one max test / rescale)
  __device__ __forceinline__ void absorb2(float za, const Part<PQ>& va, float zb, const Part<PQ>& vb) {
    const float zm = fmaxf(za, zb);
    if (zm > m) {
      const float r = ex2(m - zm);
      s *= r;
#pragma unroll
      for (int e = 0; e < PQ; ++e) acc[e] = fmul2(acc[e], make_float2(r, r));
      m = zm;
    }
    const float wa = ex2(za - m), wb = ex2(zb - m);
    s += wa + wb;
    const float2 a2 = make_float2(wa, wa), b2 = make_float2(wb, wb);
#pragma unroll
    for (int t = 0; t < PQ / 2; ++t) {
      acc[2 * t] = ffma2(make_float2(bf_lo(va.a[t]), bf_lo(va.b[t])), a2, acc[2 * t]);
      acc[2 * t + 1] = ffma2(make_float2(bf_hi(va.a[t]), bf_hi(va.b[t])), a2, acc[2 * t + 1]);
    }
#pragma unroll
    for (int t = 0; t < PQ / 2; ++t) {
      acc[2 * t] = ffma2(make_float2(bf_lo(vb.a[t]), bf_lo(vb.b[t])), b2, acc[2 * t]);
      acc[2 * t + 1] = ffma2(make_float2(bf_hi(vb.a[t]), bf_hi(vb.b[t])), b2, acc[2 * t + 1]);
    }
  }
};



// The rows of one tile an 8-lane group owns: tile rows grp and grp + 32
// (row 1 only when rows_per_group = 2; otherwise ok[1] = false).  rid = list
// entry, ok = rid < nrows (ok[1] implies ok[0]), k / v = 32-bit shared
// addresses of the staged K and V rows.
struct Rows2 {
  int rid[kR];
  bool ok[kR];
  uint32_t k[kR], v[kR];
};

// scores of a group's staged rows (k[0], k[1] when present) -> (z0, z1)
template <int PQ, typename RowsT>
__device__ __forceinline__ float2 score_rows(const RowsT& r, const Part<PQ>& q, float sqrt_d) {
  const int l8 = threadIdx.x & 7;
  if constexpr (rows_per_group(PQ) == 2) {
    return row_score2<PQ>(ld_part_s<PQ>(r.k[0], l8), ld_part_s<PQ>(r.k[1], l8), q, sqrt_d);
  } else {
    const float z = row_score<PQ>(ld_part_s<PQ>(r.k[0], l8), q, sqrt_d);
    return make_float2(z, z);
  }
}

// Stream rows [0, nrows) through shared memory, kStagesR tiles of
// 32 x rows_per_group rows deep (each 8-lane group stages and reads only its
// own rows: warp barriers only): every thread copies 16-byte chunks of its group's rows
// (cp.async, L2 only), 8 threads per row; row_of(rid) gives the cache row of
// list entry rid.  visit(const Rows2&) is called by EVERY thread for every
// tile, so visits may use full-warp shuffles; a row with ok = false has a
// stale stage slot (any bits) that the visit must not commit.  Each thread
// fetches its row indices one tile before it issues the copies, so the index
// loads are off the critical path.
template <int MODE, int PQ, typename RowOf, typename Visit>
__device__ __forceinline__ void stream_rows(uint8_t* stages, const __nv_bfloat16* kb,
                                            const __nv_bfloat16* vb, int nrows, RowOf row_of,
                                            Visit visit) {
  constexpr bool kK = MODE != kAttend, kV = MODE != kScore;
  constexpr int D = PQ * 16;
  constexpr int kRowB = D * 2;                        // bytes per row
  constexpr int kChunks = kRowB / 16;                 // 16-byte chunks per row
  constexpr int R = rows_per_group(PQ);
  constexpr int kTileR = kGroups8 * R;                // rows per tile
  constexpr int kBlkB = kTileR * kRowB;               // K block (then V block) of a stage
  constexpr int kStageB = 2 * kBlkB;
  constexpr int kRowStep = kGroups8 * kRowB;          // group row 0 -> group row 1
  const int grp = threadIdx.x >> 3, l8 = threadIdx.x & 7;
  const int ntiles = (nrows + kTileR - 1) / kTileR;
  uint32_t sb0 = smem_u32(stages);
  asm volatile("" : "+r"(sb0));                       // kept in a register, not rematerialised per tile
  const uint32_t sb = sb0 + grp * kRowB;
  const uint32_t my_cp = sb + l8 * 16;                // this thread's first chunk, stage 0
  const uint8_t* kb8 = reinterpret_cast<const uint8_t*>(kb) + l8 * 16;
  const uint8_t* vb8 = reinterpret_cast<const uint8_t*>(vb) + l8 * 16;
  auto fetch = [&](int tile, int* row) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int rid = tile * kTileR + r * kGroups8 + grp;
      row[r] = rid < nrows ? row_of(rid) : -1;        // rid >= nrows also past the last tile
    }
  };
  auto issue = [&](int stage, const int* row) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (row[r] >= 0) {
        const uint32_t st = my_cp + stage * kStageB + r * kRowStep;
        const size_t off = (size_t)row[r] * kRowB;
#pragma unroll
        for (int ch = 0; ch < kChunks; ch += 8) {
          if (kChunks % 8 != 0 && ch + l8 >= kChunks) continue;   // d = 32: 4 chunks per row
          if (kK) cp_async16_s(st + ch * 16, kb8 + off + ch * 16);
          if (kV) cp_async16_s(st + kBlkB + ch * 16, vb8 + off + ch * 16);
        }
      }
    }
    cp_async_commit();                                // one group per tile, even if empty
  };
  int ahead[kR];
#pragma unroll 1
  for (int t = 0; t < kStagesR - 1; ++t) {
    fetch(t, ahead);
    issue(t, ahead);
  }
  fetch(kStagesR - 1, ahead);
  int rs = 0, ws = kStagesR - 1;                      // read / write stages
#pragma unroll 1
  for (int tile = 0; tile < ntiles; ++tile) {
    cp_async_wait<kStagesR - 2>();                    // this thread's copies of `tile` landed
    // A group's rows are copied by the group's own 8 lanes and read only by
    // them, so a warp barrier suffices: it publishes the warp's copies and
    // frees the warp's part of stage (tile - 1).  Warps run their tiles
    // independently (no CTA barrier per tile).
    __syncwarp();
    issue(ws, ahead);
    fetch(tile + kStagesR, ahead);
    ws = ws + 1 == kStagesR ? 0 : ws + 1;
    Rows2 rw;
    rw.ok[kR - 1] = false;
    rw.rid[kR - 1] = 0;
    rw.k[kR - 1] = rw.v[kR - 1] = 0u;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      rw.rid[r] = tile * kTileR + r * kGroups8 + grp;
      rw.ok[r] = rw.rid[r] < nrows;
      rw.k[r] = sb + rs * kStageB + r * kRowStep;
      rw.v[r] = rw.k[r] + kBlkB;
    }
    rs = rs + 1 == kStagesR ? 0 : rs + 1;
    visit(rw);
  }
  cp_async_wait<0>();
  __syncthreads();
}

}  // namespace rows
}  // namespace lfps
