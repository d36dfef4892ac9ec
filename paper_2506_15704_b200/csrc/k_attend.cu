// k_attend.cu -- exact-path attention (KX output stage).
//
// Restates the output of exact_topk_step (bench.py:73-80) / attention_output
// (attention.py:66-85): one joint max-shifted softmax over [sink logits,
// selected logits] and out = sum_j w_j V[j] over [0, S) u C2.  Sink logits
// use the canonical fp32 dot of the probe scores; the selected logits are
// the stored exact Top-k scores.  V rows stream through the cp.async-staged
// pipeline of rows.cuh; every 8-lane group keeps an online softmax state and
// the 32 states are merged at the end.  fp32 math and output, checked
// against the fp64 oracle to 1e-5 relative L2.  One CTA per session.
#include "rows.cuh"

namespace lfps {

namespace {

using namespace rows;

struct AttendShared {
  float sink_z[32];
  float part_m[kGroups8];
  float part_s[kGroups8];
};

template <int PQ>
__global__ void __launch_bounds__(kThreads, kRowCtas) lfps_exact_attend_kernel(Ctx c, const __nv_bfloat16* q) {
  extern __shared__ __align__(128) uint8_t stages[];
  __shared__ AttendShared sh;
  const int s = blockIdx.x, tid = threadIdx.x;
  const int l8 = tid & 7, grp = tid >> 3;
  const int b = s / c.Hq, h = (s % c.Hq) / c.G;
  const int S = c.S;
  const int k2 = c.counts[(size_t)s * CNT_N + CNT_C2];
  const int* c2i = c.c2_idx + (size_t)s * c.list_cap;
  const float* c2z = c.c2_score + (size_t)s * c.list_cap;
  // contiguous: the unit's base, unit-local rows; block table: pool rows
  const RowMap rmap(c, b, h);
  const __nv_bfloat16* kb = c.bt ? c.K : krow(c, b, h, 0);
  const __nv_bfloat16* vb = c.bt ? c.V : vrow(c, b, h, 0);
  auto rm = [&](int r) { return c.bt ? rmap(r) : r; };
  const Part<PQ> qp = ld_part<PQ>(q + (size_t)s * c.d, l8);
  stream_rows<kScore, PQ>(
      stages, kb, vb, S, [&](int rid) { return rm(rid); },
      [&](const Rows2& r) {
        const float2 z = score_rows<PQ>(r, qp, c.sqrt_d_f32);
        if (l8 == 0 && r.ok[0]) sh.sink_z[r.rid[0]] = z.x;
        if (l8 == 0 && r.ok[1]) sh.sink_z[r.rid[1]] = z.y;
      });
  Attn<PQ> at;
  at.init();
  auto zof = [&](int rid) { return (rid < S ? sh.sink_z[rid] : __ldg(c2z + rid - S)) * kLog2e; };
  stream_rows<kAttend, PQ>(
      stages, kb, vb, S + k2, [&](int rid) { return rm(rid < S ? rid : __ldg(c2i + rid - S)); },
      [&](const Rows2& r) {
        if (r.ok[1]) {
          at.absorb2(zof(r.rid[0]), ld_part_s<PQ>(r.v[0], l8), zof(r.rid[1]), ld_part_s<PQ>(r.v[1], l8));
        } else if (r.ok[0]) {
          at.absorb(zof(r.rid[0]), ld_part_s<PQ>(r.v[0], l8));
        }
      });
  // merge the 32 group states (stages reused as scratch)
  constexpr int D = PQ * 16;
  constexpr int kG = kThreads / D;
  constexpr int kPer = kGroups8 / kG;
  float* part = reinterpret_cast<float*>(stages);
#pragma unroll
  for (int e = 0; e < PQ; ++e) {
    part[grp * D + l8 * PQ + e] = at.acc[e].x;
    part[grp * D + (l8 + 8) * PQ + e] = at.acc[e].y;
  }
  if (l8 == 0) { sh.part_m[grp] = at.m; sh.part_s[grp] = at.s; }
  __syncthreads();
  float M = -INFINITY;
#pragma unroll 8
  for (int x = 0; x < kGroups8; ++x) M = fmaxf(M, sh.part_m[x]);
  const int t = tid % D, g = tid / D;
  float num = 0.0f, den = 0.0f;
#pragma unroll
  for (int xi = 0; xi < kPer; ++xi) {
    const int x = g * kPer + xi;
    if (sh.part_m[x] == -INFINITY) continue;
    const float f = ex2(sh.part_m[x] - M);
    num = fmaf(f, part[x * D + t], num);
    den = fmaf(f, sh.part_s[x], den);
  }
  __syncthreads();
  part[g * D + t] = num;
  part[kG * D + g * D + t] = den;
  __syncthreads();
  if (tid < D) {
    float nsum = 0.0f, dsum = 0.0f;
#pragma unroll
    for (int x = 0; x < kG; ++x) {
      nsum += part[x * D + tid];
      dsum += part[kG * D + x * D + tid];
    }
    c.out[(size_t)s * c.d + tid] = nsum / dsum;
  }
}

template <int PQ>
cudaError_t launch_attend_d(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st) {
  const size_t smem = rows_smem(c.d);
  static DeviceOnce once;
  cudaError_t e = once.run([&] {
    return cudaFuncSetAttribute(lfps_exact_attend_kernel<PQ>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (e != cudaSuccess) return e;
  lfps_exact_attend_kernel<PQ><<<c.NS, kThreads, smem, st>>>(c, q);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attend(const Ctx& c, const __nv_bfloat16* q, int /*exact_mode*/, cudaStream_t st) {
  switch (c.d) {
    case 32: return launch_attend_d<2>(c, q, st);
    case 64: return launch_attend_d<4>(c, q, st);
    case 128: return launch_attend_d<8>(c, q, st);
    case 256: return launch_attend_d<16>(c, q, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lfps
