// k_finish_pair.cu -- the finish (k_finish.cu) of TWO q-heads of a GQA unit
// in one CTA, over the union of their probe rows (LFPS_FLAG_PAIR_FINISH).
//
// The q-heads of a unit probe nearly the same rows (the union of a unit's
// four lists is ~8% larger than one list at C4), so one pass over the union
// serves both heads: the row staging (cp.async), the K/V shared-memory
// loads, the bf16 widening of V and the loop overhead are paid once per
// row instead of once per row and head.  Each head keeps its own canonical
// scores (computed for every union row, kept only for its members), its
// online softmax state, its C2 score list (indexed by the row's rank in the
// head's own probe list) and its checks -- bit-identical to the per-session
// kernel.
//
// Measured at C4: 157 µs against 95 µs for the per-session kernel (118
// registers -> 2 CTAs/SM: the row loop's latency is no longer hidden), so it
// is opt-in.  Only the fused case (C2 = probe for both heads) runs here; anything else
// (a gated head, k < |probe|, an oversized union) falls back to the
// per-session finish of both heads, one after the other.
//
// Union build: the two lists are marked in shared-memory bitmaps (logical
// index), OR-ed, and compacted with block scans into U[] in shared memory
// (behind the row stages): (row | members << 30, rank in head 0's list |
// rank in head 1's list << 16).
#include "finish.cuh"

namespace lfps {

namespace {

using namespace fin;

constexpr int kMaxPairRows = 2048;         // union entries staged in shared memory (16 KiB)

template <int PQ>
__global__ void __launch_bounds__(kThreads, 2) lfps_finish_pair_kernel(Ctx c, const __nv_bfloat16* q) {
  extern __shared__ __align__(128) uint8_t stages[];
  __shared__ FinishShared sh;
  const int tid = threadIdx.x, l8 = tid & 7;
  const int s0 = c.s_off + 2 * blockIdx.x, s1 = s0 + 1;
  pdl_wait();
  const int b = s0 / c.Hq, h = (s0 % c.Hq) / c.G;
  const int n = c.n_ctx[b];
  const int S = c.S;
  const int m = n - S;
  int* cnt0 = c.counts + (size_t)s0 * CNT_N;
  int* cnt1 = c.counts + (size_t)s1 * CNT_N;
  const int byp0 = c.bypass[s0], byp1 = c.bypass[s1];
  const int p0 = cnt0[CNT_PROBE], p1 = cnt1[CNT_PROBE];
  int k = (int)rint(c.frac * (double)n);
  if (k < 1) k = 1;
  const int W = (m + 31) / 32;
  const bool pair = !byp0 && !byp1 && k >= p0 && k >= p1 && p0 + p1 <= kMaxPairRows &&
                    2 * (size_t)W * 4 <= rows_smem(PQ * 16);
  if (!pair) {
    finish_session<PQ>(c, q, s0, stages, sh);
    __syncthreads();
    finish_session<PQ>(c, q, s1, stages, sh);
    pdl_trigger();
    return;
  }
  const long long t0 = now_clk();
  const int* pl0 = c.probe_idx + (size_t)s0 * c.list_cap;
  const int* pl1 = c.probe_idx + (size_t)s1 * c.list_cap;
  int2* U = reinterpret_cast<int2*>(stages + rows_smem(PQ * 16));   // [kMaxPairRows], behind the stages
  if (tid == 0) {
    cnt0[CNT_K] = k; cnt0[CNT_C2] = p0;
    cnt1[CNT_K] = k; cnt1[CNT_C2] = p1;
  }

  // ---- union of the two probe lists ---------------------------------------------------
  uint32_t* bm0 = reinterpret_cast<uint32_t*>(stages);
  uint32_t* bm1 = bm0 + W;
  for (int w = tid; w < 2 * W; w += kThreads) bm0[w] = 0u;
  __syncthreads();
  for (int j = tid; j < p0; j += kThreads) {
    const int i = __ldg(pl0 + j) - S;
    atomicOr(bm0 + (i >> 5), 1u << (i & 31));
  }
  for (int j = tid; j < p1; j += kThreads) {
    const int i = __ldg(pl1 + j) - S;
    atomicOr(bm1 + (i >> 5), 1u << (i & 31));
  }
  __syncthreads();
  int nu = 0, r0base = 0, r1base = 0;                   // running totals over the rounds
  for (int w0 = 0; w0 < W; w0 += kThreads) {
    const int w = w0 + tid;
    const uint32_t a = w < W ? bm0[w] : 0u, bb = w < W ? bm1[w] : 0u, u = a | bb;
    int tu, ta, tb;
    const int pu = scan256(__popc(u), sh.warp_sums, &tu);
    const int pa = scan256(__popc(a), sh.warp_sums, &ta);
    const int pb = scan256(__popc(bb), sh.warp_sums, &tb);
    int at = nu + pu, ra = r0base + pa, rb = r1base + pb;
    for (uint32_t x = u; x; x &= x - 1) {
      const int bit = __ffs(x) - 1;
      const uint32_t bitm = 1u << bit;
      const int ina = (a & bitm) != 0, inb = (bb & bitm) != 0;
      U[at++] = make_int2((int)((unsigned)(S + w * 32 + bit) | ((unsigned)ina << 30) |
                                ((unsigned)inb << 31)),
                          ra | (rb << 16));
      ra += ina;
      rb += inb;
    }
    nu += tu; r0base += ta; r1base += tb;
  }
  __syncthreads();                                       // U complete; bitmaps free

  // ---- one pass over the sinks and the union rows for both heads ---------------------
  const __nv_bfloat16* kb = krow(c, b, h, 0);
  const __nv_bfloat16* vb = vrow(c, b, h, 0);
  const Part<PQ> qa = ld_part<PQ>(q + (size_t)s0 * c.d, l8);
  const Part<PQ> qb = ld_part<PQ>(q + (size_t)s1 * c.d, l8);
  float* c2z0 = c.c2_score + (size_t)s0 * c.list_cap;
  float* c2z1 = c.c2_score + (size_t)s1 * c.list_cap;
  Attn<PQ> at0, at1;
  at0.init();
  at1.init();
  float chk0 = 0.0f, chk1 = 0.0f, mx0 = -INFINITY, mx1 = -INFINITY;
  const int2* US = U - S;
  stream_rows<kFused, PQ>(
      stages, kb, vb, S + nu, [&](int rid) { return rid < S ? rid : US[rid].x & 0x3fffffff; },
      [&](const Rows2& r) {
        const float2 za = score_rows<PQ>(r, qa, c.sqrt_d_f32);
        const float2 zb = score_rows<PQ>(r, qb, c.sqrt_d_f32);
#pragma unroll
        for (int i = 0; i < kR; ++i) {
          if (!r.ok[i]) continue;                       // only in the last tile
          const int rid = r.rid[i];
          const float z0 = i ? za.y : za.x, z1 = i ? zb.y : zb.x;
          int in0 = 1, in1 = 1, r0 = 0, r1 = 0;
          if (rid >= S) {
            const int2 e = US[rid];
            in0 = (e.x >> 30) & 1;
            in1 = ((unsigned)e.x >> 31) & 1;
            r0 = e.y & 0xffff;
            r1 = (unsigned)e.y >> 16;
          }
          const bool c2row = rid >= S;
          chk0 = in0 ? __fmaf_rn(z0, 0.0f, chk0) : chk0;
          chk1 = in1 ? __fmaf_rn(z1, 0.0f, chk1) : chk1;
          mx0 = (in0 && c2row) ? fmaxf(mx0, z0) : mx0;
          mx1 = (in1 && c2row) ? fmaxf(mx1, z1) : mx1;
          if (l8 == 0 && c2row) {
            if (in0) c2z0[r0] = z0;
            if (in1) c2z1[r1] = z1;
          }
          // online softmax of both heads over one widened V row; a head that
          // does not hold the row leaves its state untouched
          const float zl0 = z0 * kLog2e, zl1 = z1 * kLog2e;
          if (in0 && zl0 > at0.m) {
            const float f = ex2(at0.m - zl0);
            at0.s *= f;
#pragma unroll
            for (int e2 = 0; e2 < PQ; ++e2) at0.acc[e2] = fmul2(at0.acc[e2], make_float2(f, f));
            at0.m = zl0;
          }
          if (in1 && zl1 > at1.m) {
            const float f = ex2(at1.m - zl1);
            at1.s *= f;
#pragma unroll
            for (int e2 = 0; e2 < PQ; ++e2) at1.acc[e2] = fmul2(at1.acc[e2], make_float2(f, f));
            at1.m = zl1;
          }
          const float w0 = in0 ? ex2(zl0 - at0.m) : 0.0f;
          const float w1 = in1 ? ex2(zl1 - at1.m) : 0.0f;
          at0.s += w0;
          at1.s += w1;
          const Part<PQ> v = ld_part_s<PQ>(r.v[i], l8);
          const float2 a2 = make_float2(w0, w0), b2 = make_float2(w1, w1);
#pragma unroll
          for (int t = 0; t < PQ / 2; ++t) {
            const float2 lo = make_float2(bf_lo(v.a[t]), bf_lo(v.b[t]));
            const float2 hi = make_float2(bf_hi(v.a[t]), bf_hi(v.b[t]));
            if (in0) {
              at0.acc[2 * t] = ffma2(lo, a2, at0.acc[2 * t]);
              at0.acc[2 * t + 1] = ffma2(hi, a2, at0.acc[2 * t + 1]);
            }
            if (in1) {
              at1.acc[2 * t] = ffma2(lo, b2, at1.acc[2 * t]);
              at1.acc[2 * t + 1] = ffma2(hi, b2, at1.acc[2 * t + 1]);
            }
          }
        }
      });
  int* c2i0 = c.c2_idx + (size_t)s0 * c.list_cap;
  int* c2i1 = c.c2_idx + (size_t)s1 * c.list_cap;
  for (int j = tid; j < p0; j += kThreads) c2i0[j] = __ldg(pl0 + j);
  for (int j = tid; j < p1; j += kThreads) c2i1[j] = __ldg(pl1 + j);
  finish_tail<PQ>(c, s0, stages, sh, at0, chk0, mx0, t0);
  __syncthreads();
  finish_tail<PQ>(c, s1, stages, sh, at1, chk1, mx1, t0);
  pdl_trigger();
}

template <int PQ>
cudaError_t launch_pair_d(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st) {
  const size_t smem = rows_smem(c.d) + kMaxPairRows * sizeof(int2);
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(lfps_finish_pair_kernel<PQ>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(lfps_finish_pair_kernel<PQ>,
                               cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    set = true;
  }
  return launch_pdl(lfps_finish_pair_kernel<PQ>, dim3(c.s_cnt / 2), dim3(kThreads), smem, st, c, q);
}

}  // namespace

// G even and an even session range: the head-pair finish; otherwise the
// caller uses the per-session kernel.
cudaError_t launch_finish_pair(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st) {
  if (c.G % 2 != 0 || c.s_off % 2 != 0 || c.s_cnt % 2 != 0) return cudaErrorNotSupported;
  switch (c.d) {
    case 32: return launch_pair_d<2>(c, q, st);
    case 64: return launch_pair_d<4>(c, q, st);
    case 128: return launch_pair_d<8>(c, q, st);
    case 256: return launch_pair_d<16>(c, q, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lfps
